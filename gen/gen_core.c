/* Planted-community graph generator core (input generation only; holds none of
 * the method's arithmetic).  See gen/planted.py for the recipe.
 *
 * gen_dcsbm: every node v emits floor(theta_v*scale + u_v) stubs; each stub
 * targets v's own community with probability 1-mu (target ~ theta inside the
 * community, by binary search of the theta prefix sums `cum`), else any node
 * (target ~ theta).  Self-loops are dropped; the multigraph is symmetrised,
 * each row sorted and de-duplicated.  Output is a CSR in malloc'd buffers the
 * caller frees with gen_free().  Randomness: splitmix64 streams keyed by
 * (seed, v) -- deterministic and independent of the thread count.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

static inline uint64_t splitmix64(uint64_t *s) {
    uint64_t z = (*s += 0x9E3779B97F4A7C15ull);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}
static inline double u01(uint64_t *s) { return (double)(splitmix64(s) >> 11) * 0x1.0p-53; }

static int64_t upper_search(const double *cum, int64_t lo, int64_t hi, double x) {
    /* largest i in [lo, hi) with cum[i] <= x (cum non-decreasing) */
    int64_t a = lo, b = hi - 1;
    while (a < b) {
        int64_t mid = a + (b - a + 1) / 2;
        if (cum[mid] <= x) a = mid; else b = mid - 1;
    }
    return a;
}

static int cmp_i32(const void *a, const void *b) {
    int32_t x = *(const int32_t *)a, y = *(const int32_t *)b;
    return (x > y) - (x < y);
}

void gen_free(void *p) { free(p); }

/* returns 0 on success; *indptr_out int64[n+1], *indices_out int32[*nnz_out] */
int gen_dcsbm(int64_t n, int32_t ncomm, const int64_t *cbeg, const int32_t *comm,
              const double *theta, const double *cum, double mu, double scale, uint64_t seed,
              int64_t **indptr_out, int32_t **indices_out, int64_t *nnz_out) {
    int64_t *nst = (int64_t *)malloc(sizeof(int64_t) * (n + 1));
    if (!nst) return 1;
    nst[0] = 0;
    for (int64_t v = 0; v < n; ++v) {
        uint64_t s = seed * 0xD1B54A32D192ED03ull ^ ((uint64_t)v * 0x9E3779B97F4A7C15ull);
        splitmix64(&s);
        nst[v + 1] = nst[v] + (int64_t)(theta[v] * scale + u01(&s));
    }
    int64_t m = nst[n];
    int32_t *src = (int32_t *)malloc(sizeof(int32_t) * (m ? m : 1));
    int32_t *tgt = (int32_t *)malloc(sizeof(int32_t) * (m ? m : 1));
    int64_t *deg = (int64_t *)calloc(n + 1, sizeof(int64_t));
    if (!src || !tgt || !deg) return 1;
    (void)ncomm;
#pragma omp parallel for schedule(dynamic, 4096)
    for (int64_t v = 0; v < n; ++v) {
        uint64_t s = seed * 0xA24BAED4963EE407ull ^ ((uint64_t)v * 0x9FB21C651E98DF25ull);
        splitmix64(&s);
        int32_t c = comm[v];
        double lo = cum[cbeg[c]], hi = cum[cbeg[c + 1]];
        for (int64_t k = nst[v]; k < nst[v + 1]; ++k) {
            double a = u01(&s), b = u01(&s);
            int64_t t;
            if (a < 1.0 - mu) {
                t = upper_search(cum, cbeg[c], cbeg[c + 1], lo + b * (hi - lo));
            } else {
                t = upper_search(cum, 0, n, b * cum[n]);
            }
            src[k] = (int32_t)v;
            tgt[k] = (t == v) ? -1 : (int32_t)t;
        }
    }
    for (int64_t k = 0; k < m; ++k) {
        if (tgt[k] < 0) continue;
        deg[src[k] + 1]++;
        deg[tgt[k] + 1]++;
    }
    for (int64_t v = 0; v < n; ++v) deg[v + 1] += deg[v];
    int32_t *adj = (int32_t *)malloc(sizeof(int32_t) * (deg[n] ? deg[n] : 1));
    int64_t *fill = (int64_t *)malloc(sizeof(int64_t) * (n + 1));
    if (!adj || !fill) return 1;
    memcpy(fill, deg, sizeof(int64_t) * (n + 1));
    for (int64_t k = 0; k < m; ++k) {
        if (tgt[k] < 0) continue;
        adj[fill[src[k]]++] = tgt[k];
        adj[fill[tgt[k]]++] = src[k];
    }
    free(src); free(tgt); free(nst);
    int64_t *rowlen = fill;  /* reuse */
#pragma omp parallel for schedule(dynamic, 1024)
    for (int64_t v = 0; v < n; ++v) {
        int32_t *r = adj + deg[v];
        int64_t len = deg[v + 1] - deg[v], w = 0;
        qsort(r, (size_t)len, sizeof(int32_t), cmp_i32);
        for (int64_t i = 0; i < len; ++i)
            if (w == 0 || r[i] != r[w - 1]) r[w++] = r[i];
        rowlen[v] = w;
    }
    int64_t *indptr = (int64_t *)malloc(sizeof(int64_t) * (n + 1));
    if (!indptr) return 1;
    indptr[0] = 0;
    for (int64_t v = 0; v < n; ++v) indptr[v + 1] = indptr[v] + rowlen[v];
    int32_t *indices = (int32_t *)malloc(sizeof(int32_t) * (indptr[n] ? indptr[n] : 1));
    if (!indices) return 1;
#pragma omp parallel for schedule(dynamic, 4096)
    for (int64_t v = 0; v < n; ++v)
        memcpy(indices + indptr[v], adj + deg[v], sizeof(int32_t) * (size_t)rowlen[v]);
    free(adj); free(deg); free(fill);
    *indptr_out = indptr;
    *indices_out = indices;
    *nnz_out = indptr[n];
    return 0;
}
