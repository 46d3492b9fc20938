/*
 * oracle.c -- plain, slow, single-threaded CPU oracle of the COMM-RAND
 * mini-batch hot path (arXiv 2504.18082).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library.
 * It shares no code, header, table or constant generator with the CUDA path
 * (paper_2504_18082_b200/csrc); neither side includes or links the other.
 *
 * Citations: P:n = /root/reference/PAPER.md line n (canonical copy
 * P:439-1088), S:n = SPEC.md line n.  "R<k>" = reading k in DESIGN.md
 * ("Readings of the paper"), where the paper is silent or ambiguous.
 *
 * Functions (each follows the definition it cites, step by step, with no
 * blocking, fusion or reordering):
 *   or_philox4x32_10   O1  counter-based RNG (Salmon et al. 2011, Philox4x32-10)   pinned: KAT
 *   or_mulhi64         O1  unif(r, n) = floor(r * n / 2^64)                       pinned: closed form
 *   or_graph_prep      a0  community offsets + per-row intra segment               pinned: brute force
 *   or_order_roots     a1  Knob-1 root order (Table 1; S4.1 P:653-680)  pinned: invariants, chi^2
 *   or_sample_hop      a2  Knob-2 biased fanout sampling (S4.2 P:683-691)   pinned: exact law, chi^2
 *   or_community_order NEXT-2 (iii) community reordering of an unordered graph     pinned: isomorphism, brute force
 *   or_relabel_hop     a3  dedup + relabel into a block (Alg.1 l.4)     pinned: brute force
 *   or_gather          a4  X_in = X[nodes]                                 pinned: memcmp
 *   or_sage_mean       a5  GraphSAGE mean aggregation               pinned: fp64 closed form
 *
 * Build: gcc -O2 -std=c11 -ffp-contract=off -fno-fast-math -shared -fPIC
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------ O1 */
/* Philox4x32-10 (Salmon, Moraes, Dror, Shaw, SC'11 "Parallel random numbers:
 * as easy as 1, 2, 3"): 10 rounds; before rounds 2..10 the key is bumped by
 * the Weyl constants.  Round: (hi0,lo0) = M0*c0, (hi1,lo1) = M1*c2,
 * c <- (hi1^c1^k0, lo1, hi0^c3^k1, lo0). */
void or_philox4x32_10(const uint32_t ctr_in[4], const uint32_t key_in[2], uint32_t out[4]) {
    const uint32_t M0 = 0xD2511F53u, M1 = 0xCD9E8D57u;
    const uint32_t W0 = 0x9E3779B9u, W1 = 0xBB67AE85u;
    uint32_t c0 = ctr_in[0], c1 = ctr_in[1], c2 = ctr_in[2], c3 = ctr_in[3];
    uint32_t k0 = key_in[0], k1 = key_in[1];
    for (int round = 0; round < 10; ++round) {
        if (round > 0) {
            k0 += W0;
            k1 += W1;
        }
        uint64_t p0 = (uint64_t)M0 * (uint64_t)c0;
        uint64_t p1 = (uint64_t)M1 * (uint64_t)c2;
        uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
        uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
        uint32_t n0 = hi1 ^ c1 ^ k0;
        uint32_t n1 = lo1;
        uint32_t n2 = hi0 ^ c3 ^ k1;
        uint32_t n3 = lo0;
        c0 = n0; c1 = n1; c2 = n2; c3 = n3;
    }
    out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

/* unif(r, n) = floor(r * n / 2^64) (reading R14: multiply-high, no rejection) */
uint64_t or_mulhi64(uint64_t r, uint64_t n) {
    unsigned __int128 prod = (unsigned __int128)r * (unsigned __int128)n;
    return (uint64_t)(prod >> 64);
}

/* Philox call with the counter layout of reading R11:
 * ctr = (slot, id, (tag << 24) | hop, batch_or_epoch), key = (seed lo, seed hi). */
static void draw(uint64_t seed, uint32_t slot, uint32_t id, uint32_t tag, uint32_t hop,
                 uint32_t batch_or_epoch, uint32_t w[4]) {
    uint32_t ctr[4] = {slot, id, (tag << 24) | hop, batch_or_epoch};
    uint32_t key[2] = {(uint32_t)(seed & 0xffffffffu), (uint32_t)(seed >> 32)};
    or_philox4x32_10(ctr, key, w);
}
static uint64_t r01(const uint32_t w[4]) { return ((uint64_t)w[1] << 32) | w[0]; }
static uint64_t r23(const uint32_t w[4]) { return ((uint64_t)w[3] << 32) | w[2]; }

enum { TAG_SAMPLE = 1, TAG_ROOT = 2, TAG_COMM = 3 };

/* ------------------------------------------------------------------ a0 */
/* Community offsets cbeg[c] = first node of community c (graph is community-
 * ordered; reading R18) and, for every node v, the sub-segment
 * [lo[v], hi[v]) of row v whose neighbours lie in v's community (the intra-
 * community edges of S4.2; reading R5: "intra" is relative to
 * the node being expanded).  Returns 0, 1 (invalid CSR: unsorted row,
 * duplicate, id out of range) or 2 (comm not non-decreasing / id >= C /
 * a community without nodes). */
int or_graph_prep(int64_t n, const int64_t *indptr, const int32_t *indices, const int32_t *comm,
                  int32_t num_comm, int32_t *cbeg, uint32_t *lo, uint32_t *hi) {
    for (int64_t v = 0; v < n; ++v) {
        if (comm[v] < 0 || comm[v] >= num_comm) return 2;
        if (v > 0 && comm[v] < comm[v - 1]) return 2;
    }
    for (int32_t c = 0; c <= num_comm; ++c) cbeg[c] = -1;
    for (int64_t v = n - 1; v >= 0; --v) cbeg[comm[v]] = (int32_t)v;
    cbeg[num_comm] = (int32_t)n;
    for (int32_t c = 0; c < num_comm; ++c)
        if (cbeg[c] < 0) return 2;
    for (int64_t v = 0; v < n; ++v) {
        int64_t rs = indptr[v], re = indptr[v + 1];
        if (re < rs) return 1;
        for (int64_t e = rs; e < re; ++e) {
            if (indices[e] < 0 || indices[e] >= n) return 1;
            if (e > rs && indices[e] <= indices[e - 1]) return 1;
        }
        int32_t c = comm[v];
        int64_t first_ge_beg = re, first_ge_end = re;
        for (int64_t e = re - 1; e >= rs; --e) {  /* plain linear scans of the sorted row */
            if (indices[e] >= cbeg[c]) first_ge_beg = e;
            if (indices[e] >= cbeg[c + 1]) first_ge_end = e;
        }
        lo[v] = (uint32_t)(first_ge_beg - rs);
        hi[v] = (uint32_t)(first_ge_end - rs);
    }
    return 0;
}

/* ------------------------------------------------------------------ a1 */
/* Knob-1 (Table 1; S4.1 P:653-680; reading R9/R10):
 *   mode 0 RAND-ROOTS:   sort train by (key(v), v), key(v) = r01(Philox(0, v, 2<<24, epoch))
 *   mode 1 NORAND-ROOTS: train as given (ascending), identical every epoch
 *   mode 2 COMM-RAND-MIX-k: the distinct communities of the training set
 *          (C_tr) are shuffled as blocks (sorted by (ckey(c), c),
 *          ckey(c) = r01(Philox(0, c, 3<<24, epoch))); consecutive runs of
 *          S = max(1, floor(k*C_tr + 0.5)) shuffled communities form a
 *          super-block; the train nodes are ordered by (super-block, key(v), v),
 *          i.e. the contents of each super-block are shuffled.
 *   mode 3 COMM-RAND-MIX-k with STATIC adjacent-community super-blocks (SURVEY.md 8(f)
 *          NEXT-2 (ii); reading R24): the C_tr train communities in ascending id order,
 *          j = 0..C_tr-1, form super-blocks b = j / S of S ADJACENT communities (fixed across
 *          epochs); each epoch the super-blocks are shuffled as units (sorted by (sbkey(b), b),
 *          sbkey(b) = r01(Philox(1, b, 3<<24, epoch))) and the train nodes are ordered by
 *          (rank of their super-block, key(v), v).
 * Batches are consecutive B-slices of the result (caller).  Returns 0 or -1. */
typedef struct { uint64_t k1, k2; int64_t v; } key3;

static int cmp_key3(const void *a, const void *b) {
    const key3 *x = (const key3 *)a, *y = (const key3 *)b;
    if (x->k1 != y->k1) return x->k1 < y->k1 ? -1 : 1;
    if (x->k2 != y->k2) return x->k2 < y->k2 ? -1 : 1;
    if (x->v != y->v) return x->v < y->v ? -1 : 1;
    return 0;
}

int or_order_roots(int64_t n_train, const int32_t *train, const int32_t *comm, int32_t num_comm,
                   int32_t mode, double mix, uint64_t seed, uint32_t epoch, int32_t *out) {
    if (n_train <= 0) return -1;
    if (mode == 1) {
        for (int64_t i = 0; i < n_train; ++i) out[i] = train[i];
        return 0;
    }
    key3 *rows = (key3 *)malloc(sizeof(key3) * (size_t)n_train);
    if (!rows) return -1;
    uint64_t *sb_of = NULL;
    if (mode == 2) {
        /* C_tr: communities that contain training nodes, ascending */
        char *has = (char *)calloc((size_t)num_comm, 1);
        int64_t ctr = 0;
        for (int64_t i = 0; i < n_train; ++i) has[comm[train[i]]] = 1;
        for (int32_t c = 0; c < num_comm; ++c) ctr += has[c];
        key3 *cs = (key3 *)malloc(sizeof(key3) * (size_t)(ctr ? ctr : 1));
        int64_t j = 0;
        for (int32_t c = 0; c < num_comm; ++c) {
            if (!has[c]) continue;
            uint32_t w[4];
            draw(seed, 0, (uint32_t)c, TAG_COMM, 0, epoch, w);
            cs[j].k1 = r01(w);
            cs[j].k2 = 0;
            cs[j].v = c;
            ++j;
        }
        qsort(cs, (size_t)ctr, sizeof(key3), cmp_key3);   /* shuffle communities as blocks */
        int64_t S = (int64_t)(mix * (double)ctr + 0.5);    /* floor(k*C_tr + 0.5) */
        if (S < 1) S = 1;
        sb_of = (uint64_t *)calloc((size_t)num_comm, sizeof(uint64_t));
        for (int64_t rank = 0; rank < ctr; ++rank) sb_of[cs[rank].v] = (uint64_t)(rank / S);
        free(cs);
        free(has);
    } else if (mode == 3) {
        char *has = (char *)calloc((size_t)num_comm, 1);
        int64_t ctr = 0;
        for (int64_t i = 0; i < n_train; ++i) has[comm[train[i]]] = 1;
        for (int32_t c = 0; c < num_comm; ++c) ctr += has[c];
        int64_t S = (int64_t)(mix * (double)ctr + 0.5);    /* floor(k*C_tr + 0.5) */
        if (S < 1) S = 1;
        const int64_t nsb = (ctr + S - 1) / S;
        key3 *bs = (key3 *)malloc(sizeof(key3) * (size_t)(nsb ? nsb : 1));
        for (int64_t b = 0; b < nsb; ++b) {                /* one key per super-block */
            uint32_t w[4];
            draw(seed, 1, (uint32_t)b, TAG_COMM, 0, epoch, w);
            bs[b].k1 = r01(w);
            bs[b].k2 = 0;
            bs[b].v = b;
        }
        qsort(bs, (size_t)nsb, sizeof(key3), cmp_key3);    /* shuffle the super-blocks */
        uint64_t *ord = (uint64_t *)calloc((size_t)(nsb ? nsb : 1), sizeof(uint64_t));
        for (int64_t r = 0; r < nsb; ++r) ord[bs[r].v] = (uint64_t)r;
        sb_of = (uint64_t *)calloc((size_t)num_comm, sizeof(uint64_t));
        int64_t j = 0;                                     /* train-community index, by id */
        for (int32_t c = 0; c < num_comm; ++c) {
            if (!has[c]) continue;
            sb_of[c] = ord[j / S];
            ++j;
        }
        free(ord);
        free(bs);
        free(has);
    }
    for (int64_t i = 0; i < n_train; ++i) {
        uint32_t w[4];
        int32_t v = train[i];
        draw(seed, 0, (uint32_t)v, TAG_ROOT, 0, epoch, w);
        rows[i].k1 = (mode == 2 || mode == 3) ? sb_of[comm[v]] : 0;
        rows[i].k2 = r01(w);
        rows[i].v = v;
    }
    qsort(rows, (size_t)n_train, sizeof(key3), cmp_key3);
    for (int64_t i = 0; i < n_train; ++i) out[i] = (int32_t)rows[i].v;
    free(rows);
    free(sb_of);
    return 0;
}

/* ------------------------------------------------------------------ a2 */
/* Knob-2 biased neighbour sampling of one hop (S4.2 P:683-691; S5 P:717:
 * per-edge unnormalised probability p for intra-community edges and 1-p for
 * inter-community edges, DGL NeighborSampler(prob=...): weighted sampling
 * WITHOUT replacement; reading R1 "law A").  For dst i (v = dst_nodes[i]):
 *   P16 = floor(p*65536 + 0.5), wi = P16, wo = 65536 - P16 (reading R13)
 *   ni = |intra segment|, no = deg - ni; zero-weight classes are ineligible
 *   (reading R3); m = ni_e + no_e
 *   if f >= m: take every eligible neighbour (reading R4), no RNG
 *   else, W_s = Philox(s, v, (1<<24)|hop, batch) for s < f:
 *     urn:   K = number of intra draws when drawing f times from an urn of
 *            ni_e balls of weight wi and no_e balls of weight wo without
 *            replacement: at draw s, intra iff unif(r01(W_s), T) < wi*ri,
 *            T = wi*ri + wo*ro (successive sampling: P(intra) = wi ri / T)
 *     Floyd: a uniform K-subset of the intra segment from r23(W_t), t < K,
 *            and a uniform (f-K)-subset of the inter positions from
 *            r23(W_{K+t}) (Floyd's algorithm, Bentley & Floyd CACM 1987)
 *   picks are emitted in ascending row position (reading R8).
 * law = 1 selects the SLOT law instead (the north_star's
 * literal "takes an intra-community neighbour with probability p_intra"; reading R23):
 *   take-all as above; else slot s < f is intra iff unif(r01(W_s), 65536) < P16,
 *   K_draw = number of intra slots, K = min(K_draw, ni_e), kb = min(f - K_draw, no_e)
 *   (no refill: a row may return fewer than f picks), then the same Floyd steps:
 *   intra subset from r23(W_t), t < K, inter subset from r23(W_{K+t}), t < kb.
 * Returns e_h (total picks) or -1 when cap is exceeded. */
static int cmp_u32(const void *a, const void *b) {
    uint32_t x = *(const uint32_t *)a, y = *(const uint32_t *)b;
    return (x > y) - (x < y);
}

static int contains(const uint32_t *set, int64_t n, uint32_t x) {
    for (int64_t i = 0; i < n; ++i)
        if (set[i] == x) return 1;
    return 0;
}

int64_t or_sample_hop(const int32_t *dst_nodes, int64_t n_dst, const int64_t *indptr,
                      const int32_t *indices, const uint32_t *lo, const uint32_t *hi, int32_t fanout,
                      double p, uint64_t seed, int32_t hop, uint32_t batch, int64_t *indptr_h,
                      int32_t *nbr, int64_t cap, int32_t law) {
    const uint64_t P16 = (uint64_t)(p * 65536.0 + 0.5);
    const uint64_t wi = P16, wo = 65536u - P16;
    const int64_t f = fanout;
    uint32_t *intra_set = (uint32_t *)malloc(sizeof(uint32_t) * (size_t)(f + 1));
    uint32_t *inter_set = (uint32_t *)malloc(sizeof(uint32_t) * (size_t)(f + 1));
    uint32_t *sel = (uint32_t *)malloc(sizeof(uint32_t) * (size_t)(f + 1));
    uint32_t(*W)[4] = malloc(sizeof(uint32_t[4]) * (size_t)(f + 1));
    int64_t out = 0;
    indptr_h[0] = 0;
    for (int64_t i = 0; i < n_dst; ++i) {
        const int32_t v = dst_nodes[i];
        const int64_t rs = indptr[v];
        const int64_t deg = indptr[v + 1] - rs;
        const int64_t ni = (int64_t)hi[v] - (int64_t)lo[v];
        const int64_t no = deg - ni;
        const int64_t ni_e = wi > 0 ? ni : 0;
        const int64_t no_e = wo > 0 ? no : 0;
        const int64_t m = ni_e + no_e;
        if (f >= m) {
            /* full eligible neighbourhood, ascending position */
            if (out + m > cap) { out = -1; break; }
            for (int64_t q = 0; q < deg; ++q) {
                int is_intra = (q >= (int64_t)lo[v] && q < (int64_t)hi[v]);
                if ((is_intra && ni_e > 0) || (!is_intra && no_e > 0)) nbr[out++] = indices[rs + q];
            }
        } else {
            for (int64_t s = 0; s < f; ++s) draw(seed, (uint32_t)s, (uint32_t)v, TAG_SAMPLE, (uint32_t)hop, batch, W[s]);
            int64_t K = 0, kb = 0;
            if (law == 1) {
                /* slot law: K_draw intra slots, then clip each class (no refill) */
                int64_t k_draw = 0;
                for (int64_t s = 0; s < f; ++s)
                    if (or_mulhi64(r01(W[s]), 65536u) < P16) k_draw++;
                K = k_draw < ni_e ? k_draw : ni_e;
                kb = (f - k_draw) < no_e ? (f - k_draw) : no_e;
            } else {
                /* urn: number of intra picks K */
                int64_t ri = ni_e, ro = no_e;
                for (int64_t s = 0; s < f; ++s) {
                    uint64_t T = wi * (uint64_t)ri + wo * (uint64_t)ro;
                    if (or_mulhi64(r01(W[s]), T) < wi * (uint64_t)ri) {
                        K++;
                        ri--;
                    } else {
                        ro--;
                    }
                }
                kb = f - K;
            }
            /* Floyd: uniform K-subset of [0, ni_e) */
            int64_t na = 0;
            for (int64_t t = 0; t < K; ++t) {
                uint64_t j = (uint64_t)(ni_e - K + t);
                uint32_t r = (uint32_t)or_mulhi64(r23(W[t]), j + 1);
                uint32_t pick = contains(intra_set, na, r) ? (uint32_t)j : r;
                intra_set[na] = pick;
                na++;
            }
            /* Floyd: uniform kb-subset of [0, no_e) */
            int64_t nb = 0;
            for (int64_t t = 0; t < kb; ++t) {
                uint64_t j = (uint64_t)(no_e - kb + t);
                uint32_t r = (uint32_t)or_mulhi64(r23(W[K + t]), j + 1);
                uint32_t pick = contains(inter_set, nb, r) ? (uint32_t)j : r;
                inter_set[nb] = pick;
                nb++;
            }
            /* map to row positions: intra q -> lo + q; inter q -> q (q < lo) or hi + (q - lo) */
            int64_t ns = 0;
            for (int64_t t = 0; t < na; ++t) sel[ns++] = lo[v] + intra_set[t];
            for (int64_t t = 0; t < nb; ++t) {
                uint32_t q = inter_set[t];
                sel[ns++] = (q < lo[v]) ? q : hi[v] + (q - lo[v]);
            }
            qsort(sel, (size_t)ns, sizeof(uint32_t), cmp_u32);
            if (out + ns > cap) { out = -1; break; }
            for (int64_t t = 0; t < ns; ++t) nbr[out++] = indices[rs + sel[t]];
        }
        indptr_h[i + 1] = out;
    }
    free(intra_set); free(inter_set); free(sel); free(W);
    return out;
}

/* ------------------------------------------------------------------ NEXT-2 (iii) */
/* Community reordering of a graph that is NOT community-ordered (
 * the paper assumes community-ordered inputs; reading R25): the new id order
 * sorts the nodes by (community, old id); perm[new] = old, inv[old] = new; row new i is old
 * row perm[i] with every neighbour u renamed inv[u] and the row sorted ascending; the community
 * array becomes comm[perm[i]] (non-decreasing).  indptr_out [n+1], indices_out [nnz],
 * comm_out [n], perm [n], inv [n] are caller-allocated.  Returns 0. */
static const int32_t *g_sort_comm;
static int cmp_by_comm(const void *a, const void *b) {
    int32_t x = *(const int32_t *)a, y = *(const int32_t *)b;
    if (g_sort_comm[x] != g_sort_comm[y]) return g_sort_comm[x] < g_sort_comm[y] ? -1 : 1;
    return (x > y) - (x < y);
}
static int cmp_i32(const void *a, const void *b) {
    int32_t x = *(const int32_t *)a, y = *(const int32_t *)b;
    return (x > y) - (x < y);
}

int or_community_order(int64_t n, const int64_t *indptr, const int32_t *indices,
                       const int32_t *comm, int32_t *perm, int32_t *inv, int64_t *indptr_out,
                       int32_t *indices_out, int32_t *comm_out) {
    for (int64_t i = 0; i < n; ++i) perm[i] = (int32_t)i;
    g_sort_comm = comm;
    qsort(perm, (size_t)n, sizeof(int32_t), cmp_by_comm);
    for (int64_t i = 0; i < n; ++i) inv[perm[i]] = (int32_t)i;
    indptr_out[0] = 0;
    for (int64_t i = 0; i < n; ++i) {
        const int32_t v = perm[i];
        const int64_t d = indptr[v + 1] - indptr[v];
        int32_t *row = indices_out + indptr_out[i];
        for (int64_t k = 0; k < d; ++k) row[k] = inv[indices[indptr[v] + k]];
        qsort(row, (size_t)d, sizeof(int32_t), cmp_i32);
        indptr_out[i + 1] = indptr_out[i] + d;
        comm_out[i] = comm[v];
    }
    return 0;
}

/* ------------------------------------------------------------------ a3 */
/* "Build sub-graph S_i out of root nodes and sampled neighbors" (Alg. 1,
 * P:541-542; DGL block semantics): the src list of the hop is the
 * dst list followed by every sampled neighbour not yet present, in order of
 * FIRST occurrence over (dst index, position) (reading R8; dst prefix =
 * reading R7).  local[e] = index of nbr[e] in the src list.
 * `map` is caller scratch of num_nodes int32, all -1 on entry; restored to -1.
 * Returns n_{h+1}, or -1 when nodes_cap is exceeded. */
int64_t or_relabel_hop(int32_t *nodes, int64_t n_dst, int64_t nodes_cap, const int32_t *nbr,
                       int64_t e_h, int32_t *local, int32_t *map) {
    int64_t n = n_dst;
    for (int64_t i = 0; i < n_dst; ++i) map[nodes[i]] = (int32_t)i;
    for (int64_t e = 0; e < e_h; ++e) {
        int32_t u = nbr[e];
        if (map[u] < 0) {
            if (n >= nodes_cap) { n = -1; break; }
            map[u] = (int32_t)n;
            nodes[n++] = u;
        }
        local[e] = map[u];
    }
    int64_t upto = n < 0 ? nodes_cap : n;
    for (int64_t i = 0; i < upto; ++i) map[nodes[i]] = -1;
    return n;
}

/* ------------------------------------------------------------------ a4 */
/* "the model takes in input features corresponding to the nodes within a
 * batch's subgraph": X_in[i, 0:F] = X[nodes[i], 0:F], byte copy. */
void or_gather(const int32_t *nodes, int64_t n, const float *X, int64_t ld, int32_t F, float *out,
               int64_t out_ld) {
    for (int64_t i = 0; i < n; ++i)
        memcpy(out + i * out_ld, X + (int64_t)nodes[i] * ld, sizeof(float) * (size_t)F);
}

/* ------------------------------------------------------------------ a5 */
/* GraphSAGE mean aggregator over the sampled in-neighbours of each dst row
 * (Hamilton et al. 2017 as used by the paper's 3-layer GraphSAGE, P:512,
 * P:770; neighbours only, reading R12):
 *   H[d, j] = (sum over e in row d, CSR order, of Xsrc[idx[e], j]) / deg_d,
 *   H[d, :] = 0 when deg_d = 0.
 * fp32 accumulation in CSR order and IEEE division; out64 (nullable) is the
 * fp64 shadow used for the tolerance check.  src rows: Xsrc[idx[e]] when
 * src_map is NULL, else X[src_map[idx[e]]] (same values). */
void or_sage_mean(const int64_t *indptr_h, const int32_t *idx, int64_t n_dst, const float *Xsrc,
                  int64_t src_ld, const int32_t *src_map, int32_t F, float *out, int64_t out_ld,
                  double *out64) {
    for (int64_t d = 0; d < n_dst; ++d) {
        int64_t deg = indptr_h[d + 1] - indptr_h[d];
        for (int32_t j = 0; j < F; ++j) {
            float acc = 0.0f;
            double acc64 = 0.0;
            for (int64_t e = indptr_h[d]; e < indptr_h[d + 1]; ++e) {
                int64_t row = src_map ? src_map[idx[e]] : idx[e];
                float x = Xsrc[row * src_ld + j];
                acc = acc + x;
                acc64 = acc64 + (double)x;
            }
            out[d * out_ld + j] = deg > 0 ? acc / (float)deg : 0.0f;
            if (out64) out64[d * F + j] = deg > 0 ? acc64 / (double)deg : 0.0;
        }
    }
}
