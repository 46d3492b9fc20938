// features.cu -- a4 (input-feature gather) and a5 (GraphSAGE mean
// aggregation of the input-side block; reading R12), separately and fused.
//
// These are the HBM-bound steps: the paper attributes the per-epoch time to the input-
// feature volume and the COMM-RAND speedup to L2 reuse.  Rows are
// moved with 128-bit coalesced loads/stores by groups of LPR lanes (one group per row, LPR
// = the smallest power of two covering F/4 float4s, capped at 32), with several independent
// rows/edges in flight per lane (Little's law: ~6 MB in flight chip-wide at ~8 TB/s).
// Aggregation keeps columns in lanes and walks the edges of a row in CSR order, so the fp32
// sum is formed in exactly the oracle's order (bit-exact; then IEEE division).
#include <cstdlib>

#include "common.cuh"

namespace cmb {
namespace {

__device__ __forceinline__ float4 ldg4(const float4* p) {
  float4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0, %1, %2, %3}, [%4];"
               : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w)
               : "l"(p));
  return r;
}

__device__ __forceinline__ void add4(float4& a, const float4& b) {
  a.x = __fadd_rn(a.x, b.x);
  a.y = __fadd_rn(a.y, b.y);
  a.z = __fadd_rn(a.z, b.z);
  a.w = __fadd_rn(a.w, b.w);
}

// ------------------------------------------------------------------ a4 gather
// U rows in flight per lane group; NV float4 per lane per row.
template <int LPR, int NV, int U>
__global__ void __launch_bounds__(256) k_gather_v4(const float4* __restrict__ x, int64_t ld4,
                                                   const int32_t* __restrict__ ids,
                                                   const int64_t* __restrict__ n_dev,
                                                   int64_t n_cap, int f4,
                                                   float4* __restrict__ out, int64_t out_ld4) {
  const int64_t n = min(*n_dev, n_cap);
  const int lane = threadIdx.x % LPR;
  const int64_t groups = (int64_t)gridDim.x * (blockDim.x / LPR);
  const int64_t g0 = blockIdx.x * (int64_t)(blockDim.x / LPR) + threadIdx.x / LPR;
  for (int64_t base = g0; base < n; base += groups * U) {
    for (int c0 = 0; c0 < f4; c0 += LPR * NV) {
      float4 v[U][NV];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int64_t row = base + u * groups;
        const float4* src = x + (row < n ? (int64_t)__ldg(ids + row) * ld4 : 0);
#pragma unroll
        for (int k = 0; k < NV; ++k) {
          const int c = c0 + lane + k * LPR;
          if (row < n && c < f4) v[u][k] = ldg4(src + c);
        }
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int64_t row = base + u * groups;
#pragma unroll
        for (int k = 0; k < NV; ++k) {
          const int c = c0 + lane + k * LPR;
          if (row < n && c < f4) out[row * out_ld4 + c] = v[u][k];
        }
      }
    }
  }
}

__global__ void k_gather_scalar(const float* __restrict__ x, int64_t ld,
                                const int32_t* __restrict__ ids, const int64_t* __restrict__ n_dev,
                                int64_t n_cap, int f, float* __restrict__ out, int64_t out_ld) {
  const int64_t n = min(*n_dev, n_cap);
  const int lane = threadIdx.x & 31;
  const int64_t w0 = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t row = w0; row < n; row += nw) {
    const float* src = x + (int64_t)ids[row] * ld;
    for (int c = lane; c < f; c += 32) out[row * out_ld + c] = src[c];
  }
}

// Pipelined row form (the kernel of the unfused cmb_sage_mean_aggregate): one group of
// LPR lanes per dst row, rows visited with
// a grid stride, and the index chain of the rows AHEAD is issued before the feature loads of
// the current row: stage A (row i+2G) loads indptr pair + self node id, stage B (row i+G)
// loads the row's src ids lane-parallel (lane k <-> edge k; global row ids come straight from
// `gid` -- the relabel step's pre-relabel neighbour ids -- or via map[idx]), stage C (row i)
// issues 1 + deg feature-row loads (self + edges, CH in flight) and folds the edges in CSR
// order.  The dependent chain indptr -> ids -> X therefore overlaps with other rows' loads.
// L2 cache-policy hints (createpolicy): feature rows are loaded evict_last (a row referenced
// by several dst rows of the batch should survive until its next use -- the paper's L2 reuse),
// outputs (X_in, H) are stored evict_first (written once, never re-read by this kernel).
#ifndef CMB_ROW_MINB
#define CMB_ROW_MINB 4
#endif
__device__ __forceinline__ uint64_t policy_evict_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
// the L2 policy of the fused gather's feature-row loads (layout experiments: CMB_ROW_POLICY
// 1 = evict_normal, 2 = evict_first; 0, the product, = evict_last)
#ifndef CMB_ROW_POLICY
#define CMB_ROW_POLICY 0
#endif
__device__ __forceinline__ uint64_t policy_rows() {
  uint64_t p;
#if CMB_ROW_POLICY == 1
  asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(p));
#elif CMB_ROW_POLICY == 2
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
#else
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
#endif
  return p;
}
__device__ __forceinline__ float4 ldg4_hint(const float4* p, uint64_t pol) {
  float4 r;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.f32 {%0, %1, %2, %3}, [%4], %5;"
               : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w)
               : "l"(p), "l"(pol));
  return r;
}
// predicated 16-byte load whose destination is zeroed inside the same asm block: a C
// `pred ? load : 0` leaves a select after the load that waits on its scoreboard, which holds the
// NEXT load's shuffle and address back until this one has returned (the row's loads then leave
// in two round trips instead of one)
__device__ __forceinline__ float4 ldg4_pred(const float4* p, bool pred, uint64_t pol) {
  float4 r;
  asm volatile(
      "{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %5, 0;\n\t"
      "mov.b32 %0, 0;\n\tmov.b32 %1, 0;\n\tmov.b32 %2, 0;\n\tmov.b32 %3, 0;\n\t"
      "@q ld.global.nc.L1::no_allocate.L2::cache_hint.v4.f32 {%0, %1, %2, %3}, [%4], %6;\n\t}"
      : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w)
      : "l"(p), "r"(static_cast<int>(pred)), "l"(pol));
  return r;
}
__device__ __forceinline__ void st4_hint(float4* p, const float4& v, uint64_t pol) {
  asm volatile("st.global.L2::cache_hint.v4.f32 [%0], {%1, %2, %3, %4}, %5;" ::"l"(p), "f"(v.x),
               "f"(v.y), "f"(v.z), "f"(v.w), "l"(pol)
               : "memory");
}

template <int LPR, int NV, int CH>
__global__ void __launch_bounds__(256, (LPR == 16 && NV == 2 && CH == 2) ? 4 : 1)
    k_gather_mean_pipe(
    const int32_t* __restrict__ indptr, const int32_t* __restrict__ idx,
    const int32_t* __restrict__ gid, const int64_t* __restrict__ n_dst_dev, int64_t n_dst_cap,
    const float4* __restrict__ src, int64_t src_ld4, const int32_t* __restrict__ map, int f4,
    float4* __restrict__ out, int64_t out_ld4, float4* __restrict__ x_in, int64_t x_in_ld4,
    const uint32_t* __restrict__ new_mask) {
  constexpr unsigned kFull = 0xffffffffu;
  constexpr int GPW = 32 / LPR;  // lane groups (dst rows) per warp
  const uint64_t pol_keep = policy_evict_last(), pol_stream = policy_evict_first();
  auto LD = [&](const float4* p) { return ldg4_hint(p, pol_keep); };
  auto ST = [&](float4* p, const float4& v) { st4_hint(p, v, pol_stream); };
  const int64_t n_dst = min(*n_dst_dev, n_dst_cap);
  const int lane = threadIdx.x % LPR;
  // Warp-uniform walk: the GPW groups of a warp take rows rb + q (q = group in the warp) and all
  // lanes run the same trip counts (row loop, max degree over the warp's rows), so every shuffle
  // uses the full mask.  (Per-group masks made the compiler wrap each shuffle in MATCH / REDUX /
  // VOTEU convergence checks on the XU pipe: ~4 per edge, the XU at 94 % busy.)
  const int q = (threadIdx.x & 31) / LPR;
  const int64_t WG = static_cast<int64_t>(gridDim.x) * (blockDim.x / 32) * GPW;
  const int64_t w0 = (static_cast<int64_t>(blockIdx.x) * (blockDim.x / 32) + threadIdx.x / 32) * GPW;

  struct A { int32_t e0, e1, self; };
  struct B { int32_t g, l, first; };
  auto loadA = [&](int64_t row) {
    A a{0, 0, 0};
    if (row < n_dst) {
      a.e0 = __ldg(indptr + row);
      a.e1 = __ldg(indptr + row + 1);
      if (x_in) a.self = __ldg(map + row);
    }
    return a;
  };
  auto loadB = [&](const A& a, int32_t base) {  // edge base + lane of the row described by a
    B b{0, 0, 0};
    const int32_t e = a.e0 + base + lane;
    if (e < a.e1) {
      b.l = __ldg(idx + e);
      b.g = gid ? __ldg(gid + e) : (map ? __ldg(map + b.l) : b.l);
      if (x_in) b.first = static_cast<int>((__ldg(new_mask + (e >> 5)) >> (e & 31)) & 1u);
    }
    return b;
  };

  int64_t rb = w0;
  A ac = loadA(rb + q);
  B bc = loadB(ac, 0);
  A an = loadA(rb + q + WG);
  for (; rb < n_dst; rb += WG) {
    const int64_t row = rb + q;       // rows >= n_dst (tail of the last sweep) have deg 0
    const bool live = row < n_dst;
    const A aa = loadA(row + 2 * WG);  // stage A, two rows ahead
    const B bn = loadB(an, 0);         // stage B, one row ahead
    const int32_t deg = ac.e1 - ac.e0;
    int32_t degmax = deg;
#pragma unroll
    for (int o = LPR; o < 32; o <<= 1) degmax = max(degmax, __shfl_xor_sync(kFull, degmax, o));
    for (int c0 = 0; c0 < f4; c0 += LPR * NV) {
      float4 acc[NV];
#pragma unroll
      for (int k = 0; k < NV; ++k) acc[k] = make_float4(0.f, 0.f, 0.f, 0.f);
      float4 self[NV];
      if (x_in && live) {
#pragma unroll
        for (int k = 0; k < NV; ++k) {
          const int c = c0 + lane + k * LPR;
          if (c < f4) self[k] = LD(src + (int64_t)ac.self * src_ld4 + c);
        }
      }
      for (int32_t base = 0; base < degmax; base += LPR) {
        const B bb = base == 0 ? bc : loadB(ac, base);  // rows with deg > LPR: rest on demand
        const int cnt = min(LPR, deg - base);           // <= 0 for a group already done
        const int cmax = min(LPR, degmax - base);
        for (int j0 = 0; j0 < cmax; j0 += CH) {
          float4 v[CH][NV];
#pragma unroll
          for (int u = 0; u < CH; ++u) {
            const int j = j0 + u;
            const int32_t r = __shfl_sync(kFull, bb.g, j & (LPR - 1), LPR);
#pragma unroll
            for (int k = 0; k < NV; ++k) {
              const int c = c0 + lane + k * LPR;
              if (j < cnt && c < f4) v[u][k] = LD(src + (int64_t)r * src_ld4 + c);
            }
          }
#pragma unroll
          for (int u = 0; u < CH; ++u) {
            const int j = j0 + u;
            const int fj = __shfl_sync(kFull, bb.first, j & (LPR - 1), LPR);
            const int32_t lj = __shfl_sync(kFull, bb.l, j & (LPR - 1), LPR);
            if (j < cnt) {
#pragma unroll
              for (int k = 0; k < NV; ++k) add4(acc[k], v[u][k]);
              if (fj) {  // first occurrence of a new src node: a4 for it, from this load
#pragma unroll
                for (int k = 0; k < NV; ++k) {
                  const int c = c0 + lane + k * LPR;
                  if (c < f4) ST(x_in + (int64_t)lj * x_in_ld4 + c, v[u][k]);
                }
              }
            }
          }
        }
      }
      const float fd = static_cast<float>(deg);
#pragma unroll
      for (int k = 0; k < NV; ++k) {
        const int c = c0 + lane + k * LPR;
        if (c < f4 && live) {
          float4 h = make_float4(0.f, 0.f, 0.f, 0.f);
          if (deg > 0) {
            h.x = __fdiv_rn(acc[k].x, fd);
            h.y = __fdiv_rn(acc[k].y, fd);
            h.z = __fdiv_rn(acc[k].z, fd);
            h.w = __fdiv_rn(acc[k].w, fd);
          }
          ST(out + row * out_ld4 + c, h);
          if (x_in) ST(x_in + row * x_in_ld4 + c, self[k]);
        }
      }
    }
    ac = an;
    bc = bn;
    an = aa;
  }
}

}  // namespace
}  // namespace cmb

#include "gather_row.cuh"
#include "cache.cuh"

namespace cmb {
namespace {

__global__ void k_sage_mean_scalar(const int32_t* __restrict__ indptr,
                                   const int32_t* __restrict__ idx,
                                   const int64_t* __restrict__ n_dst_dev, int64_t n_dst_cap,
                                   const float* __restrict__ src, int64_t src_ld,
                                   const int32_t* __restrict__ map, int f, float* __restrict__ out,
                                   int64_t out_ld, float* __restrict__ x_in, int64_t x_in_ld,
                                   const uint32_t* __restrict__ new_mask) {
  const int64_t n_dst = min(*n_dst_dev, n_dst_cap);
  const int lane = threadIdx.x & 31;
  const int64_t w0 = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t d = w0; d < n_dst; d += nw) {
    const int32_t e0 = indptr[d], e1 = indptr[d + 1];
    for (int c = lane; c < f; c += 32) {
      if (x_in) x_in[d * x_in_ld + c] = src[(int64_t)map[d] * src_ld + c];
      float acc = 0.f;
      for (int32_t e = e0; e < e1; ++e) {
        const int32_t l = idx[e];
        const float xv = src[(map ? (int64_t)map[l] : (int64_t)l) * src_ld + c];
        acc = __fadd_rn(acc, xv);
        if (x_in && ((new_mask[e >> 5] >> (e & 31)) & 1u)) x_in[(int64_t)l * x_in_ld + c] = xv;
      }
      out[d * out_ld + c] = e1 > e0 ? __fdiv_rn(acc, static_cast<float>(e1 - e0)) : 0.f;
    }
  }
}

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

int lanes_for(int f4) {
  int l = 1;
  while (l < f4 && l < 32) l <<= 1;
  return l < 4 ? 4 : l;  // groups of >= 4 lanes keep one row per 64-byte segment
}

template <int LPR, int NV>
void launch_gather(int grid, cudaStream_t s, const float* x, int64_t ld, const int32_t* ids,
                   const int64_t* n_dev, int64_t n_cap, int f4, float* out, int64_t out_ld) {
  k_gather_v4<LPR, NV, 4><<<grid, 256, 0, s>>>(reinterpret_cast<const float4*>(x), ld / 4, ids,
                                               n_dev, n_cap, f4, reinterpret_cast<float4*>(out),
                                               out_ld / 4);
}

cmb_status gather_dispatch(const float* x, int64_t ld, int f, const int32_t* ids,
                           const int64_t* n_dev, int64_t n_cap, float* out, int64_t out_ld,
                           int sms, cudaStream_t s) {
  if (n_cap <= 0) return CMB_OK;
  const int f4 = (f + 3) / 4;
  const bool vec = aligned16(x) && aligned16(out) && ld % 4 == 0 && out_ld % 4 == 0;
  if (!vec) {
    k_gather_scalar<<<sms * 8, 256, 0, s>>>(x, ld, ids, n_dev, n_cap, f, out, out_ld);
    CMB_CUDA(cudaGetLastError());
    return CMB_OK;
  }
  const int lpr = lanes_for(f4);
  const int rows_per_block = 256 / lpr;
  int64_t want = (n_cap + rows_per_block * 4 - 1) / (rows_per_block * 4);
  const int grid = static_cast<int>(want < sms * 16 ? (want > 0 ? want : 1) : sms * 16);
  switch (lpr) {
    case 4: launch_gather<4, 1>(grid, s, x, ld, ids, n_dev, n_cap, f4, out, out_ld); break;
    case 8: launch_gather<8, 1>(grid, s, x, ld, ids, n_dev, n_cap, f4, out, out_ld); break;
    case 16: launch_gather<16, 1>(grid, s, x, ld, ids, n_dev, n_cap, f4, out, out_ld); break;
    default:
      if (f4 <= 32) launch_gather<32, 1>(grid, s, x, ld, ids, n_dev, n_cap, f4, out, out_ld);
      else launch_gather<32, 2>(grid, s, x, ld, ids, n_dev, n_cap, f4, out, out_ld);
  }
  CMB_CUDA(cudaGetLastError());
  return CMB_OK;
}

template <int LPR, int NV, int CH>
void launch_mean(int sms, cudaStream_t s, const int32_t* indptr, const int32_t* idx,
                 const int32_t* gid, const int64_t* n_dev, int64_t n_cap, const float* src,
                 int64_t src_ld, const int32_t* map, int f4, float* out, int64_t out_ld,
                 float* x_in, int64_t x_in_ld, const uint32_t* mask) {
  const int64_t gpb = 256 / LPR;  // lane groups per 256-thread block
  // pipelined row form: a persistent-style grid (a few blocks per SM, grid-stride rows) so
  // every group walks many rows and its look-ahead pipeline stays full
  int64_t want = (n_cap + gpb - 1) / gpb;
  const int64_t cap_grid = static_cast<int64_t>(sms) * 8;
  const int grid = static_cast<int>(want < cap_grid ? (want > 0 ? want : 1) : cap_grid);
  k_gather_mean_pipe<LPR, NV, CH><<<grid, 256, 0, s>>>(
      indptr, idx, gid, n_dev, n_cap, reinterpret_cast<const float4*>(src), src_ld / 4, map, f4,
      reinterpret_cast<float4*>(out), out_ld / 4, reinterpret_cast<float4*>(x_in), x_in_ld / 4,
      mask);
}

// the default fused form: one warp per dst row (gather_row.cuh), all batches of the set in one
// launch.  DMAX = edge rows issued per round: the block's fanout (deg_hint = e_cap / n_cap)
// clamped to [4, 6] (8 spills at 64 registers: reddit's fanout-10 block runs best at 6, 178 vs
// 212 us)
template <class Rows>
cmb_status launch_rows(int sms, cudaStream_t s, const GatherSet& set, const Rows& rows, int f4,
                       int deg_hint) {
  const int dmax = deg_hint < 6 ? deg_hint : 6;
  int64_t n_cap = 0;
  for (int j = 0; j < set.nb; ++j) n_cap += set.n_dst_cap[j];
  const int64_t want = (n_cap + 7) / 8;  // 8 warps (rows) per 256-thread block
  // CMB_ROW_MINB resident 256-thread blocks per SM (4: 64 registers); a compile-time constant for
  // layout experiments (tools/), never a run-time switch
  const int64_t cap = static_cast<int64_t>(sms) * CMB_ROW_MINB;
  const int grid = static_cast<int>(want < cap ? (want > 0 ? want : 1) : cap);
#define CMB_ROWK(D_)                                                                          \
  if (f4 > 32) CMB_ROWK3(D_, true); else CMB_ROWK3(D_, false)
#define CMB_ROWK3(D_, W_)                                                                     \
  k_gather_mean_row<D_, CMB_ROW_MINB, W_, Rows><<<grid, 256, 0, s>>>(set, rows, f4)
  if (dmax <= 4) { CMB_ROWK(4); }
  else if (dmax <= 5) { CMB_ROWK(5); }
  else { CMB_ROWK(6); }
#undef CMB_ROWK
#undef CMB_ROWK3
  CMB_CUDA(cudaGetLastError());
  return CMB_OK;
}

// one batch's operands as entry j of a set
void set_batch(GatherSet& set, int j, const int32_t* indptr, const int32_t* idx,
               const int32_t* gid, const int64_t* n_dev, int64_t n_cap, const int32_t* map,
               float* out, int64_t out_ld, float* x_in, int64_t x_in_ld, const uint32_t* mask,
               const int32_t* order) {
  set.indptr[j] = indptr;
  set.idx[j] = idx;
  set.gid[j] = gid;
  set.n_dst_dev[j] = n_dev;
  set.n_dst_cap[j] = n_cap;
  set.map[j] = map;
  set.mask[j] = mask;
  set.order[j] = order;
  set.out[j] = reinterpret_cast<float4*>(out);
  set.out_ld4[j] = out_ld / 4;
  set.x_in[j] = reinterpret_cast<float4*>(x_in);
  set.x_in_ld4[j] = x_in_ld / 4;
}

template <class Rows>
cmb_status launch_row(int sms, cudaStream_t s, const int32_t* indptr, const int32_t* idx,
                      const int32_t* gid, const int64_t* n_dev, int64_t n_cap, const Rows& rows,
                      const int32_t* map, int f4, float* out, int64_t out_ld, float* x_in,
                      int64_t x_in_ld, const uint32_t* mask, int deg_hint,
                      const int32_t* order = nullptr) {
  GatherSet set{};
  set.nb = 1;
  set_batch(set, 0, indptr, idx, gid, n_dev, n_cap, map, out, out_ld, x_in, x_in_ld, mask, order);
  return launch_rows(sms, s, set, rows, f4, deg_hint);
}

cmb_status mean_dispatch(const int32_t* indptr, const int32_t* idx, const int32_t* gid,
                         const int64_t* n_dev, int64_t n_cap, const float* src, int64_t src_ld,
                         const int32_t* map, int f, float* out, int64_t out_ld, float* x_in,
                         int64_t x_in_ld, const uint32_t* mask, int sms, cudaStream_t s,
                         int32_t* status = nullptr, int deg_hint = 8,
                         const int32_t* order = nullptr) {
  if (n_cap <= 0) return CMB_OK;
  const int f4 = (f + 3) / 4;
  const bool vec = aligned16(src) && aligned16(out) && src_ld % 4 == 0 && out_ld % 4 == 0 &&
                   (!x_in || (aligned16(x_in) && x_in_ld % 4 == 0));
  if (vec && x_in && gid)
    return launch_row(sms, s, indptr, idx, gid, n_dev, n_cap,
                      DenseRows{reinterpret_cast<const float4*>(src),
                                static_cast<uint32_t>(src_ld / 4)},
                      map, f4, out,
                      out_ld, x_in, x_in_ld, mask, deg_hint, order);
  if (!vec) {
    k_sage_mean_scalar<<<sms * 8, 256, 0, s>>>(indptr, idx, n_dev, n_cap, src, src_ld, map, f,
                                               out, out_ld, x_in, x_in_ld, mask);
    CMB_CUDA(cudaGetLastError());
    return CMB_OK;
  }
  const int lpr = lanes_for(f4);
#define CMB_MEAN(L_, NV_, CH_)                                                                 \
  launch_mean<L_, NV_, CH_>(sms, s, indptr, idx, gid, n_dev, n_cap, src, src_ld, map, f4, out, \
                            out_ld, x_in, x_in_ld, mask)
  switch (lpr) {
    case 4: CMB_MEAN(4, 1, 4); break;
    case 8: CMB_MEAN(8, 1, 8); break;
    case 16: CMB_MEAN(16, 1, 8); break;
    default:
      if (f4 <= 32) {
        // measured best on B200 (products F = 100): 16 lanes x 2 float4 per row, two dst rows
        // per warp, 2 edges in flight per lane
        CMB_MEAN(16, 2, 2);
      } else if (f4 <= 64) CMB_MEAN(32, 2, 4);
      else if (f4 <= 128) CMB_MEAN(32, 4, 2);
      else CMB_MEAN(32, 5, 2);  // F = 602 -> 151 float4 = 32 x 5 (column tiles beyond)
  }
#undef CMB_MEAN
  CMB_CUDA(cudaGetLastError());
  return CMB_OK;
}

}  // namespace
}  // namespace cmb

using namespace cmb;

extern "C" {

cmb_status cmb_gather_features(const cmb_graph* g, const int32_t* node_ids, const int64_t* n_dev,
                               int64_t n_cap, float* out, int64_t out_ld, void* stream) {
  CMB_NVTX("cmb.a4.gather_features");
  CMB_ARG(g && node_ids && n_dev && out, "cmb_gather_features: null argument");
  CMB_ARG(g->d.x != nullptr, "cmb_gather_features: graph has no feature table");
  CMB_ARG(n_cap >= 0 && out_ld >= g->d.f, "cmb_gather_features: n_cap < 0 or out_ld < F");
  return gather_dispatch(g->d.x, g->d.ld, g->d.f, node_ids, n_dev, n_cap, out, out_ld,
                         g->num_sms, static_cast<cudaStream_t>(stream));
}

cmb_status cmb_gather_rows(const float* x, int64_t ld, int64_t row0, int32_t feat_dim,
                           const int32_t* ids, const int64_t* n_dev, int64_t n_cap, float* out,
                           int64_t out_ld, void* stream) {
  CMB_NVTX("cmb.a6.gather_rows");
  CMB_ARG(x && ids && n_dev && out, "cmb_gather_rows: null argument");
  CMB_ARG(feat_dim >= 1 && ld >= feat_dim && out_ld >= feat_dim && n_cap >= 0 && row0 >= 0,
          "cmb_gather_rows: bad feat_dim / ld / n_cap / row0");
  int dev = 0, sms = 148;
  CMB_CUDA(cudaGetDevice(&dev));
  CMB_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  // row id v lives at x[(v - row0) * ld]: shift the base (alignment is preserved)
  return gather_dispatch(x - row0 * ld, ld, feat_dim, ids, n_dev, n_cap, out, out_ld, sms,
                         static_cast<cudaStream_t>(stream));
}

cmb_status cmb_sage_mean_aggregate(const int32_t* indptr, const int32_t* indices,
                                   const int64_t* n_dst_dev, int64_t n_dst_cap, const float* src,
                                   int64_t src_ld, const int32_t* src_map, int32_t feat_dim,
                                   float* out, int64_t out_ld, void* stream) {
  CMB_NVTX("cmb.a5.sage_mean_aggregate");
  CMB_ARG(indptr && indices && n_dst_dev && src && out, "cmb_sage_mean_aggregate: null argument");
  CMB_ARG(feat_dim >= 1 && src_ld >= feat_dim && out_ld >= feat_dim && n_dst_cap >= 0,
          "cmb_sage_mean_aggregate: bad feat_dim / ld / n_dst_cap");
  int dev = 0, sms = 148;
  CMB_CUDA(cudaGetDevice(&dev));
  CMB_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  return mean_dispatch(indptr, indices, nullptr, n_dst_dev, n_dst_cap, src, src_ld, src_map,
                       feat_dim, out, out_ld, nullptr, 0, nullptr, sms,
                       static_cast<cudaStream_t>(stream));
}

cmb_status cmb_gather_aggregate_sharded(const cmb_graph* g, const cmb_blocks* b, int32_t n_hops,
                                        int64_t n_last_dst_cap, int64_t nodes_cap,
                                        const float* const* shards, int32_t world,
                                        int64_t rows_per_shard, int64_t shard_ld, int32_t feat_dim,
                                        float* x_in, int64_t x_in_ld, float* h_out, int64_t h_ld,
                                        void* stream) {
  CMB_NVTX("cmb.a4a5.gather_aggregate_sharded");
  CMB_ARG(g && b && shards && x_in && h_out, "cmb_gather_aggregate_sharded: null argument");
  CMB_ARG(n_hops >= 1 && n_hops <= CMB_MAX_HOPS, "cmb_gather_aggregate_sharded: bad n_hops");
  CMB_ARG(world >= 1 && world <= kMaxShards, "cmb_gather_aggregate_sharded: world %d outside [1, %d]",
          world, kMaxShards);
  CMB_ARG(rows_per_shard >= 1 && rows_per_shard * world >= g->d.n &&
              rows_per_shard <= INT32_MAX,
          "cmb_gather_aggregate_sharded: rows_per_shard * world must cover the %lld nodes",
          static_cast<long long>(g->d.n));
  CMB_ARG(feat_dim >= 1 && shard_ld >= feat_dim && x_in_ld >= feat_dim && h_ld >= feat_dim,
          "cmb_gather_aggregate_sharded: bad feat_dim / ld");
  CMB_ARG(shard_ld % 4 == 0 && x_in_ld % 4 == 0 && h_ld % 4 == 0 && aligned16(x_in) &&
              aligned16(h_out),
          "cmb_gather_aggregate_sharded: rows must be 16-B aligned");
  CMB_ARG(b->new_src_mask && b->last_src_ids,
          "cmb_gather_aggregate_sharded: blocks->new_src_mask and last_src_ids are required");
  CMB_ARG(n_last_dst_cap <= nodes_cap, "cmb_gather_aggregate_sharded: n_last_dst_cap > nodes_cap");
  ShardedRows rows{};
  for (int r = 0; r < world; ++r) {
    CMB_ARG(shards[r] && aligned16(shards[r]), "cmb_gather_aggregate_sharded: shard %d", r);
    rows.base[r] = reinterpret_cast<const float4*>(shards[r]);
  }
  rows.ld4 = static_cast<uint32_t>(shard_ld / 4);
  rows.rows_per_shard = static_cast<uint32_t>(rows_per_shard);
  rows.inv = ((1ull << 32) + rows_per_shard - 1) / rows_per_shard;
  const int L = n_hops;
  return launch_row(g->num_sms, static_cast<cudaStream_t>(stream), b->indptr[L - 1],
                    b->indices[L - 1], b->last_src_ids, b->sizes + (L - 1), n_last_dst_cap, rows,
                    b->nodes, (feat_dim + 3) / 4, h_out, h_ld, x_in, x_in_ld, b->new_src_mask,
                    n_last_dst_cap > 0 ? static_cast<int>(b->indices_cap[L - 1] / n_last_dst_cap)
                                       : 8,
                    b->dst_order);
}

cmb_status cmb_cache_gather_aggregate(const cmb_graph* g, const cmb_blocks* b, int32_t n_hops,
                                      int64_t n_last_dst_cap, int64_t nodes_cap,
                                      const cmb_feature_cache* c, int32_t feat_dim,
                                      uint32_t batch_tag, float* x_in, int64_t x_in_ld,
                                      float* h_out, int64_t h_ld, int64_t* stats, void* stream) {
  CMB_NVTX("cmb.a4a5.cache_gather_aggregate");
  CMB_ARG(g && b && c && x_in && h_out, "cmb_cache_gather_aggregate: null argument");
  CMB_ARG(n_hops >= 1 && n_hops <= CMB_MAX_HOPS, "cmb_cache_gather_aggregate: bad n_hops");
  CMB_ARG(c->workspace && c->host_x && c->cache_rows, "cmb_cache_gather_aggregate: bad cache");
  CMB_ARG(c->num_nodes == g->d.n, "cmb_cache_gather_aggregate: cache built for another graph");
  CMB_ARG(batch_tag != 0xFFFFFFFFu, "cmb_cache_gather_aggregate: batch_tag 0xFFFFFFFF reserved");
  const int L = n_hops;
  CMB_ARG(nodes_cap <= c->max_rows && b->indices_cap[L - 1] <= c->max_edges &&
              c->capacity >= c->max_rows,
          "cmb_cache_gather_aggregate: batch larger than the cache was sized for");
  CMB_ARG(feat_dim >= 1 && c->host_ld >= feat_dim && c->cache_ld >= feat_dim &&
              c->cache_ld % 4 == 0 && x_in_ld % 4 == 0 && h_ld % 4 == 0 &&
              aligned16(c->cache_rows) && aligned16(x_in) && aligned16(h_out),
          "cmb_cache_gather_aggregate: bad feat_dim / ld / alignment");
  CMB_ARG(b->new_src_mask != nullptr, "cmb_cache_gather_aggregate: new_src_mask required");
  size_t need = 0;
  CacheWs w = carve_cache_ws(c->workspace, c->num_nodes, c->capacity, c->max_rows, c->max_edges,
                             &need);
  CMB_ARG(c->workspace_bytes >= need, "cmb_cache_gather_aggregate: workspace < %zu bytes", need);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  cmb_status st = cache_prepare(w, c->capacity, b->nodes, b->sizes + L, nodes_cap,
                                b->indices[L - 1], b->sizes + L + 1 + (L - 1),
                                b->indices_cap[L - 1], c->host_x, c->host_ld, feat_dim,
                                c->cache_rows, c->cache_ld, batch_tag, stats, g->num_sms, s);
  if (st != CMB_OK) return st;
  // every row of the batch is resident now: the fused kernel reads cache slots (gid = slot of
  // each edge's src node, map = slot of each node of the batch)
  return launch_row(g->num_sms, s, b->indptr[L - 1], b->indices[L - 1], w.gslot,
                    b->sizes + (L - 1), n_last_dst_cap,
                    DenseRows{reinterpret_cast<const float4*>(c->cache_rows),
                              static_cast<uint32_t>(c->cache_ld / 4)},
                    w.slot_i, (feat_dim + 3) / 4, h_out, h_ld, x_in, x_in_ld, b->new_src_mask,
                    n_last_dst_cap > 0 ? static_cast<int>(b->indices_cap[L - 1] / n_last_dst_cap)
                                       : 8,
                    b->dst_order);
}

cmb_status cmb_gather_aggregate_multi(const cmb_graph* g, const cmb_blocks* const* blocks,
                                      const cmb_batch_features* feats, int32_t n_batches,
                                      int32_t n_hops, void* stream) {
  CMB_NVTX("cmb.a4a5.gather_aggregate_multi");
  CMB_ARG(g && blocks && feats, "cmb_gather_aggregate_multi: null argument");
  CMB_ARG(n_batches >= 1 && n_batches <= kMaxGatherBatches,
          "cmb_gather_aggregate_multi: n_batches %d outside [1, %d]", n_batches,
          kMaxGatherBatches);
  CMB_ARG(n_hops >= 1 && n_hops <= CMB_MAX_HOPS, "cmb_gather_aggregate_multi: bad n_hops");
  CMB_ARG(g->d.x != nullptr && g->d.ld % 4 == 0 && aligned16(g->d.x),
          "cmb_gather_aggregate_multi: needs a 16-B aligned feature table (ld %% 4 == 0)");
  const int L = n_hops;
  GatherSet set{};
  set.nb = n_batches;
  int deg_hint = 8;
  for (int j = 0; j < n_batches; ++j) {
    const cmb_blocks* b = blocks[j];
    const cmb_batch_features& f = feats[j];
    CMB_ARG(b && f.x_in && f.h_out && b->new_src_mask && b->last_src_ids,
            "cmb_gather_aggregate_multi: batch %d: null blocks / outputs / mask / src ids", j);
    CMB_ARG(f.x_in_ld >= g->d.f && f.h_ld >= g->d.f && f.x_in_ld % 4 == 0 && f.h_ld % 4 == 0 &&
                aligned16(f.x_in) && aligned16(f.h_out) && f.n_last_dst_cap <= f.nodes_cap,
            "cmb_gather_aggregate_multi: batch %d: outputs must be 16-B aligned rows, ld >= F", j);
    set_batch(set, j, b->indptr[L - 1], b->indices[L - 1], b->last_src_ids, b->sizes + (L - 1),
              f.n_last_dst_cap, b->nodes, f.h_out, f.h_ld, f.x_in, f.x_in_ld, b->new_src_mask,
              b->dst_order);
    if (f.n_last_dst_cap > 0) deg_hint = static_cast<int>(b->indices_cap[L - 1] / f.n_last_dst_cap);
  }
  return launch_rows(g->num_sms, static_cast<cudaStream_t>(stream), set,
                     DenseRows{reinterpret_cast<const float4*>(g->d.x),
                               static_cast<uint32_t>(g->d.ld / 4)},
                     (g->d.f + 3) / 4, deg_hint);
}

cmb_status cmb_gather_aggregate(const cmb_graph* g, const cmb_blocks* b, int32_t n_hops,
                                int64_t n_last_dst_cap, int64_t nodes_cap, float* x_in,
                                int64_t x_in_ld, float* h_out, int64_t h_ld, void* stream) {
  CMB_NVTX("cmb.a4a5.gather_aggregate");
  CMB_ARG(g && b && x_in && h_out, "cmb_gather_aggregate: null argument");
  CMB_ARG(n_hops >= 1 && n_hops <= CMB_MAX_HOPS, "cmb_gather_aggregate: bad n_hops");
  CMB_ARG(g->d.x != nullptr, "cmb_gather_aggregate: graph has no feature table");
  CMB_ARG(b->new_src_mask != nullptr, "cmb_gather_aggregate: blocks->new_src_mask is required");
  CMB_ARG(x_in_ld >= g->d.f && h_ld >= g->d.f, "cmb_gather_aggregate: ld < F");
  CMB_ARG(n_last_dst_cap <= nodes_cap, "cmb_gather_aggregate: n_last_dst_cap > nodes_cap");
  const int L = n_hops;
  const int f4 = (g->d.f + 3) / 4;
  return mean_dispatch(b->indptr[L - 1], b->indices[L - 1], b->last_src_ids, b->sizes + (L - 1),
                       n_last_dst_cap, g->d.x, g->d.ld, b->nodes, g->d.f, h_out, h_ld, x_in,
                       x_in_ld, b->new_src_mask, g->num_sms, static_cast<cudaStream_t>(stream),
                       g->status,
                       n_last_dst_cap > 0 ? static_cast<int>(b->indices_cap[L - 1] / n_last_dst_cap)
                                          : 8,
                       b->dst_order);
}

}  // extern "C"
