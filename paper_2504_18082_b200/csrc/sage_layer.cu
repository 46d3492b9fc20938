// sage_layer.cu -- NEXT-4: the input-side GraphSAGE-mean layer fused with a4 + a5
// on the 5th-generation tensor cores (reading R26; Eq. (1) in the GraphSAGE form
// of its footnote; hidden dim 256):
//
//     Y[d, :] = sigma( X[nodes[d]] W_self + mean_{e in row d} X[gid[e]] W_neigh + b ),  d < n_{L-1}
//
// One persistent CTA per SM (512 threads), tiles of M = 128 dst rows.  Per tile:
//  1. gather: every warp builds 8 rows of the A operand [X_dst | H] (K = 2 halves of kh*64
//     columns) straight from the feature table -- all edge-id shuffles of a group of RIF rows
//     first, then the self row and the deg neighbour rows of each row issued back to back
//     (RIF x (1 + DMAX) 16-byte loads in flight per lane), the next tile's indptr / dst ids /
//     edge ids prefetched behind them; H = fp32 sum in CSR order times RN(1/deg); converted to
//     bf16 and stored into shared memory in the UMMA canonical K-major SWIZZLE_128B layout
//     (8-row x 128-byte atoms, 16-byte chunk j of row r at chunk j ^ (r & 7): a warp writing
//     one row touches 8 distinct chunk slots, no bank conflicts);
//  2. one thread issues 2*ceil(F/16) tcgen05.mma.cta_group::1.kind::f16 (M=128, N=Fo, K=16,
//     bf16 x bf16 -> fp32 in TMEM) against the packed weight image, resident in shared memory
//     for the whole launch, and commits them to an mbarrier;
//  3. epilogue: warp w reads TMEM lanes 32*(w%4).. (its lane quarter) with tcgen05.ld 32x32b.x16,
//     adds the bias, applies ReLU and stores fp32 or bf16 rows (L2 evict_first).
// Measured (profiles/r01_ncu_full_k_sage_layer.txt): the tensor pipe is ~7% busy; the kernel is
// bound by the latency of the random row loads, like a4+a5.  A warp-specialised form (4 epilogue
// warps, 8 gather warps, double-buffered TMEM) was slower (160 vs 116 us on products): fewer
// gather warps means fewer loads in flight, and the register file, not the barriers, is the limit.
// H and X_in never reach HBM: the layer reads the feature rows once per reference and writes only
// Y, which is what makes it HBM-bound rather than tensor-bound (K = 2F <= 256: ~2*K flops per
// 4*(1+deg)*F bytes read).
#include <cuda_bf16.h>

#include <cstdlib>

#include "common.cuh"

namespace cmb {
namespace sl {

constexpr int kThreads = 512;
constexpr int kWarps = kThreads / 32;
constexpr int kM = 128;              // UMMA M (rows per tile)
constexpr int kRowsPerWarp = kM / kWarps;  // 8
constexpr int kAtomBytes = 128;      // one row of a SWIZZLE_128B atom (64 bf16)

__host__ __device__ inline uint32_t w_img_bytes(int kh, int fo, int halves = 2) {
  return static_cast<uint32_t>(halves * kh) * static_cast<uint32_t>(fo) * kAtomBytes;
}
__host__ __device__ inline uint32_t a_bytes(int kh) {
  return static_cast<uint32_t>(2 * kh) * kM * kAtomBytes;
}
inline size_t smem_bytes(int kh, int fo) {
  return 1024 /*alignment slack*/ + w_img_bytes(kh, fo) + a_bytes(kh) + 64 /*barrier, tmem slot*/ +
         static_cast<size_t>(fo) * 4 /*bias*/;
}
// sw128_off (common.cuh): byte offset of an element in the K-major SWIZZLE_128B operand image

// ----------------------------------------------------------------- PTX wrappers (tcgen05, mbarrier)
__device__ __forceinline__ uint32_t saddr(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
// UMMA shared-memory descriptor: start >> 4 [0,14), LBO >> 4 [16,30) (unused for swizzled K-major),
// SBO >> 4 [32,46) = 1024 B between 8-row groups, version 1 [46,48), layout SWIZZLE_128B = 2 [61,64)
__device__ __forceinline__ uint64_t sw128_desc(uint32_t addr) {
  return static_cast<uint64_t>((addr & 0x3FFFFu) >> 4) | (static_cast<uint64_t>(1024 >> 4) << 32) |
         (1ull << 46) | (2ull << 61);
}
// instruction descriptor of kind::f16: D fp32 [4,6)=1, A bf16 [7,10)=1, B bf16 [10,13)=1, both
// K-major, N >> 3 at [17,23), M >> 4 at [24,29)
__host__ __device__ inline uint32_t idesc_bf16(int m, int n) {
  return (1u << 4) | (1u << 7) | (1u << 10) | (static_cast<uint32_t>(n >> 3) << 17) |
         (static_cast<uint32_t>(m >> 4) << 24);
}
__device__ __forceinline__ void mma_bf16(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t idesc,
                                         uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem_d),
      "l"(a), "l"(b), "r"(idesc), "r"(accumulate));
}
__device__ __forceinline__ void mma_commit(uint32_t bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   bar)
               : "memory");
}
__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  uint32_t done = 0;
  while (!done) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}\n"
        : "=r"(done)
        : "r"(bar), "r"(parity)
        : "memory");
  }
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes)
               : "memory");
}
// global -> shared bulk copy (TMA engine, no registers) completing on an mbarrier; the image is
// moved in 32-KB pieces, the barrier expects the whole byte count
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes,
                                         uint32_t bar) {
  mbar_expect_tx(bar, bytes);
  for (uint32_t off = 0; off < bytes; off += 32768u) {
    const uint32_t n = bytes - off < 32768u ? bytes - off : 32768u;
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
            "r"(dst + off),
        "l"(static_cast<const char*>(src) + off), "r"(n), "r"(bar)
        : "memory");
  }
}
// shared -> global bulk copy (TMA engine) in 32-KB pieces, one bulk group; the source may be
// overwritten after bulk_s2g_wait_read()
__device__ __forceinline__ void bulk_s2g(void* dst, uint32_t src, uint32_t bytes) {
  for (uint32_t off = 0; off < bytes; off += 32768u) {
    const uint32_t n = bytes - off < 32768u ? bytes - off : 32768u;
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(
                     static_cast<char*>(dst) + off),
                 "r"(src + off), "r"(n)
                 : "memory");
  }
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}
__device__ __forceinline__ void bulk_s2g_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
}
__device__ __forceinline__ void bulk_s2g_wait_all() {
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}
__device__ __forceinline__ void fence_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, uint32_t (&v)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, "
      "%12, %13, %14, %15}, [%16];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
        "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]),
        "=r"(v[14]), "=r"(v[15])
      : "r"(taddr));
}
__device__ __forceinline__ void tmem_ld_wait() {
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

// predicated 16-byte load whose destination is zeroed inside the same asm block (no select after
// the load, so no later register move waits on this load's scoreboard and the loads of several
// rows stay in flight together), with an L2 cache policy (createpolicy): feature rows are loaded
// evict_last so a row several dst rows of the batch reference survives until its next use (the
// paper's L2 reuse)
__device__ __forceinline__ float4 ldg4_or_zero(const float4* p, bool pred, uint64_t pol) {
  float4 r;
  asm volatile(
      "{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %5, 0;\n\t"
      "mov.b32 %0, 0;\n\tmov.b32 %1, 0;\n\tmov.b32 %2, 0;\n\tmov.b32 %3, 0;\n\t"
      "@q ld.global.nc.L1::no_allocate.L2::cache_hint.v4.f32 {%0, %1, %2, %3}, [%4], %6;\n\t}"
      : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w)
      : "l"(p), "r"(static_cast<int>(pred)), "l"(pol));
  return r;
}
__device__ __forceinline__ uint64_t l2_evict_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t l2_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ void st16_hint(uint4* p, uint4 v, uint64_t pol) {
  asm volatile("st.global.L2::cache_hint.v4.b32 [%0], {%1, %2, %3, %4}, %5;" ::"l"(p), "r"(v.x),
               "r"(v.y), "r"(v.z), "r"(v.w), "l"(pol)
               : "memory");
}
__device__ __forceinline__ uint2 pack_bf16x4(float4 v) {
  const __nv_bfloat162 lo = __floats2bfloat162_rn(v.x, v.y);
  const __nv_bfloat162 hi = __floats2bfloat162_rn(v.z, v.w);
  return make_uint2(*reinterpret_cast<const uint32_t*>(&lo), *reinterpret_cast<const uint32_t*>(&hi));
}

// ----------------------------------------------------------------- weight packing
// w_img[element (n, k)] = bf16(W_h[c][n]) for k = half h, column c < F; 0 for the padding columns.
// w_neigh == NULL: one half only (the GCN form, W = w_self)
// trans != 0: the halves are the transposes of row-major [fo x F] matrices (w[n * F + c]), the
// image of the input-gradient GEMM dZ W^T of a hidden layer (K = its out_dim, N = its in_dim)
__global__ void k_pack_weights(const float* __restrict__ w_self, const float* __restrict__ w_neigh,
                               int F, int fo, int kh, __nv_bfloat16* __restrict__ img,
                               int trans = 0) {
  const int kcols = kh * 64;
  const int64_t total = static_cast<int64_t>((w_neigh ? 2 : 1) * kcols) * fo;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int n = static_cast<int>(i % fo);
    const int k = static_cast<int>(i / fo);
    const int h = k / kcols, c = k % kcols;
    float v = 0.f;
    if (c < F)
      v = (h == 0 ? w_self : w_neigh)[trans ? static_cast<int64_t>(n) * F + c
                                            : static_cast<int64_t>(c) * fo + n];
    img[sw128_off(n, h, c, kh, fo) >> 1] = __float2bfloat16_rn(v);
  }
}

// ----------------------------------------------------------------- the fused layer kernel
// Builds the A operand [X_dst | H] of 128-row tiles (bf16, K-major SWIZZLE_128B, one 16-KB atom
// per 64 columns of each half) straight from the feature table.  Each of the 16 warps owns 8 rows
// of a tile: all edge-id shuffles of a group of RIF rows first, then the self row and the deg edge
// rows of each row issued back to back as predicated loads; H = fp32 sum in CSR order times
// RN(1/deg).  The next tile's indptr / dst ids / edge ids are loaded behind the current loads.
template <int DMAX, int RIF>
struct ATileGather {
  const int32_t* indptr;
  const int32_t* gid;
  const int32_t* map;
  const float4* x;
  int64_t ld4;
  int F, kh;
  int64_t n_dst, ntiles;
  int warp, lane;
  uint64_t pol;
  int32_t ip, self, g[kRowsPerWarp];  // current tile: lane-held indptr (9) and dst ids (8)
  int nr;
  int32_t nip, nself, ng[kRowsPerWarp];  // next tile
  int nnr;
  float4 ps[RIF], pv[RIF][DMAX];  // the first row group of the current tile, loaded ahead
  int pdeg[RIF];

  __device__ __forceinline__ void load_head(int64_t tile, int32_t& ip_, int32_t& self_, int& nr_) {
    const int64_t rbase = tile * kM + warp * kRowsPerWarp;
    const int64_t rem = n_dst - rbase;
    nr_ = (tile >= ntiles || rem <= 0) ? 0 : (rem >= kRowsPerWarp ? kRowsPerWarp : static_cast<int>(rem));
    ip_ = (lane <= nr_ && nr_ > 0) ? __ldg(indptr + rbase + lane) : 0;
    self_ = lane < nr_ ? __ldg(map + rbase + lane) : 0;
  }
  // lane j of g_[k] = global id of edge j of row k
  __device__ __forceinline__ void load_edges(int32_t ip_, int nr_, int32_t (&g_)[kRowsPerWarp]) {
#pragma unroll
    for (int k = 0; k < kRowsPerWarp; ++k) {
      const int32_t lo = __shfl_sync(0xffffffffu, ip_, k);
      const int32_t hi = __shfl_sync(0xffffffffu, ip_, k + 1);
      g_[k] = (k < nr_ && lane < hi - lo) ? __ldg(gid + lo + lane) : 0;
    }
  }
  __device__ __forceinline__ void start(int64_t tile) {
    load_head(tile, ip, self, nr);
    load_edges(ip, nr, g);
  }
  __device__ __forceinline__ void advance() {
    ip = nip;
    self = nself;
    nr = nnr;
#pragma unroll
    for (int k = 0; k < kRowsPerWarp; ++k) g[k] = ng[k];
  }
  // gathers the current tile into sA (rows past n_dst: skipped, or zero-filled if zero_dead) and
  // starts loading the indices of tile `next`.  gcn: one half only, the row of the self-loop,
  // row-normalised adjacency (X_dst + sum of the edge rows) / (deg + 1) (reading R28)
  // issues the loads of the current tile's first row group into ps / pv (build(pre = true)
  // consumes them): lets a kernel keep loads in flight across its MMA wait and epilogue
  __device__ __forceinline__ void issue_group0() {
    constexpr unsigned kFull = 0xffffffffu;
    const bool col_data = lane < ((F + 3) >> 2);
#pragma unroll
    for (int u = 0; u < RIF; ++u) {
      const int32_t lo = __shfl_sync(kFull, ip, u);
      const int32_t hi = __shfl_sync(kFull, ip, u + 1);
      pdeg[u] = u < nr ? hi - lo : 0;
      const int32_t sv = __shfl_sync(kFull, self, u);
      int32_t gj[DMAX];
#pragma unroll
      for (int j = 0; j < DMAX; ++j) gj[j] = __shfl_sync(kFull, g[u], j);
      const bool live = u < nr && col_data;
      ps[u] = ldg4_or_zero(x + static_cast<int64_t>(sv) * ld4 + lane, live, pol);
#pragma unroll
      for (int j = 0; j < DMAX; ++j)
        pv[u][j] = ldg4_or_zero(x + static_cast<int64_t>(gj[j]) * ld4 + lane, live && j < pdeg[u], pol);
    }
  }
  __device__ __forceinline__ void build(int64_t next, uint8_t* sA, bool zero_dead, bool gcn = false,
                                        bool pre = false) {
    constexpr unsigned kFull = 0xffffffffu;
    const int f4 = (F + 3) >> 2;
    const int c0 = lane * 4;             // this lane's 4 columns of each half
    const bool col_live = c0 < kh * 64;  // inside the operand's K extent
    const bool col_data = lane < f4;     // holds (some) feature columns
    const float4 zero = make_float4(0.f, 0.f, 0.f, 0.f);
    load_head(next, nip, nself, nnr);
#pragma unroll
    for (int k0 = 0; k0 < kRowsPerWarp; k0 += RIF) {
      float4 s[RIF], v[RIF][DMAX];
      int deg[RIF];
      if (k0 == 0 && pre) {
#pragma unroll
        for (int u = 0; u < RIF; ++u) {
          s[u] = ps[u];
          deg[u] = pdeg[u];
#pragma unroll
          for (int j = 0; j < DMAX; ++j) v[u][j] = pv[u][j];
        }
      } else {
        int32_t sv[RIF], gj[RIF][DMAX];
#pragma unroll
        for (int u = 0; u < RIF; ++u) {  // all shuffles first, then every load back to back
          const int k = k0 + u;
          const int32_t lo = __shfl_sync(kFull, ip, k);
          const int32_t hi = __shfl_sync(kFull, ip, k + 1);
          deg[u] = k < nr ? hi - lo : 0;
          sv[u] = __shfl_sync(kFull, self, k);
#pragma unroll
          for (int j = 0; j < DMAX; ++j) gj[u][j] = __shfl_sync(kFull, g[k], j);
        }
#pragma unroll
        for (int u = 0; u < RIF; ++u) {
          const bool live = k0 + u < nr && col_data;
          s[u] = ldg4_or_zero(x + static_cast<int64_t>(sv[u]) * ld4 + lane, live, pol);
#pragma unroll
          for (int j = 0; j < DMAX; ++j)
            v[u][j] = ldg4_or_zero(x + static_cast<int64_t>(gj[u][j]) * ld4 + lane,
                                   live && j < deg[u], pol);
        }
      }
      if (k0 == 0) load_edges(nip, nnr, ng);  // next tile's edge ids, behind this group's loads
#pragma unroll
      for (int u = 0; u < RIF; ++u) {
        const int k = k0 + u;
        float4 acc = zero;
#pragma unroll
        for (int j = 0; j < DMAX; ++j) {
          acc.x = __fadd_rn(acc.x, v[u][j].x);
          acc.y = __fadd_rn(acc.y, v[u][j].y);
          acc.z = __fadd_rn(acc.z, v[u][j].z);
          acc.w = __fadd_rn(acc.w, v[u][j].w);
        }
        for (int j0 = DMAX; j0 < deg[u]; j0 += DMAX) {  // rows longer than DMAX, CSR order
#pragma unroll
          for (int j = 0; j < DMAX; ++j) {
            const int32_t e = __shfl_sync(kFull, g[k], (j0 + j) & 31);
            const float4 w = ldg4_or_zero(x + static_cast<int64_t>(e) * ld4 + lane,
                                          col_data && j0 + j < deg[u], pol);
            acc.x = __fadd_rn(acc.x, w.x);
            acc.y = __fadd_rn(acc.y, w.y);
            acc.z = __fadd_rn(acc.z, w.z);
            acc.w = __fadd_rn(acc.w, w.w);
          }
        }
        if (col_live && (k < nr || zero_dead)) {
          float4 hm = zero;
          if (deg[u] > 0) {
            const float y = __frcp_rn(static_cast<float>(deg[u]));
            hm = make_float4(acc.x * y, acc.y * y, acc.z * y, acc.w * y);
          }
          float4 sf = s[u];
          if (gcn) {
            const float y = __frcp_rn(static_cast<float>(deg[u] + 1));
            sf = make_float4(__fadd_rn(sf.x, acc.x) * y, __fadd_rn(sf.y, acc.y) * y,
                             __fadd_rn(sf.z, acc.z) * y, __fadd_rn(sf.w, acc.w) * y);
          }
          if (c0 + 4 > F) {  // columns at or beyond F are operand padding: exact zeros
            if (c0 + 0 >= F) sf.x = hm.x = 0.f;
            if (c0 + 1 >= F) sf.y = hm.y = 0.f;
            if (c0 + 2 >= F) sf.z = hm.z = 0.f;
            if (c0 + 3 >= F) sf.w = hm.w = 0.f;
          }
          const int r = warp * kRowsPerWarp + k;
          *reinterpret_cast<uint2*>(sA + sw128_off(r, 0, c0, kh, kM)) = pack_bf16x4(sf);
          if (!gcn) *reinterpret_cast<uint2*>(sA + sw128_off(r, 1, c0, kh, kM)) = pack_bf16x4(hm);
        }
      }
    }
  }
};

template <int DMAX, int RIF>
__global__ void __launch_bounds__(kThreads, 1)
    k_sage_layer(const int32_t* __restrict__ indptr, const int32_t* __restrict__ gid,
                 const int64_t* __restrict__ n_dst_dev, int64_t n_dst_cap,
                 const float4* __restrict__ x, int64_t ld4, const int32_t* __restrict__ map,
                 int F, int kh, const uint4* __restrict__ w_img, const float* __restrict__ bias,
                 int fo, int tmem_cols, int relu, int out_bf16, void* __restrict__ out,
                 int64_t out_ld, int halves, uint8_t* __restrict__ a_save = nullptr) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024 - (saddr(smem_raw) & 1023)) & 1023);
  const uint32_t wbytes = w_img_bytes(kh, fo, halves);
  uint8_t* sW = smem;
  uint8_t* sA = sW + wbytes;
  uint64_t* bar = reinterpret_cast<uint64_t*>(sA + a_bytes(kh));
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bar + 1);
  float* sbias = reinterpret_cast<float*>(bar + 8);

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t n_dst = min(*n_dst_dev, n_dst_cap);
  const int64_t ntiles = (n_dst + kM - 1) / kM;
  const uint64_t pol_keep = l2_evict_last(), pol_stream = l2_evict_first();

  // weight image -> shared memory once per launch by a bulk copy (waited for by the MMA thread
  // before the first MMA, so it lands while the first tile is gathered); bias by plain loads
  const uint32_t wbar = saddr(bar + 2);
  for (int i = tid; i < fo; i += kThreads) sbias[i] = bias ? __ldg(bias + i) : 0.f;
  if (tid == 0) {
    mbar_init(saddr(bar), 1);
    mbar_init(wbar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    bulk_g2s(saddr(sW), w_img, wbytes, wbar);
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     saddr(tmem_slot)),
                 "r"(tmem_cols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  fence_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  const int steps = (F + 15) >> 4;        // K = 16 MMA steps per half
  const uint32_t idesc = idesc_bf16(kM, fo);
  const uint32_t sA_addr = saddr(sA), sW_addr = saddr(sW);
  uint32_t phase = 0;

  ATileGather<DMAX, RIF> ga;
  ga.indptr = indptr;
  ga.gid = gid;
  ga.map = map;
  ga.x = x;
  ga.ld4 = ld4;
  ga.F = F;
  ga.kh = kh;
  ga.n_dst = n_dst;
  ga.ntiles = ntiles;
  ga.warp = warp;
  ga.lane = lane;
  ga.pol = pol_keep;
  ga.start(blockIdx.x);
  ga.issue_group0();

  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    // ---------------------------------------------------------------- 1. gather -> A (bf16)
    ga.build(tile + gridDim.x, sA, a_save != nullptr, halves == 1, /*pre=*/true);
    fence_async_smem();  // generic-proxy smem writes -> visible to the tensor core (async proxy)
    __syncthreads();
    // the built A tile (the exact operand image, dead rows zero) -> HBM for the backward, by the
    // TMA engine while the MMAs and the epilogue run (R27: the backward reads it back instead of
    // re-gathering the feature rows)
    if (a_save && tid == 32)
      bulk_s2g(a_save + tile * static_cast<int64_t>(a_bytes(kh)), sA_addr, a_bytes(kh));

    // ---------------------------------------------------------------- 2. MMA (one thread)
    if (tid == 0) {
      if (tile == blockIdx.x) mbar_wait(wbar, 0);  // the weight image has landed
      tc_fence_after();
      uint32_t acc_flag = 0;
      for (int h = 0; h < halves; ++h) {
        for (int st = 0; st < steps; ++st) {
          const uint32_t atom = static_cast<uint32_t>(h * kh + (st >> 2));
          const uint32_t koff = static_cast<uint32_t>(st & 3) * 32u;
          const uint64_t da = sw128_desc(sA_addr + atom * (kM * kAtomBytes) + koff);
          const uint64_t db = sw128_desc(sW_addr + atom * (fo * kAtomBytes) + koff);
          mma_bf16(tmem, da, db, idesc, acc_flag);
          acc_flag = 1;
        }
      }
      mma_commit(saddr(bar));
    }
    ga.advance();       // the next tile's first row group loads while the MMAs run and the
    ga.issue_group0();  // accumulator is drained (A is rewritten only after the next sync)
    mbar_wait(saddr(bar), phase);
    phase ^= 1;
    tc_fence_after();

    // ---------------------------------------------------------------- 3. epilogue
    {
      const int q = warp & 3;
      const int64_t row = tile * kM + q * 32 + lane;
      const bool live = row < n_dst;
      for (int ch = warp >> 2; ch < fo / 16; ch += kWarps / 4) {
        uint32_t v[16];
        tmem_ld16(tmem + (static_cast<uint32_t>(q * 32) << 16) + static_cast<uint32_t>(ch * 16), v);
        tmem_ld_wait();
        float y[16];
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          y[i] = __fadd_rn(__uint_as_float(v[i]), sbias[ch * 16 + i]);
          if (relu) y[i] = fmaxf(y[i], 0.f);
        }
        if (live) {
          if (out_bf16) {
            uint4* o = reinterpret_cast<uint4*>(static_cast<__nv_bfloat16*>(out) + row * out_ld +
                                                ch * 16);
            uint32_t p[8];
#pragma unroll
            for (int i = 0; i < 8; ++i) {
              const __nv_bfloat162 b2 = __floats2bfloat162_rn(y[2 * i], y[2 * i + 1]);
              p[i] = *reinterpret_cast<const uint32_t*>(&b2);
            }
            st16_hint(o, make_uint4(p[0], p[1], p[2], p[3]), pol_stream);
            st16_hint(o + 1, make_uint4(p[4], p[5], p[6], p[7]), pol_stream);
          } else {
            uint4* o = reinterpret_cast<uint4*>(static_cast<float*>(out) + row * out_ld + ch * 16);
#pragma unroll
            for (int i = 0; i < 4; ++i)
              st16_hint(o + i, make_uint4(__float_as_uint(y[4 * i]), __float_as_uint(y[4 * i + 1]),
                                          __float_as_uint(y[4 * i + 2]), __float_as_uint(y[4 * i + 3])),
                        pol_stream);
          }
        }
      }
    }
    if (a_save && tid == 32) bulk_s2g_wait_read();  // the saved tile has left shared memory
    tc_fence_before();
    __syncthreads();  // TMEM drained and A free before the next tile overwrites them
  }
  if (a_save && tid == 32) bulk_s2g_wait_all();

  if (tid == 0 && ntiles <= blockIdx.x) mbar_wait(wbar, 0);  // no tile: the copy must still land
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                 "r"(tmem_cols)
                 : "memory");
  }
}

// ----------------------------------------------------------------- NEXT-4 backward (reading R27)
// Weight gradients of the layer: dW = [X_dst | H]^T dZ, db = sum_rows dZ, dZ = dY * 1[Y > 0].
// The reduction runs over the dst rows, so the tensor-core problem is transposed with respect to
// the forward: M = the 2*kh*64 feature rows of A, N = Fo, K = the batch rows.  Each CTA rebuilds
// the A tile of its 128-row tiles exactly as the forward does (same shared-memory image) and
// reads it as an MN-major operand (features contiguous; LBO = 16 KB between 64-feature atoms,
// SBO = 1 KB between 8-row groups); the dZ tile is staged in the same 128-byte-swizzled
// MN-major layout.  The per-CTA accumulators ([M_all x Fo] fp32, kh x Fo TMEM columns) are
// written as partials and summed over CTAs in fp64 by a second kernel (deterministic).
constexpr int kMaxBwdCtas = 160;

__host__ __device__ inline uint32_t b_bytes(int fo) {  // dZ tile: one 16-KB atom per 64 columns
  return static_cast<uint32_t>((fo + 63) / 64) * kM * kAtomBytes;
}
inline size_t bwd_smem_bytes(int kh, int fo) {
  return 1024 + a_bytes(kh) + b_bytes(fo) + 64 + static_cast<size_t>(fo) * 4;
}
// MN-major SWIZZLE_128B descriptor: LBO = byte stride between 64-element MN atoms, SBO = byte
// stride between 8-row K groups
__device__ __forceinline__ uint64_t sw128_mn_desc(uint32_t addr, uint32_t lbo) {
  return static_cast<uint64_t>((addr & 0x3FFFFu) >> 4) | (static_cast<uint64_t>(lbo >> 4) << 16) |
         (static_cast<uint64_t>(1024 >> 4) << 32) | (1ull << 46) | (2ull << 61);
}

// 8 columns (8c .. 8c+7) of row `row` of dY as bf16: a bf16 dY is loaded as is; an fp32 one (the
// input gradient of the next layer, R32, accumulated in fp32) is rounded to bf16 here, so the
// chain needs no cast pass
__device__ __forceinline__ uint4 load_dy8(const void* dy, int dy_f32, int64_t row, int64_t ld,
                                          int c) {
  if (!dy_f32)
    return __ldg(reinterpret_cast<const uint4*>(static_cast<const __nv_bfloat16*>(dy) + row * ld) + c);
  const float4* p = reinterpret_cast<const float4*>(static_cast<const float*>(dy) + row * ld) + 2 * c;
  const float4 a = __ldg(p), b = __ldg(p + 1);
  const uint2 lo = pack_bf16x4(a), hi = pack_bf16x4(b);
  return make_uint4(lo.x, lo.y, hi.x, hi.y);
}

template <int DMAX, int RIF>
__global__ void __launch_bounds__(kThreads, 1)
    k_sage_layer_bwd(const int32_t* __restrict__ indptr, const int32_t* __restrict__ gid,
                     const int64_t* __restrict__ n_dst_dev, int64_t n_dst_cap,
                     const float4* __restrict__ x, int64_t ld4, const int32_t* __restrict__ map,
                     int F, int kh, const void* __restrict__ dy, int64_t dy_ld, int dy_f32,
                     const __nv_bfloat16* __restrict__ y, int64_t y_ld, int fo, int tmem_alloc,
                     float* __restrict__ part, float* __restrict__ part_db,
                     const uint8_t* __restrict__ a_saved = nullptr, int gcn = 0) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024 - (saddr(smem_raw) & 1023)) & 1023);
  uint8_t* sA = smem;
  uint8_t* sB = sA + a_bytes(kh);
  uint64_t* bar = reinterpret_cast<uint64_t*>(sB + b_bytes(fo));
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bar + 1);
  float* sdb = reinterpret_cast<float*>(bar + 8);

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t n_dst = min(*n_dst_dev, n_dst_cap);
  const int64_t ntiles = (n_dst + kM - 1) / kM;
  const uint64_t pol_keep = l2_evict_last();
  const int m_all = 2 * kh * 64;
  // M = 128 blocks of feature rows (= kh); the GCN form (reading R35) has one operand half, the
  // aggregate A'X_in in atoms [0, kh): its blocks cover them (an odd kh's last block also spans
  // the first atom of the unused half, whose output rows are never reduced)
  const int nmb = gcn ? (kh + 1) / 2 : m_all / kM;

  for (int i = tid; i < fo; i += kThreads) sdb[i] = 0.f;
  if (tid == 0) {
    mbar_init(saddr(bar), 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     saddr(tmem_slot)),
                 "r"(tmem_alloc)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  ATileGather<DMAX, RIF> ga;
  ga.indptr = indptr;
  ga.gid = gid;
  ga.map = map;
  ga.x = x;
  ga.ld4 = ld4;
  ga.F = F;
  ga.kh = kh;
  ga.n_dst = n_dst;
  ga.ntiles = ntiles;
  ga.warp = warp;
  ga.lane = lane;
  ga.pol = pol_keep;
  if (!a_saved) ga.start(blockIdx.x);
  const uint32_t lbar = saddr(bar + 2);  // a_saved: the tile image's bulk load
  uint32_t lphase = 0;
  if (a_saved && tid == 0) {
    mbar_init(lbar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  // dZ staging: thread owns the 8-column chunk c = tid % (fo/8) of rows tid / (fo/8) + i*step
  const int cpr = fo / 8;           // chunks per row (a power of two dividing kThreads)
  const int c = tid % cpr;
  const int rstep = kThreads / cpr;
  float dbacc[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) dbacc[i] = 0.f;

  const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | (1u << 15) | (1u << 16) |
                         (static_cast<uint32_t>(fo >> 3) << 17) | (static_cast<uint32_t>(kM >> 4) << 24);
  const uint32_t sA_addr = saddr(sA), sB_addr = saddr(sB);
  uint32_t phase = 0;
  int it = 0;
  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++it) {
    if (a_saved) {  // the forward's A tile: one bulk load, overlapped with the dZ staging below
      if (tid == 0)
        bulk_g2s(sA_addr, a_saved + tile * static_cast<int64_t>(a_bytes(kh)), a_bytes(kh), lbar);
    } else {
      ga.build(tile + gridDim.x, sA, true, gcn != 0);
    }
    // dZ staging, four of the thread's rows at a time: all their loads first (one round trip),
    // then mask, column sums and the swizzled shared-memory stores
    for (int r0 = tid / cpr; r0 < kM; r0 += 4 * rstep) {
      uint4 v[4], m[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int r = r0 + u * rstep;
        const int64_t row = tile * kM + r;
        const bool live = r < kM && row < n_dst;
        v[u] = live ? load_dy8(dy, dy_f32, row, dy_ld, c) : make_uint4(0u, 0u, 0u, 0u);
        m[u] = (live && y) ? __ldg(reinterpret_cast<const uint4*>(y + row * y_ld) + c)
                           : make_uint4(0u, 0u, 0u, 0u);
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int r = r0 + u * rstep;
        if (r >= kM) break;
        if (y) {
          const uint32_t* mw = reinterpret_cast<const uint32_t*>(&m[u]);
          uint32_t* vw = reinterpret_cast<uint32_t*>(&v[u]);
#pragma unroll
          for (int i = 0; i < 4; ++i) {  // keep dY where Y > 0 (bf16 sign bit clear, nonzero)
            const uint32_t lo = mw[i] & 0xFFFFu, hi = mw[i] >> 16;
            const uint32_t keep = ((lo != 0u && !(lo & 0x8000u)) ? 0xFFFFu : 0u) |
                                  ((hi != 0u && !(hi & 0x8000u)) ? 0xFFFF0000u : 0u);
            vw[i] &= keep;
          }
        }
        const __nv_bfloat162* p2 = reinterpret_cast<const __nv_bfloat162*>(&v[u]);
#pragma unroll
        for (int i = 0; i < 4; ++i) {  // dead rows are zero: adding them changes nothing
          const float2 f2 = __bfloat1622float2(p2[i]);
          dbacc[2 * i] += f2.x;
          dbacc[2 * i + 1] += f2.y;
        }
        const uint32_t off = static_cast<uint32_t>(c >> 3) * (kM * kAtomBytes) + (r >> 3) * 1024 +
                             (r & 7) * 128 + (((c & 7) ^ (r & 7)) << 4);
        *reinterpret_cast<uint4*>(sB + off) = v[u];
      }
    }
    if (a_saved) {
      mbar_wait(lbar, lphase);
      lphase ^= 1;
    }
    fence_async_smem();
    __syncthreads();
    if (tid == 0) {
      tc_fence_after();
      for (int mb = 0; mb < nmb; ++mb) {
        for (int ks = 0; ks < kM / 16; ++ks) {
          const uint64_t da = sw128_mn_desc(sA_addr + (2 * mb) * (kM * kAtomBytes) + ks * 2048,
                                            kM * kAtomBytes);
          const uint64_t db = sw128_mn_desc(sB_addr + ks * 2048, kM * kAtomBytes);
          mma_bf16(tmem + static_cast<uint32_t>(mb * fo), da, db, idesc,
                   (it > 0 || ks > 0) ? 1u : 0u);
        }
      }
      mma_commit(saddr(bar));
    }
    mbar_wait(saddr(bar), phase);  // A and B may be overwritten once the MMAs have read them
    phase ^= 1;
    tc_fence_after();
    __syncthreads();
    if (!a_saved) ga.advance();
  }

  // ---------------------------------------------------------------- partials
  {
    const int q = warp & 3;
    for (int mb = 0; mb < nmb; ++mb) {
      const int m = mb * kM + q * 32 + lane;
      float* dst = part + (static_cast<int64_t>(blockIdx.x) * m_all + m) * fo;
      for (int ch = warp >> 2; ch < fo / 16; ch += kWarps / 4) {
        uint32_t v[16];
        tmem_ld16(tmem + (static_cast<uint32_t>(q * 32) << 16) +
                      static_cast<uint32_t>(mb * fo + ch * 16), v);
        tmem_ld_wait();
#pragma unroll
        for (int i = 0; i < 4; ++i)
          reinterpret_cast<float4*>(dst + ch * 16)[i] =
              it > 0 ? make_float4(__uint_as_float(v[4 * i]), __uint_as_float(v[4 * i + 1]),
                                   __uint_as_float(v[4 * i + 2]), __uint_as_float(v[4 * i + 3]))
                     : make_float4(0.f, 0.f, 0.f, 0.f);
      }
    }
  }
  {  // db: the per-thread column sums added in a fixed order (deterministic; dZ's tile is free)
    float* buf = reinterpret_cast<float*>(sB);
#pragma unroll
    for (int i = 0; i < 8; ++i) buf[(tid / cpr) * fo + c * 8 + i] = dbacc[i];
    __syncthreads();
    for (int i = tid; i < fo; i += kThreads) {
      float t = 0.f;
      for (int j = 0; j < rstep; ++j) t += buf[j * fo + i];
      sdb[i] = t;
    }
  }
  tc_fence_before();
  __syncthreads();
  for (int i = tid; i < fo; i += kThreads) part_db[static_cast<int64_t>(blockIdx.x) * fo + i] = sdb[i];
  if (warp == 0) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                 "r"(tmem_alloc)
                 : "memory");
  }
}

// dw[h][f][o] = sum over CTAs of part[cta][h*kh*64 + f][o], db[o] = sum of part_db[cta][o], in
// fp64 and a fixed order (deterministic): a 256-thread block owns 32 consecutive outputs; its 8
// warps sum the partials p = w, w + 8, ... (coalesced 128-B rows), then warp 0 adds the 8 sums.
__global__ void __launch_bounds__(256) k_sage_bwd_reduce(const float* __restrict__ part,
                                                         const float* __restrict__ part_db,
                                                         int nparts, int F, int kh, int fo,
                                                         float* __restrict__ dw,
                                                         float* __restrict__ db, int halves = 2) {
  __shared__ double red[8][32];
  const int m_all = 2 * kh * 64;
  const int64_t nw = static_cast<int64_t>(halves) * F * fo;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int64_t i = static_cast<int64_t>(blockIdx.x) * 32 + lane;
  double s = 0.0;
  if (i < nw) {
    const int o = static_cast<int>(i % fo);
    const int f = static_cast<int>((i / fo) % F);
    const int h = static_cast<int>(i / (static_cast<int64_t>(F) * fo));
    const int64_t off = static_cast<int64_t>(h * kh * 64 + f) * fo + o;
    for (int p = w; p < nparts; p += 8) s += __ldg(part + static_cast<int64_t>(p) * m_all * fo + off);
  } else if (i < nw + fo) {
    const int o = static_cast<int>(i - nw);
    for (int p = w; p < nparts; p += 8) s += __ldg(part_db + static_cast<int64_t>(p) * fo + o);
  }
  red[w][lane] = s;
  __syncthreads();
  if (w == 0 && i < nw + fo) {
    double t = 0.0;
#pragma unroll
    for (int g = 0; g < 8; ++g) t += red[g][lane];
    if (i < nw) dw[i] = static_cast<float>(t);
    else db[i - nw] = static_cast<float>(t);
  }
}

// ----------------------------------------------------------------- NEXT-4 hidden layers
// Layers after the first (reading R29): the input is the previous layer's output Yp (bf16,
// [n_{h+1} x Fin], row = local src id of hop h; the dst rows d < n_h are its prefix), so
//     Y[d] = sigma( Yp[d] W_self + mean_{e in row d of hop h} Yp[idx[e]] W_neigh + b ).
// K = 2 Fin = 512 at the paper's hidden dim (256) does not fit in shared memory next to
// its weights, so every 128-row tile runs two K phases (self, then neighbour mean), each staging
// its A half (128 x Fin bf16, 64 KB) and its W half (Fin x Fo bf16, 128 KB; from L2) before
// Fin/16 tcgen05 MMAs accumulate into the same TMEM columns.  One lane owns 8 columns (one
// 16-byte load per row); the neighbour mean is summed in fp32 in CSR order.
__device__ __forceinline__ uint4 ldg16_or_zero(const uint4* p, bool pred) {
  uint4 r;
  asm volatile(
      "{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %5, 0;\n\t"
      "mov.b32 %0, 0;\n\tmov.b32 %1, 0;\n\tmov.b32 %2, 0;\n\tmov.b32 %3, 0;\n\t"
      "@q ld.global.nc.L1::no_allocate.v4.u32 {%0, %1, %2, %3}, [%4];\n\t}"
      : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
      : "l"(p), "r"(static_cast<int>(pred)));
  return r;
}
__device__ __forceinline__ void add_bf16x8(float (&acc)[8], const uint4& v) {
  const __nv_bfloat162* p = reinterpret_cast<const __nv_bfloat162*>(&v);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const float2 f = __bfloat1622float2(p[i]);
    acc[2 * i] = __fadd_rn(acc[2 * i], f.x);
    acc[2 * i + 1] = __fadd_rn(acc[2 * i + 1], f.y);
  }
}
inline size_t hid_smem_bytes(int kin, int fo) {
  return 1024 + static_cast<size_t>(kin) * kM * kAtomBytes + static_cast<size_t>(kin) * fo * kAtomBytes +
         64 + static_cast<size_t>(fo) * 4;
}

// One K half of a hidden layer's A tile in shared memory (K-major SWIZZLE_128B, one 16-KB atom per
// 64 columns): ph 0 = the bf16 neighbour means of the warp's rows rbase .. rbase + nr - 1 (edge
// ids of all its rows first, then two rows at a time, each row's edges in chunks of DMAX loads
// issued together, summed in fp32 in CSR order, times RN(1/deg)); ph 1 = those rows of Yp.  The
// warp's rows nr .. rpw - 1 (past n_dst) are written as zeros, so a tile never holds stale rows.
template <int DMAX>
__device__ __forceinline__ void hid_build_half(int ph, const int32_t* __restrict__ idx,
                                               const uint4* __restrict__ yp, int64_t yp_ld8,
                                               int32_t ip, int64_t rbase, int nr, int rpw,
                                               int warp, int lane, bool col, uint8_t* sA) {
  constexpr unsigned kFull = 0xffffffffu;
  if (ph == 0) {
    // edge ids of all 8 rows first (one round trip), then two rows at a time, each row's
    // edges in chunks of DMAX loads issued together, summed in fp32 in CSR order
    int32_t g[kRowsPerWarp];
#pragma unroll
    for (int k = 0; k < kRowsPerWarp; ++k) {
      const int32_t lo = __shfl_sync(kFull, ip, k);
      const int32_t hi = __shfl_sync(kFull, ip, k + 1);
      g[k] = (k < nr && lane < hi - lo) ? __ldg(idx + lo + lane) : 0;
    }
#pragma unroll
    for (int k0 = 0; k0 < kRowsPerWarp; k0 += 2) {
      int deg[2];
      float acc[2][8];
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        const int k = k0 + u;
        const int32_t lo = __shfl_sync(kFull, ip, k);
        const int32_t hi = __shfl_sync(kFull, ip, k + 1);
        deg[u] = k < nr ? hi - lo : 0;
#pragma unroll
        for (int i = 0; i < 8; ++i) acc[u][i] = 0.f;
      }
      const int dm = deg[0] > deg[1] ? deg[0] : deg[1];
      for (int j0 = 0; j0 < dm; j0 += DMAX) {
        uint4 v[2][DMAX];
#pragma unroll
        for (int u = 0; u < 2; ++u) {
#pragma unroll
          for (int j = 0; j < DMAX; ++j) {
            const int32_t e = __shfl_sync(kFull, g[k0 + u], (j0 + j) & 31);
            v[u][j] = ldg16_or_zero(yp + static_cast<int64_t>(e) * yp_ld8 + lane,
                                    col && j0 + j < deg[u]);
          }
        }
#pragma unroll
        for (int u = 0; u < 2; ++u)
#pragma unroll
          for (int j = 0; j < DMAX; ++j)
            if (j0 + j < deg[u]) add_bf16x8(acc[u], v[u][j]);
      }
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        const int k = k0 + u;
        uint4 m = make_uint4(0u, 0u, 0u, 0u);
        if (deg[u] > 0) {
          const float y = __frcp_rn(static_cast<float>(deg[u]));
          uint32_t pk[4];
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            const __nv_bfloat162 b2 =
                __floats2bfloat162_rn(acc[u][2 * i] * y, acc[u][2 * i + 1] * y);
            pk[i] = *reinterpret_cast<const uint32_t*>(&b2);
          }
          m = make_uint4(pk[0], pk[1], pk[2], pk[3]);
        }
        if (col && k < rpw) {
          const int r = warp * rpw + k, atom = lane >> 3, j = lane & 7;
          *reinterpret_cast<uint4*>(sA + atom * (kM * kAtomBytes) + (r >> 3) * 1024 +
                                    (r & 7) * 128 + ((j ^ (r & 7)) << 4)) = m;
        }
      }
    }
  } else {
    uint4 sv[kRowsPerWarp];
#pragma unroll
    for (int k = 0; k < kRowsPerWarp; ++k)
      sv[k] = ldg16_or_zero(yp + (rbase + k) * yp_ld8 + lane, k < nr && col);
#pragma unroll
    for (int k = 0; k < kRowsPerWarp; ++k) {
      if (col && k < rpw) {
        const int r = warp * rpw + k, atom = lane >> 3, j = lane & 7;
        *reinterpret_cast<uint4*>(sA + atom * (kM * kAtomBytes) + (r >> 3) * 1024 +
                                  (r & 7) * 128 + ((j ^ (r & 7)) << 4)) = sv[k];
      }
    }
  }
}

template <int DMAX>
__global__ void __launch_bounds__(kThreads, 1)
    k_sage_hidden(const int32_t* __restrict__ indptr, const int32_t* __restrict__ idx,
                  const int64_t* __restrict__ n_dst_dev, int64_t n_dst_cap,
                  const uint4* __restrict__ yp, int64_t yp_ld8, int kin,
                  const uint4* __restrict__ w_img, const float* __restrict__ bias, int fo,
                  int tmem_cols, int relu, int out_bf16, void* __restrict__ out, int64_t out_ld,
                  int rows_per_tile, int halves = 2, void* __restrict__ out2 = nullptr,
                  int64_t out2_ld = 0) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024 - (saddr(smem_raw) & 1023)) & 1023);
  const uint32_t abytes = static_cast<uint32_t>(kin) * kM * kAtomBytes;
  const uint32_t wbytes = static_cast<uint32_t>(kin) * fo * kAtomBytes;  // one half
  uint8_t* sA = smem;
  uint8_t* sW = sA + abytes;
  uint64_t* bar = reinterpret_cast<uint64_t*>(sW + wbytes);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bar + 1);
  float* sbias = reinterpret_cast<float*>(bar + 8);

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  constexpr unsigned kFull = 0xffffffffu;
  const int64_t n_dst = min(*n_dst_dev, n_dst_cap);
  // R = rows_per_tile (32, 64 or 128) real rows per 128-row MMA tile: a layer with few dst rows
  // (the last layer: 1024 roots) is spread over more CTAs, R / 16 rows per warp
  const int R = rows_per_tile, rpw = R / kWarps;
  const int64_t ntiles = (n_dst + R - 1) / R;
  const uint32_t wbar = saddr(bar + 2);
  uint32_t wphase = 0;
  for (int i = tid; i < fo; i += kThreads) sbias[i] = bias ? __ldg(bias + i) : 0.f;
  if (tid == 0) {
    mbar_init(saddr(bar), 1);
    mbar_init(wbar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     saddr(tmem_slot)),
                 "r"(tmem_cols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t idesc = idesc_bf16(kM, fo);
  const uint32_t sA_addr = saddr(sA), sW_addr = saddr(sW);
  const bool col = lane < kin * 8;  // lane owns columns 8*lane .. 8*lane+7
  const uint64_t pol_stream = l2_evict_first();
  uint32_t phase = 0;

  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int64_t rbase = tile * R + warp * rpw;
    const int64_t rem = n_dst - rbase;
    const int nr = rem <= 0 ? 0 : (rem >= rpw ? rpw : static_cast<int>(rem));
    // phase 0 = the neighbour half (A = bf16 neighbour means, W half 1), phase 1 = the self half
    // (A = the dst rows of Yp, W half 0); each W half is bulk-copied from L2 while A is built
    const int32_t ip = (lane <= nr && nr > 0) ? __ldg(indptr + rbase + lane) : 0;
    // halves == 1: the self phase only, against the image's first half (input gradients, R32);
    // dual (halves == 1, out2 != NULL): A = the self rows built once, multiplied by the image's
    // first half into TMEM columns [0, fo) and by its second half into [fo, 2 fo) -> out, out2
    const int ph0 = halves == 1 ? 1 : 0;
    const bool dual = halves == 1 && out2 != nullptr;
    for (int k = 0; k < (dual ? 2 : 2 - ph0); ++k) {
      const int ph = dual ? 1 : ph0 + k;
      const int whalf = dual ? k : (ph == 0 ? 1 : 0);
      if (tid == 0) bulk_g2s(saddr(sW), w_img + whalf * (wbytes / 16), wbytes, wbar);
      if (!(dual && k == 1))
        hid_build_half<DMAX>(ph, idx, yp, yp_ld8, ip, rbase, nr, rpw, warp, lane, col, sA);
      fence_async_smem();
      __syncthreads();
      if (tid == 0) {
        mbar_wait(wbar, wphase);
        tc_fence_after();
        const uint32_t dcol = dual ? static_cast<uint32_t>(k * fo) : 0u;
        for (int st = 0; st < kin * 4; ++st) {
          const uint32_t atom = static_cast<uint32_t>(st >> 2);
          const uint32_t koff = static_cast<uint32_t>(st & 3) * 32u;
          mma_bf16(tmem + dcol, sw128_desc(sA_addr + atom * (kM * kAtomBytes) + koff),
                   sw128_desc(sW_addr + atom * (fo * kAtomBytes) + koff), idesc,
                   ((!dual && ph > ph0) || st > 0) ? 1u : 0u);
        }
        mma_commit(saddr(bar));
      }
      mbar_wait(saddr(bar), phase);  // A / W free again, accumulator complete after phase 1
      phase ^= 1;
      wphase ^= 1;
      tc_fence_after();
      __syncthreads();
    }
    // ---- epilogue (as the first layer's; dual: both accumulators, to out and out2)
    for (int qo = 0; qo < (dual ? 2 : 1); ++qo) {
      void* const dst = qo ? out2 : out;
      const int64_t dst_ld = qo ? out2_ld : out_ld;
      const int q = warp & 3;
      const int64_t row = tile * R + q * 32 + lane;
      const bool live = q * 32 + lane < R && row < n_dst;
      for (int ch = warp >> 2; ch < fo / 16; ch += kWarps / 4) {
        uint32_t v[16];
        tmem_ld16(tmem + (static_cast<uint32_t>(q * 32) << 16) +
                      static_cast<uint32_t>(qo * fo + ch * 16), v);
        tmem_ld_wait();
        float y[16];
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          y[i] = __fadd_rn(__uint_as_float(v[i]), sbias[ch * 16 + i]);
          if (relu) y[i] = fmaxf(y[i], 0.f);
        }
        if (live) {
          if (out_bf16) {
            uint4* o = reinterpret_cast<uint4*>(static_cast<__nv_bfloat16*>(dst) + row * dst_ld +
                                                ch * 16);
            uint32_t p[8];
#pragma unroll
            for (int i = 0; i < 8; ++i) {
              const __nv_bfloat162 b2 = __floats2bfloat162_rn(y[2 * i], y[2 * i + 1]);
              p[i] = *reinterpret_cast<const uint32_t*>(&b2);
            }
            st16_hint(o, make_uint4(p[0], p[1], p[2], p[3]), pol_stream);
            st16_hint(o + 1, make_uint4(p[4], p[5], p[6], p[7]), pol_stream);
          } else {
            uint4* o = reinterpret_cast<uint4*>(static_cast<float*>(dst) + row * dst_ld + ch * 16);
#pragma unroll
            for (int i = 0; i < 4; ++i)
              st16_hint(o + i, make_uint4(__float_as_uint(y[4 * i]), __float_as_uint(y[4 * i + 1]),
                                          __float_as_uint(y[4 * i + 2]), __float_as_uint(y[4 * i + 3])),
                        pol_stream);
          }
        }
      }
    }
    tc_fence_before();
    __syncthreads();
  }
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                 "r"(tmem_cols)
                 : "memory");
  }
}

// ----------------------------------------------------------------- NEXT-4: hidden backward (R31)
// Weight gradients of a hidden layer (reading R31 = R27 on the R29 layer):
//     dZ = dY * 1[Y > 0],  dW_self = Yp[0:n_dst]^T dZ,  dW_neigh = H^T dZ,  db = sum_d dZ[d],
// H = the bf16 neighbour means the forward builds.  As in k_sage_layer_bwd the reduction runs over
// the dst rows (M = features, N = Fo, K = rows; A read MN-major from the forward's K-major image,
// dZ staged MN-major).  One half's accumulator ([kin2*64 x Fo] fp32 = kin2/2 M blocks of Fo TMEM
// columns, 512 at Fin = Fo = 256) is all TMEM holds, so every CTA makes two passes over its tiles
// -- neighbour half, then self half -- and drains TMEM into its partial between them; partials
// are summed in fp64 by k_sage_bwd_reduce (deterministic).  R real rows per 128-row tile as in the
// forward; the rest of the tile is zero in A and in dZ.
inline size_t hid_bwd_smem_bytes(int kin2, int fo) {
  return 1024 + static_cast<size_t>(kin2) * kM * kAtomBytes + b_bytes(fo) + 64 +
         static_cast<size_t>(fo) * 4;
}

template <int DMAX>
__global__ void __launch_bounds__(kThreads, 1)
    k_sage_hidden_bwd(const int32_t* __restrict__ indptr, const int32_t* __restrict__ idx,
                      const int64_t* __restrict__ n_dst_dev, int64_t n_dst_cap,
                      const uint4* __restrict__ yp, int64_t yp_ld8, int kin,
                      const void* __restrict__ dy, int64_t dy_ld, int dy_f32,
                      const __nv_bfloat16* __restrict__ y, int64_t y_ld, int fo, int tmem_alloc,
                      int rows_per_tile, float* __restrict__ part, float* __restrict__ part_db,
                      __nv_bfloat16* __restrict__ dz_out, int64_t dz_ld) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024 - (saddr(smem_raw) & 1023)) & 1023);
  const int kin2 = (kin + 1) & ~1;  // atoms of the A image (whole 128-feature M blocks)
  const uint32_t abytes = static_cast<uint32_t>(kin2) * kM * kAtomBytes;
  uint8_t* sA = smem;
  uint8_t* sB = sA + abytes;
  uint64_t* bar = reinterpret_cast<uint64_t*>(sB + b_bytes(fo));
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bar + 1);
  float* sdb = reinterpret_cast<float*>(bar + 8);

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t n_dst = min(*n_dst_dev, n_dst_cap);
  const int R = rows_per_tile, rpw = R / kWarps;
  const int64_t ntiles = (n_dst + R - 1) / R;
  const int m_all = 2 * kin2 * 64;
  const int nmb = kin2 / 2;  // M blocks of one half

  // A and dZ start as zeros: rows R..127 of a tile and the padding atom are never written
  for (uint32_t i = tid; i < (abytes + b_bytes(fo)) / 16; i += kThreads)
    reinterpret_cast<uint4*>(sA)[i] = make_uint4(0u, 0u, 0u, 0u);
  for (int i = tid; i < fo; i += kThreads) sdb[i] = 0.f;
  if (tid == 0) {
    mbar_init(saddr(bar), 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     saddr(tmem_slot)),
                 "r"(tmem_alloc)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  const int cpr = fo / 8;  // dZ staging: thread owns 8-column chunk c of rows tid / cpr + i*rstep
  const int c = tid % cpr;
  const int rstep = kThreads / cpr;
  float dbacc[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) dbacc[i] = 0.f;
  const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | (1u << 15) | (1u << 16) |
                         (static_cast<uint32_t>(fo >> 3) << 17) | (static_cast<uint32_t>(kM >> 4) << 24);
  const uint32_t sA_addr = saddr(sA), sB_addr = saddr(sB);
  const bool col = lane < kin * 8;
  uint32_t phase = 0;

  for (int ph = 0; ph < 2; ++ph) {  // ph 0: neighbour half (dW_neigh), ph 1: self half (dW_self)
    int it = 0;
    for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++it) {
      const int64_t rbase = tile * R + warp * rpw;
      const int64_t rem = n_dst - rbase;
      const int nr = rem <= 0 ? 0 : (rem >= rpw ? rpw : static_cast<int>(rem));
      const int32_t ip = (ph == 0 && lane <= nr && nr > 0) ? __ldg(indptr + rbase + lane) : 0;
      hid_build_half<DMAX>(ph, idx, yp, yp_ld8, ip, rbase, nr, rpw, warp, lane, col, sA);
      // four of the thread's rows at a time: all their loads first, then mask / dZ out / sums
      for (int r0 = tid / cpr; r0 < R; r0 += 4 * rstep) {
        uint4 v[4], m[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int r = r0 + u * rstep;
          const int64_t row = tile * R + r;
          const bool live = r < R && row < n_dst;
          v[u] = live ? load_dy8(dy, dy_f32, row, dy_ld, c) : make_uint4(0u, 0u, 0u, 0u);
          m[u] = (live && y) ? __ldg(reinterpret_cast<const uint4*>(y + row * y_ld) + c)
                             : make_uint4(0u, 0u, 0u, 0u);
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int r = r0 + u * rstep;
          if (r >= R) break;
          const int64_t row = tile * R + r;
          if (y) {
            const uint32_t* mw = reinterpret_cast<const uint32_t*>(&m[u]);
            uint32_t* vw = reinterpret_cast<uint32_t*>(&v[u]);
#pragma unroll
            for (int i = 0; i < 4; ++i) {  // keep dY where Y > 0 (bf16 sign bit clear, nonzero)
              const uint32_t lo = mw[i] & 0xFFFFu, hi = mw[i] >> 16;
              const uint32_t keep = ((lo != 0u && !(lo & 0x8000u)) ? 0xFFFFu : 0u) |
                                    ((hi != 0u && !(hi & 0x8000u)) ? 0xFFFF0000u : 0u);
              vw[i] &= keep;
            }
          }
          if (ph == 0 && row < n_dst) {
            if (dz_out)  // the masked dZ, the A operand of the input-gradient GEMMs (R32)
              *reinterpret_cast<uint4*>(dz_out + row * dz_ld + c * 8) = v[u];
            const __nv_bfloat162* p2 = reinterpret_cast<const __nv_bfloat162*>(&v[u]);
#pragma unroll
            for (int i = 0; i < 4; ++i) {
              const float2 f2 = __bfloat1622float2(p2[i]);
              dbacc[2 * i] += f2.x;
              dbacc[2 * i + 1] += f2.y;
            }
          }
          const uint32_t off = static_cast<uint32_t>(c >> 3) * (kM * kAtomBytes) + (r >> 3) * 1024 +
                               (r & 7) * 128 + (((c & 7) ^ (r & 7)) << 4);
          *reinterpret_cast<uint4*>(sB + off) = v[u];
        }
      }
      fence_async_smem();
      __syncthreads();
      if (tid == 0) {
        tc_fence_after();
        for (int mb = 0; mb < nmb; ++mb) {
          for (int ks = 0; ks < kM / 16; ++ks) {
            const uint64_t da = sw128_mn_desc(sA_addr + (2 * mb) * (kM * kAtomBytes) + ks * 2048,
                                              kM * kAtomBytes);
            const uint64_t db = sw128_mn_desc(sB_addr + ks * 2048, kM * kAtomBytes);
            mma_bf16(tmem + static_cast<uint32_t>(mb * fo), da, db, idesc,
                     (it > 0 || ks > 0) ? 1u : 0u);
          }
        }
        mma_commit(saddr(bar));
      }
      mbar_wait(saddr(bar), phase);  // A and dZ may be overwritten once the MMAs have read them
      phase ^= 1;
      tc_fence_after();
      __syncthreads();
    }
    // drain this half's accumulator into the CTA's partial (half h = 1 - ph in the reduce's order)
    const int h = 1 - ph;
    const int q = warp & 3;
    for (int mb = 0; mb < nmb; ++mb) {
      const int m = h * kin2 * 64 + mb * kM + q * 32 + lane;
      float* dst = part + (static_cast<int64_t>(blockIdx.x) * m_all + m) * fo;
      for (int ch = warp >> 2; ch < fo / 16; ch += kWarps / 4) {
        uint32_t v[16];
        tmem_ld16(tmem + (static_cast<uint32_t>(q * 32) << 16) +
                      static_cast<uint32_t>(mb * fo + ch * 16), v);
        tmem_ld_wait();
#pragma unroll
        for (int i = 0; i < 4; ++i)
          reinterpret_cast<float4*>(dst + ch * 16)[i] =
              it > 0 ? make_float4(__uint_as_float(v[4 * i]), __uint_as_float(v[4 * i + 1]),
                                   __uint_as_float(v[4 * i + 2]), __uint_as_float(v[4 * i + 3]))
                     : make_float4(0.f, 0.f, 0.f, 0.f);
      }
    }
    tc_fence_before();  // the next pass's MMAs overwrite the columns just read
    __syncthreads();
    tc_fence_after();
  }
  {  // db: the per-thread column sums added in a fixed order (deterministic; dZ's tile is free)
    float* buf = reinterpret_cast<float*>(sB);
#pragma unroll
    for (int i = 0; i < 8; ++i) buf[(tid / cpr) * fo + c * 8 + i] = dbacc[i];
    __syncthreads();
    for (int i = tid; i < fo; i += kThreads) {
      float t = 0.f;
      for (int j = 0; j < rstep; ++j) t += buf[j * fo + i];
      sdb[i] = t;
    }
  }
  __syncthreads();
  for (int i = tid; i < fo; i += kThreads) part_db[static_cast<int64_t>(blockIdx.x) * fo + i] = sdb[i];
  if (warp == 0) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                 "r"(tmem_alloc)
                 : "memory");
  }
}

// ----------------------------------------------------------------- NEXT-4: a5 backward (R30)
// dX[idx[e]] += dH[d] / deg_d over the transposed block: one warp per dst row (grid stride), the
// row's edge ids lane-parallel, lane c scaling float4 column c of dH[d] by RN(1/deg) once and
// adding it into every src row with a vector fp32 reduction (one REDG.F32x4 per edge per lane,
// resolved at L2 -- no read-modify-write round trip in the SM).
__device__ __forceinline__ void red_add4(float* p, const float4& v) {
  asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(p), "f"(v.x), "f"(v.y),
               "f"(v.z), "f"(v.w)
               : "memory");
}
__global__ void __launch_bounds__(256) k_sage_mean_bwd(const int32_t* __restrict__ indptr,
                                                       const int32_t* __restrict__ idx,
                                                       const int64_t* __restrict__ n_dst_dev,
                                                       int64_t n_dst_cap, const float* __restrict__ dh,
                                                       int64_t dh_ld, int F, float* __restrict__ dx,
                                                       int64_t dx_ld) {
  constexpr unsigned kFull = 0xffffffffu;
  const int64_t n_dst = min(*n_dst_dev, n_dst_cap);
  const int lane = threadIdx.x & 31;
  const int64_t W = static_cast<int64_t>(gridDim.x) * (blockDim.x >> 5);
  const int f4 = (F + 3) >> 2;
  for (int64_t row = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; row < n_dst;
       row += W) {
    const int32_t e0 = __ldg(indptr + row), e1 = __ldg(indptr + row + 1);
    const int deg = e1 - e0;
    if (deg <= 0) continue;  // warp-uniform
    const float y = __frcp_rn(static_cast<float>(deg));
    for (int eb = 0; eb < deg; eb += 32) {  // sampled rows have deg <= 32: one pass
      const int32_t my = eb + lane < deg ? __ldg(idx + e0 + eb + lane) : 0;
      const int ne = deg - eb < 32 ? deg - eb : 32;
      for (int c0 = 0; c0 < f4; c0 += 32) {
        const int c = c0 + lane;
        float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
        if (c < f4) {
          v = __ldg(reinterpret_cast<const float4*>(dh + row * dh_ld) + c);
          v = make_float4(v.x * y, v.y * y, v.z * y, v.w * y);
          if (4 * c + 4 > F) {  // the columns past F stay untouched (added as 0)
            if (4 * c + 1 >= F) v.y = 0.f;
            if (4 * c + 2 >= F) v.z = 0.f;
            if (4 * c + 3 >= F) v.w = 0.f;
          }
        }
        for (int j = 0; j < ne; ++j) {
          const int32_t s = __shfl_sync(kFull, my, j);
          if (c < f4) red_add4(dx + static_cast<int64_t>(s) * dx_ld + 4 * c, v);
        }
      }
    }
  }
}

inline bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

}  // namespace sl
}  // namespace cmb

using namespace cmb;

extern "C" {

size_t cmb_sage_weights_bytes(int32_t feat_dim, int32_t out_dim) {
  if (feat_dim < 1 || feat_dim > 128 || out_dim < 16 || out_dim > 256 || out_dim % 16) return 0;
  return sl::w_img_bytes((feat_dim + 63) / 64, out_dim);
}

cmb_status cmb_sage_pack_weights(const float* w_self, const float* w_neigh, int32_t feat_dim,
                                 int32_t out_dim, void* w_img, size_t w_img_bytes, void* stream) {
  CMB_ARG(w_self && w_neigh && w_img, "cmb_sage_pack_weights: null argument");
  const size_t need = cmb_sage_weights_bytes(feat_dim, out_dim);
  CMB_ARG(need != 0, "cmb_sage_pack_weights: need 1 <= feat_dim <= 128, out_dim in [16, 256] "
                     "and a multiple of 16 (got %d, %d)", feat_dim, out_dim);
  CMB_ARG(w_img_bytes >= need, "cmb_sage_pack_weights: w_img_bytes %zu < %zu", w_img_bytes, need);
  CMB_ARG(sl::aligned16(w_img), "cmb_sage_pack_weights: w_img must be 16-byte aligned");
  cmb_status st = require_sm100();
  if (st != CMB_OK) return st;
  const int kh = (feat_dim + 63) / 64;
  const int64_t total = static_cast<int64_t>(2 * kh * 64) * out_dim;
  sl::k_pack_weights<<<static_cast<int>((total + 255) / 256), 256, 0,
                       static_cast<cudaStream_t>(stream)>>>(
      w_self, w_neigh, feat_dim, out_dim, kh, static_cast<__nv_bfloat16*>(w_img));
  CMB_CUDA(cudaGetLastError());
  return CMB_OK;
}

static cmb_status layer_forward(const cmb_graph* g, const cmb_blocks* b, int32_t n_hops,
                                int64_t n_last_dst_cap, const void* w_img, const float* bias,
                                int32_t out_dim, int32_t relu, int32_t out_bf16, void* out,
                                int64_t out_ld, void* stream, int halves,
                                void* a_save = nullptr) {
  CMB_ARG(g && b && w_img && out, "cmb_sage_layer_forward: null argument");
  CMB_ARG(n_hops >= 1 && n_hops <= CMB_MAX_HOPS, "cmb_sage_layer_forward: bad n_hops");
  CMB_ARG(g->d.x != nullptr, "cmb_sage_layer_forward: graph has no feature table");
  const int F = g->d.f;
  CMB_ARG(cmb_sage_weights_bytes(F, out_dim) != 0,
          "cmb_sage_layer_forward: need feat_dim <= 128 and out_dim in [16, 256], a multiple of 16 "
          "(got %d, %d)", F, out_dim);
  CMB_ARG(b->last_src_ids != nullptr, "cmb_sage_layer_forward: blocks->last_src_ids is required");
  CMB_ARG(g->d.ld % 4 == 0 && sl::aligned16(g->d.x), "cmb_sage_layer_forward: feature rows must "
                                                      "be 16-byte aligned (ld %% 4 == 0)");
  CMB_ARG(out_ld >= out_dim && out_ld % (out_bf16 ? 8 : 4) == 0 && sl::aligned16(out),
          "cmb_sage_layer_forward: out_ld must be >= out_dim and keep rows 16-byte aligned");
  CMB_ARG(sl::aligned16(w_img), "cmb_sage_layer_forward: w_img must be 16-byte aligned");
  CMB_ARG(n_last_dst_cap >= 0 && n_last_dst_cap <= b->nodes_cap,
          "cmb_sage_layer_forward: bad n_last_dst_cap");
  if (n_last_dst_cap == 0) return CMB_OK;
  const int L = n_hops;
  const int kh = (F + 63) / 64;
  const int cols = out_dim <= 32 ? 32 : out_dim <= 64 ? 64 : out_dim <= 128 ? 128 : 256;
  const size_t smem = sl::smem_bytes(kh, out_dim);
  const size_t smem_max = sl::smem_bytes(2, 256);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const int64_t tiles = (n_last_dst_cap + sl::kM - 1) / sl::kM;
  const int grid = static_cast<int>(tiles < g->num_sms ? tiles : g->num_sms);
  const int dmax = static_cast<int>(b->indices_cap[L - 1] / n_last_dst_cap);  // max fanout
  CMB_SMEM((&sl::k_sage_layer<5, 2>), smem_max);
  CMB_SMEM((&sl::k_sage_layer<10, 2>), smem_max);
#define CMB_LAYER_ARGS                                                                        \
  b->indptr[L - 1], b->last_src_ids, b->sizes + (L - 1), n_last_dst_cap,                     \
      reinterpret_cast<const float4*>(g->d.x), g->d.ld / 4, b->nodes, F, kh,                 \
      static_cast<const uint4*>(w_img), bias, out_dim, cols, relu, out_bf16, out, out_ld, halves, \
      static_cast<uint8_t*>(a_save)
  if (dmax <= 5)
    sl::k_sage_layer<5, 2><<<grid, sl::kThreads, smem, s>>>(CMB_LAYER_ARGS);
  else
    sl::k_sage_layer<10, 2><<<grid, sl::kThreads, smem, s>>>(CMB_LAYER_ARGS);
#undef CMB_LAYER_ARGS
  CMB_CUDA(cudaGetLastError());
  return CMB_OK;
}

cmb_status cmb_sage_layer_forward(const cmb_graph* g, const cmb_blocks* b, int32_t n_hops,
                                  int64_t n_last_dst_cap, const void* w_img, const float* bias,
                                  int32_t out_dim, int32_t relu, int32_t out_bf16, void* out,
                                  int64_t out_ld, void* stream) {
  CMB_NVTX("cmb.next4.sage_layer_forward");
  return layer_forward(g, b, n_hops, n_last_dst_cap, w_img, bias, out_dim, relu, out_bf16, out,
                       out_ld, stream, 2);
}

size_t cmb_sage_saved_a_bytes(int32_t feat_dim, int64_t n_last_dst_cap) {
  if (feat_dim < 1 || feat_dim > 128 || n_last_dst_cap < 0) return 0;
  return static_cast<size_t>((n_last_dst_cap + sl::kM - 1) / sl::kM) * sl::a_bytes((feat_dim + 63) / 64);
}

cmb_status cmb_sage_layer_forward_save(const cmb_graph* g, const cmb_blocks* b, int32_t n_hops,
                                       int64_t n_last_dst_cap, const void* w_img,
                                       const float* bias, int32_t out_dim, int32_t relu,
                                       int32_t out_bf16, void* out, int64_t out_ld, void* a_save,
                                       size_t a_save_bytes, void* stream) {
  CMB_NVTX("cmb.next4.sage_layer_forward_save");
  CMB_ARG(a_save && g, "cmb_sage_layer_forward_save: null argument");
  const size_t need = cmb_sage_saved_a_bytes(g->d.f, n_last_dst_cap);
  CMB_ARG(a_save_bytes >= need && sl::aligned16(a_save),
          "cmb_sage_layer_forward_save: a_save smaller than %zu bytes or unaligned", need);
  return layer_forward(g, b, n_hops, n_last_dst_cap, w_img, bias, out_dim, relu, out_bf16, out,
                       out_ld, stream, 2, a_save);
}

size_t cmb_gcn_weights_bytes(int32_t feat_dim, int32_t out_dim) {
  const size_t n = cmb_sage_weights_bytes(feat_dim, out_dim);
  return n / 2;
}

cmb_status cmb_gcn_pack_weights(const float* w, int32_t feat_dim, int32_t out_dim, void* w_img,
                                size_t w_img_bytes, void* stream) {
  CMB_ARG(w && w_img, "cmb_gcn_pack_weights: null argument");
  const size_t need = cmb_gcn_weights_bytes(feat_dim, out_dim);
  CMB_ARG(need != 0, "cmb_gcn_pack_weights: need 1 <= feat_dim <= 128, out_dim in [16, 256] "
                     "and a multiple of 16 (got %d, %d)", feat_dim, out_dim);
  CMB_ARG(w_img_bytes >= need, "cmb_gcn_pack_weights: w_img_bytes %zu < %zu", w_img_bytes, need);
  CMB_ARG(sl::aligned16(w_img), "cmb_gcn_pack_weights: w_img must be 16-byte aligned");
  cmb_status st = require_sm100();
  if (st != CMB_OK) return st;
  const int kh = (feat_dim + 63) / 64;
  const int64_t total = static_cast<int64_t>(kh * 64) * out_dim;
  sl::k_pack_weights<<<static_cast<int>((total + 255) / 256), 256, 0,
                       static_cast<cudaStream_t>(stream)>>>(
      w, nullptr, feat_dim, out_dim, kh, static_cast<__nv_bfloat16*>(w_img));
  CMB_CUDA(cudaGetLastError());
  return CMB_OK;
}

cmb_status cmb_gcn_layer_forward(const cmb_graph* g, const cmb_blocks* b, int32_t n_hops,
                                 int64_t n_last_dst_cap, const void* w_img, const float* bias,
                                 int32_t out_dim, int32_t relu, int32_t out_bf16, void* out,
                                 int64_t out_ld, void* stream) {
  CMB_NVTX("cmb.next4.gcn_layer_forward");
  return layer_forward(g, b, n_hops, n_last_dst_cap, w_img, bias, out_dim, relu, out_bf16, out,
                       out_ld, stream, 1);
}

size_t cmb_sage_backward_workspace_bytes(int32_t feat_dim, int32_t out_dim) {
  if (cmb_sage_weights_bytes(feat_dim, out_dim) == 0 || (out_dim & (out_dim - 1))) return 0;
  const size_t kh = (feat_dim + 63) / 64;
  return static_cast<size_t>(sl::kMaxBwdCtas) * (2 * kh * 64 + 1) * out_dim * sizeof(float);
}

static cmb_status layer_backward(const cmb_graph* g, const cmb_blocks* b, int32_t n_hops,
                                 int64_t n_last_dst_cap, const void* dy, int64_t dy_ld,
                                 int32_t dy_f32, const void* y, int64_t y_ld, int32_t out_dim,
                                 float* dw, float* db, void* workspace, size_t workspace_bytes,
                                 void* stream, const void* a_saved, int gcn = 0) {
  CMB_ARG(g && b && dy && dw && db && workspace, "cmb_sage_layer_backward: null argument");
  CMB_ARG(n_hops >= 1 && n_hops <= CMB_MAX_HOPS, "cmb_sage_layer_backward: bad n_hops");
  CMB_ARG(g->d.x != nullptr, "cmb_sage_layer_backward: graph has no feature table");
  const int F = g->d.f;
  const size_t need = cmb_sage_backward_workspace_bytes(F, out_dim);
  CMB_ARG(need != 0, "cmb_sage_layer_backward: need feat_dim <= 128 and out_dim a power of two "
                     "in [16, 256] (got %d, %d)", F, out_dim);
  CMB_ARG(workspace_bytes >= need && sl::aligned16(workspace),
          "cmb_sage_layer_backward: workspace < %zu bytes or unaligned", need);
  CMB_ARG(b->last_src_ids != nullptr, "cmb_sage_layer_backward: blocks->last_src_ids is required");
  CMB_ARG(g->d.ld % 4 == 0 && sl::aligned16(g->d.x),
          "cmb_sage_layer_backward: feature rows must be 16-byte aligned (ld %% 4 == 0)");
  CMB_ARG(dy_ld >= out_dim && dy_ld % (dy_f32 ? 4 : 8) == 0 && sl::aligned16(dy) &&
              (!y || (y_ld >= out_dim && y_ld % 8 == 0 && sl::aligned16(y))),
          "cmb_sage_layer_backward: dy (bf16 or fp32) / y (bf16) rows must be 16-byte aligned "
          "with ld >= out_dim");
  CMB_ARG(n_last_dst_cap >= 0 && n_last_dst_cap <= b->nodes_cap,
          "cmb_sage_layer_backward: bad n_last_dst_cap");
  const int L = n_hops;
  const int kh = (F + 63) / 64;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const int64_t tiles = (n_last_dst_cap + sl::kM - 1) / sl::kM;
  int grid = static_cast<int>(tiles < g->num_sms ? tiles : g->num_sms);
  if (grid > sl::kMaxBwdCtas) grid = sl::kMaxBwdCtas;
  float* part = static_cast<float*>(workspace);
  float* part_db = part + static_cast<size_t>(sl::kMaxBwdCtas) * 2 * kh * 64 * out_dim;
  if (grid > 0) {
    int cols = kh * out_dim;
    int alloc = 32;
    while (alloc < cols) alloc <<= 1;
    const size_t smem = sl::bwd_smem_bytes(kh, out_dim);
    CMB_SMEM((&sl::k_sage_layer_bwd<5, 2>), sl::bwd_smem_bytes(2, 256));
    CMB_SMEM((&sl::k_sage_layer_bwd<10, 2>), sl::bwd_smem_bytes(2, 256));
    const int dmax = static_cast<int>(b->indices_cap[L - 1] / n_last_dst_cap);
#define CMB_BWD_ARGS                                                                          \
  b->indptr[L - 1], b->last_src_ids, b->sizes + (L - 1), n_last_dst_cap,                     \
      reinterpret_cast<const float4*>(g->d.x), g->d.ld / 4, b->nodes, F, kh,                 \
      dy, dy_ld, dy_f32, static_cast<const __nv_bfloat16*>(y), y_ld,                         \
      out_dim, alloc, part, part_db, static_cast<const uint8_t*>(a_saved), gcn
    if (dmax <= 5)
      sl::k_sage_layer_bwd<5, 2><<<grid, sl::kThreads, smem, s>>>(CMB_BWD_ARGS);
    else
      sl::k_sage_layer_bwd<10, 2><<<grid, sl::kThreads, smem, s>>>(CMB_BWD_ARGS);
#undef CMB_BWD_ARGS
    CMB_CUDA(cudaGetLastError());
  }
  const int halves = gcn ? 1 : 2;
  const int64_t nout = static_cast<int64_t>(halves) * F * out_dim + out_dim;
  sl::k_sage_bwd_reduce<<<static_cast<int>((nout + 31) / 32), 256, 0, s>>>(
      part, part_db, grid, F, kh, out_dim, dw, db, halves);
  CMB_CUDA(cudaGetLastError());
  return CMB_OK;
}

cmb_status cmb_sage_layer_backward(const cmb_graph* g, const cmb_blocks* b, int32_t n_hops,
                                   int64_t n_last_dst_cap, const void* dy, int64_t dy_ld,
                                   int32_t dy_f32, const void* y, int64_t y_ld, int32_t out_dim,
                                   float* dw, float* db, void* workspace, size_t workspace_bytes,
                                   void* stream) {
  CMB_NVTX("cmb.next4.sage_layer_backward");
  return layer_backward(g, b, n_hops, n_last_dst_cap, dy, dy_ld, dy_f32, y, y_ld, out_dim, dw, db,
                        workspace, workspace_bytes, stream, nullptr);
}

cmb_status cmb_sage_layer_backward_saved(const cmb_graph* g, const cmb_blocks* b, int32_t n_hops,
                                         int64_t n_last_dst_cap, const void* a_saved,
                                         size_t a_saved_bytes, const void* dy, int64_t dy_ld,
                                         int32_t dy_f32, const void* y, int64_t y_ld,
                                         int32_t out_dim, float* dw, float* db, void* workspace,
                                         size_t workspace_bytes, void* stream) {
  CMB_NVTX("cmb.next4.sage_layer_backward_saved");
  CMB_ARG(a_saved && g, "cmb_sage_layer_backward_saved: null argument");
  const size_t need = cmb_sage_saved_a_bytes(g->d.f, n_last_dst_cap);
  CMB_ARG(a_saved_bytes >= need && sl::aligned16(a_saved),
          "cmb_sage_layer_backward_saved: a_saved smaller than %zu bytes or unaligned", need);
  return layer_backward(g, b, n_hops, n_last_dst_cap, dy, dy_ld, dy_f32, y, y_ld, out_dim, dw, db,
                        workspace, workspace_bytes, stream, a_saved);
}

cmb_status cmb_gcn_layer_backward(const cmb_graph* g, const cmb_blocks* b, int32_t n_hops,
                                  int64_t n_last_dst_cap, const void* dy, int64_t dy_ld,
                                  int32_t dy_f32, const void* y, int64_t y_ld, int32_t out_dim,
                                  float* dw, float* db, void* workspace, size_t workspace_bytes,
                                  void* stream) {
  CMB_NVTX("cmb.next4.gcn_layer_backward");
  return layer_backward(g, b, n_hops, n_last_dst_cap, dy, dy_ld, dy_f32, y, y_ld, out_dim, dw, db,
                        workspace, workspace_bytes, stream, nullptr, 1);
}

size_t cmb_sage_hidden_weights_bytes(int32_t in_dim, int32_t out_dim) {
  if (in_dim < 64 || in_dim > 256 || in_dim % 64 || out_dim < 16 || out_dim > 256 || out_dim % 16)
    return 0;
  return sl::w_img_bytes(in_dim / 64, out_dim);
}

cmb_status cmb_sage_hidden_pack_weights(const float* w_self, const float* w_neigh, int32_t in_dim,
                                        int32_t out_dim, void* w_img, size_t w_img_bytes,
                                        void* stream) {
  CMB_ARG(w_self && w_neigh && w_img, "cmb_sage_hidden_pack_weights: null argument");
  const size_t need = cmb_sage_hidden_weights_bytes(in_dim, out_dim);
  CMB_ARG(need != 0, "cmb_sage_hidden_pack_weights: need in_dim in {64, 128, 192, 256} and "
                     "out_dim in [16, 256], a multiple of 16 (got %d, %d)", in_dim, out_dim);
  CMB_ARG(w_img_bytes >= need && sl::aligned16(w_img),
          "cmb_sage_hidden_pack_weights: w_img smaller than %zu bytes or unaligned", need);
  cmb_status st = require_sm100();
  if (st != CMB_OK) return st;
  const int kh = in_dim / 64;
  const int64_t total = static_cast<int64_t>(2 * kh * 64) * out_dim;
  sl::k_pack_weights<<<static_cast<int>((total + 255) / 256), 256, 0,
                       static_cast<cudaStream_t>(stream)>>>(
      w_self, w_neigh, in_dim, out_dim, kh, static_cast<__nv_bfloat16*>(w_img));
  CMB_CUDA(cudaGetLastError());
  return CMB_OK;
}

cmb_status cmb_sage_hidden_forward(const cmb_blocks* b, int32_t hop, int64_t n_dst_cap,
                                   const void* y_prev, int64_t y_prev_ld, int32_t in_dim,
                                   const void* w_img, const float* bias, int32_t out_dim,
                                   int32_t relu, int32_t out_bf16, void* out, int64_t out_ld,
                                   void* stream) {
  CMB_NVTX("cmb.next4.sage_hidden_forward");
  CMB_ARG(b && y_prev && w_img && out, "cmb_sage_hidden_forward: null argument");
  CMB_ARG(hop >= 0 && hop < CMB_MAX_HOPS && b->indptr[hop] && b->indices[hop],
          "cmb_sage_hidden_forward: bad hop");
  CMB_ARG(cmb_sage_hidden_weights_bytes(in_dim, out_dim) != 0,
          "cmb_sage_hidden_forward: need in_dim in {64, 128, 192, 256}, out_dim in [16, 256] and "
          "a multiple of 16 (got %d, %d)", in_dim, out_dim);
  CMB_ARG(y_prev_ld >= in_dim && y_prev_ld % 8 == 0 && sl::aligned16(y_prev),
          "cmb_sage_hidden_forward: y_prev rows must be 16-byte aligned bf16, ld >= in_dim");
  CMB_ARG(out_ld >= out_dim && out_ld % (out_bf16 ? 8 : 4) == 0 && sl::aligned16(out),
          "cmb_sage_hidden_forward: out_ld must be >= out_dim and keep rows 16-byte aligned");
  CMB_ARG(sl::aligned16(w_img), "cmb_sage_hidden_forward: w_img must be 16-byte aligned");
  CMB_ARG(n_dst_cap >= 0, "cmb_sage_hidden_forward: bad n_dst_cap");
  if (n_dst_cap == 0) return CMB_OK;
  cmb_status st = require_sm100();
  if (st != CMB_OK) return st;
  int dev = 0, sms = 0;
  CMB_CUDA(cudaGetDevice(&dev));
  CMB_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  const int kin = in_dim / 64;
  const int cols = out_dim <= 32 ? 32 : out_dim <= 64 ? 64 : out_dim <= 128 ? 128 : 256;
  const size_t smem = sl::hid_smem_bytes(kin, out_dim);
  CMB_SMEM((&sl::k_sage_hidden<8>), sl::hid_smem_bytes(4, 256));
  // fewer real rows per tile when the layer has fewer than one 128-row tile per SM
  int R = 128;
  while (R > 32 && (n_dst_cap + R - 1) / R < sms) R >>= 1;
  const int64_t tiles = (n_dst_cap + R - 1) / R;
  const int grid = static_cast<int>(tiles < sms ? tiles : sms);
  sl::k_sage_hidden<8><<<grid, sl::kThreads, smem, static_cast<cudaStream_t>(stream)>>>(
      b->indptr[hop], b->indices[hop], b->sizes + hop, n_dst_cap,
      static_cast<const uint4*>(y_prev), y_prev_ld / 8, kin, static_cast<const uint4*>(w_img), bias,
      out_dim, cols, relu, out_bf16, out, out_ld, R);
  CMB_CUDA(cudaGetLastError());
  return CMB_OK;
}

size_t cmb_sage_hidden_backward_workspace_bytes(int32_t in_dim, int32_t out_dim) {
  if (cmb_sage_hidden_weights_bytes(in_dim, out_dim) == 0 || (out_dim & (out_dim - 1))) return 0;
  const size_t kin2 = ((in_dim / 64) + 1) & ~1;
  return static_cast<size_t>(sl::kMaxBwdCtas) * (2 * kin2 * 64 + 1) * out_dim * sizeof(float);
}

cmb_status cmb_sage_hidden_backward(const cmb_blocks* b, int32_t hop, int64_t n_dst_cap,
                                    const void* y_prev, int64_t y_prev_ld, int32_t in_dim,
                                    const void* dy, int64_t dy_ld, int32_t dy_f32, const void* y,
                                    int64_t y_ld, int32_t out_dim, float* dw, float* db, void* workspace,
                                    size_t workspace_bytes, void* dz_out, int64_t dz_ld,
                                    void* stream) {
  CMB_NVTX("cmb.next4.sage_hidden_backward");
  CMB_ARG(b && y_prev && dy && dw && db && workspace, "cmb_sage_hidden_backward: null argument");
  CMB_ARG(!dz_out || (dz_ld >= out_dim && dz_ld % 8 == 0 && sl::aligned16(dz_out)),
          "cmb_sage_hidden_backward: dz_out rows must be 16-byte aligned bf16 with ld >= out_dim");
  CMB_ARG(hop >= 0 && hop < CMB_MAX_HOPS && b->indptr[hop] && b->indices[hop],
          "cmb_sage_hidden_backward: bad hop");
  const size_t need = cmb_sage_hidden_backward_workspace_bytes(in_dim, out_dim);
  CMB_ARG(need != 0, "cmb_sage_hidden_backward: need in_dim in {64, 128, 192, 256} and out_dim a "
                     "power of two in [16, 256] (got %d, %d)", in_dim, out_dim);
  CMB_ARG(workspace_bytes >= need && sl::aligned16(workspace),
          "cmb_sage_hidden_backward: workspace < %zu bytes or unaligned", need);
  CMB_ARG(y_prev_ld >= in_dim && y_prev_ld % 8 == 0 && sl::aligned16(y_prev),
          "cmb_sage_hidden_backward: y_prev rows must be 16-byte aligned bf16, ld >= in_dim");
  CMB_ARG(dy_ld >= out_dim && dy_ld % (dy_f32 ? 4 : 8) == 0 && sl::aligned16(dy) &&
              (!y || (y_ld >= out_dim && y_ld % 8 == 0 && sl::aligned16(y))),
          "cmb_sage_hidden_backward: dy (bf16 or fp32) / y (bf16) rows must be 16-byte aligned "
          "with ld >= out_dim");
  CMB_ARG(n_dst_cap >= 0, "cmb_sage_hidden_backward: bad n_dst_cap");
  cmb_status st = require_sm100();
  if (st != CMB_OK) return st;
  int dev = 0, sms = 0;
  CMB_CUDA(cudaGetDevice(&dev));
  CMB_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  const int kin = in_dim / 64, kin2 = (kin + 1) & ~1;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  int R = 128;
  while (R > 32 && (n_dst_cap + R - 1) / R < sms) R >>= 1;
  const int64_t tiles = (n_dst_cap + R - 1) / R;
  int grid = static_cast<int>(tiles < sms ? tiles : sms);
  if (grid > sl::kMaxBwdCtas) grid = sl::kMaxBwdCtas;
  float* part = static_cast<float*>(workspace);
  float* part_db = part + static_cast<size_t>(sl::kMaxBwdCtas) * 2 * kin2 * 64 * out_dim;
  if (grid > 0) {
    int alloc = 32;
    while (alloc < (kin2 / 2) * out_dim) alloc <<= 1;
    CMB_SMEM((&sl::k_sage_hidden_bwd<8>), sl::hid_bwd_smem_bytes(4, 256));
    sl::k_sage_hidden_bwd<8><<<grid, sl::kThreads, sl::hid_bwd_smem_bytes(kin2, out_dim), s>>>(
        b->indptr[hop], b->indices[hop], b->sizes + hop, n_dst_cap,
        static_cast<const uint4*>(y_prev), y_prev_ld / 8, kin, dy, dy_ld, dy_f32,
        static_cast<const __nv_bfloat16*>(y), y_ld, out_dim, alloc, R, part, part_db,
        static_cast<__nv_bfloat16*>(dz_out), dz_ld);
    CMB_CUDA(cudaGetLastError());
  }
  const int64_t nout = 2ll * in_dim * out_dim + out_dim;
  sl::k_sage_bwd_reduce<<<static_cast<int>((nout + 31) / 32), 256, 0, s>>>(
      part, part_db, grid, in_dim, kin2, out_dim, dw, db);
  CMB_CUDA(cudaGetLastError());
  return CMB_OK;
}

cmb_status cmb_sage_hidden_pack_weights_t(const float* w_self, const float* w_neigh,
                                          int32_t in_dim, int32_t out_dim, void* wt_img,
                                          size_t wt_img_bytes, void* stream) {
  CMB_ARG(w_self && w_neigh && wt_img, "cmb_sage_hidden_pack_weights_t: null argument");
  CMB_ARG(in_dim >= 16 && in_dim <= 256 && in_dim % 16 == 0 && out_dim >= 1 && out_dim <= 256,
          "cmb_sage_hidden_pack_weights_t: need in_dim in [16, 256] a multiple of 16 and "
          "1 <= out_dim <= 256 (got %d, %d)", in_dim, out_dim);
  const int kt = (out_dim + 63) / 64;  // K = out_dim, padded to whole 64-column atoms
  const size_t need = sl::w_img_bytes(kt, in_dim);
  CMB_ARG(wt_img_bytes >= need && sl::aligned16(wt_img),
          "cmb_sage_hidden_pack_weights_t: wt_img smaller than %zu bytes or unaligned", need);
  cmb_status st = require_sm100();
  if (st != CMB_OK) return st;
  const int64_t total = static_cast<int64_t>(2 * kt * 64) * in_dim;
  sl::k_pack_weights<<<static_cast<int>((total + 255) / 256), 256, 0,
                       static_cast<cudaStream_t>(stream)>>>(
      w_self, w_neigh, out_dim, in_dim, kt, static_cast<__nv_bfloat16*>(wt_img), 1);
  CMB_CUDA(cudaGetLastError());
  return CMB_OK;
}

size_t cmb_sage_hidden_weights_t_bytes(int32_t in_dim, int32_t out_dim) {
  if (in_dim < 16 || in_dim > 256 || in_dim % 16 || out_dim < 1 || out_dim > 256) return 0;
  return sl::w_img_bytes((out_dim + 63) / 64, in_dim);
}

cmb_status cmb_sage_hidden_input_grad(const cmb_blocks* b, int32_t hop, int64_t n_dst_cap,
                                      int64_t n_src_cap, const void* dz, int64_t dz_ld,
                                      int32_t out_dim, const void* wt_img, int32_t in_dim,
                                      float* dx, int64_t dx_ld, float* dh, int64_t dh_ld,
                                      void* stream) {
  CMB_NVTX("cmb.next4.sage_hidden_input_grad");
  CMB_ARG(b && dz && wt_img && dx && dh, "cmb_sage_hidden_input_grad: null argument");
  CMB_ARG(hop >= 0 && hop < CMB_MAX_HOPS && b->indptr[hop] && b->indices[hop],
          "cmb_sage_hidden_input_grad: bad hop");
  CMB_ARG(cmb_sage_hidden_weights_t_bytes(in_dim, out_dim) != 0,
          "cmb_sage_hidden_input_grad: need in_dim in [16, 256] a multiple of 16 and "
          "1 <= out_dim <= 256 (got %d, %d)", in_dim, out_dim);
  const int kt = (out_dim + 63) / 64;
  CMB_ARG(dz_ld >= kt * 64 && dz_ld % 8 == 0 && sl::aligned16(dz),
          "cmb_sage_hidden_input_grad: dz rows must be 16-byte aligned bf16 with ld >= "
          "out_dim rounded up to 64 (columns out_dim.. zero)");
  CMB_ARG(dx_ld >= in_dim && dx_ld % 4 == 0 && sl::aligned16(dx) && dh_ld >= in_dim &&
              dh_ld % 4 == 0 && sl::aligned16(dh),
          "cmb_sage_hidden_input_grad: dx / dh rows must be 16-byte aligned fp32, ld >= in_dim");
  CMB_ARG(n_dst_cap >= 0 && n_src_cap >= n_dst_cap, "cmb_sage_hidden_input_grad: bad capacities");
  cmb_status st = require_sm100();
  if (st != CMB_OK) return st;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  CMB_CUDA(cudaMemsetAsync(dx, 0, static_cast<size_t>(n_src_cap) * dx_ld * sizeof(float), s));
  if (n_dst_cap == 0) return CMB_OK;
  int dev = 0, sms = 0;
  CMB_CUDA(cudaGetDevice(&dev));
  CMB_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  CMB_SMEM((&sl::k_sage_hidden<8>), sl::hid_smem_bytes(4, 256));
  int R = 128;
  while (R > 32 && (n_dst_cap + R - 1) / R < sms) R >>= 1;
  const int64_t tiles = (n_dst_cap + R - 1) / R;
  const int grid = static_cast<int>(tiles < sms ? tiles : sms);
  int cols = 32;  // two accumulators of in_dim columns each
  while (cols < 2 * in_dim) cols <<= 1;
  const size_t smem = sl::hid_smem_bytes(kt, in_dim);
  // dX[d] = dZ[d] W_self^T for d < n_dst (stored) and dH = dZ W_neigh^T in ONE launch (A = dZ
  // staged once, the two image halves into two TMEM accumulators); then dX += M^T dH (R30)
  sl::k_sage_hidden<8><<<grid, sl::kThreads, smem, s>>>(
      b->indptr[hop], b->indices[hop], b->sizes + hop, n_dst_cap, static_cast<const uint4*>(dz),
      dz_ld / 8, kt, static_cast<const uint4*>(wt_img), nullptr, in_dim, cols, 0, 0, dx, dx_ld, R,
      1, dh, dh_ld);
  CMB_CUDA(cudaGetLastError());
  const int64_t want = (n_dst_cap + 7) / 8;
  const int mgrid = static_cast<int>(want < 8ll * sms ? want : 8ll * sms);
  sl::k_sage_mean_bwd<<<mgrid, 256, 0, s>>>(b->indptr[hop], b->indices[hop], b->sizes + hop,
                                            n_dst_cap, dh, dh_ld, in_dim, dx, dx_ld);
  CMB_CUDA(cudaGetLastError());
  return CMB_OK;
}

cmb_status cmb_sage_mean_backward(const int32_t* indptr, const int32_t* indices,
                                  const int64_t* n_dst_dev, int64_t n_dst_cap, const float* dh,
                                  int64_t dh_ld, int32_t feat_dim, float* dx, int64_t dx_ld,
                                  void* stream) {
  CMB_NVTX("cmb.next4.sage_mean_backward");
  CMB_ARG(indptr && indices && n_dst_dev && dh && dx, "cmb_sage_mean_backward: null argument");
  CMB_ARG(feat_dim >= 1 && dh_ld >= feat_dim && dx_ld >= feat_dim && dh_ld % 4 == 0 &&
              dx_ld % 4 == 0 && sl::aligned16(dh) && sl::aligned16(dx),
          "cmb_sage_mean_backward: rows must be 16-byte aligned fp32 with ld >= feat_dim");
  CMB_ARG(n_dst_cap >= 0, "cmb_sage_mean_backward: bad n_dst_cap");
  if (n_dst_cap == 0) return CMB_OK;
  cmb_status st = require_sm100();
  if (st != CMB_OK) return st;
  int dev = 0, sms = 0;
  CMB_CUDA(cudaGetDevice(&dev));
  CMB_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  const int64_t want = (n_dst_cap + 7) / 8;
  const int grid = static_cast<int>(want < 8ll * sms ? (want > 0 ? want : 1) : 8ll * sms);
  sl::k_sage_mean_bwd<<<grid, 256, 0, static_cast<cudaStream_t>(stream)>>>(
      indptr, indices, n_dst_dev, n_dst_cap, dh, dh_ld, feat_dim, dx, dx_ld);
  CMB_CUDA(cudaGetLastError());
  return CMB_OK;
}

}  // extern "C"
