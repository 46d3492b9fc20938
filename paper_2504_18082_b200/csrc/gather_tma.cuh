// gather_tma.cuh -- the TMA tile::gather4 form of the fused a4 + a5 kernel (included by
// features.cu; arithmetic as in the comment there).
//
// Each warp walks windows of 32 consecutive dst rows (grid stride over windows).  A window is
// a sequence of BATCHES of <= 32 feature rows: one SELF batch (its dst rows: X_in[d] =
// X[nodes[d]]) and EDGE batches (its edges [indptr[d0], indptr[d0+32]) in chunks of 32).  The
// producer side of the warp resolves a batch's row ids lane-parallel (coalesced index loads),
// arms the stage's mbarrier with the byte count and lanes 0..7 each issue ONE
// cp.async.bulk.tensor.2d.tile::gather4 -- four feature rows (W fp32 each) into 4 consecutive
// shared-memory slots -- so a 32-row batch costs 8 TMA instructions (SASS UTMALDG).  The
// consumer side waits on the mbarrier and folds the rows from shared memory in edge (= CSR)
// order: acc += row, X_in store at a first occurrence, H = acc / deg (IEEE) at the last edge of
// a row -- the oracle's fp32 order.  Up to kStages batches are in flight per warp, held in
// shared memory instead of registers.
#pragma once

namespace cmb {
namespace tma {

constexpr int kWarps = 4;   // warps per block
constexpr int kRows = 32;   // rows per batch (8 gather4 groups)

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
// four rows r0..r3, columns [0, W) of the 2D feature tensor -> 4 * W * 4 contiguous bytes
__device__ __forceinline__ void gather4(void* dst, const CUtensorMap* map, int r0, int r1, int r2,
                                        int r3, uint64_t* bar, uint64_t pol) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cta.global.tile::gather4.mbarrier::complete_tx::bytes"
      ".L2::cache_hint [%0], [%1, {%2, %3, %4, %5, %6}], [%7], %8;" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(0), "r"(r0), "r"(r1), "r"(r2), "r"(r3),
      "r"(smem_u32(bar)), "l"(pol)
      : "memory");
}

struct BatchHdr {
  int64_t d0;   // first dst row of the window
  int32_t cnt;  // rows in the batch
  int32_t self; // 1 = SELF batch
};

// bytes of one 4-row group in shared memory (TMA destinations are 128-byte aligned)
__host__ __device__ constexpr uint32_t group_bytes(uint32_t rb) { return (4 * rb + 127) / 128 * 128; }

__host__ __device__ constexpr size_t smem_bytes(uint32_t rb, int stages) {
  return (size_t)kWarps * stages * (kRows / 4) * group_bytes(rb) +   // row slots
         (size_t)kWarps * stages * kRows * sizeof(int2) +            // per-slot {li, meta}
         (size_t)kWarps * stages * sizeof(BatchHdr) +                // per-stage header
         (size_t)kWarps * stages * sizeof(uint64_t);                 // per-stage mbarrier
}

}  // namespace tma

template <int NV>
__global__ void __launch_bounds__(tma::kWarps * 32) k_gather_mean_tma(
    const __grid_constant__ CUtensorMap xmap, int stages, const int32_t* __restrict__ indptr,
    const int32_t* __restrict__ idx, const int32_t* __restrict__ gid,
    const int64_t* __restrict__ n_dst_dev, int64_t n_dst_cap, const int32_t* __restrict__ map,
    int f4, uint32_t rb, float4* __restrict__ out, int64_t out_ld4, float4* __restrict__ x_in,
    int64_t x_in_ld4, const uint32_t* __restrict__ new_mask) {
  using namespace tma;
  extern __shared__ __align__(128) unsigned char smem[];
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const uint32_t gb = group_bytes(rb);
  const size_t stage_bytes = (size_t)(kRows / 4) * gb;
  unsigned char* slots = smem + (size_t)warp * stages * stage_bytes;
  unsigned char* tail = smem + (size_t)kWarps * stages * stage_bytes;
  int2* smeta = reinterpret_cast<int2*>(tail) + warp * stages * kRows;
  BatchHdr* hdr =
      reinterpret_cast<BatchHdr*>(tail + (size_t)kWarps * stages * kRows * sizeof(int2)) +
      warp * stages;
  uint64_t* bars =
      reinterpret_cast<uint64_t*>(tail + (size_t)kWarps * stages * kRows * sizeof(int2) +
                                  (size_t)kWarps * stages * sizeof(BatchHdr)) +
      warp * stages;
  if (lane == 0) {
    for (int i = 0; i < stages; ++i) mbar_init(bars + i, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncwarp();
  uint64_t pol_keep, pol_stream;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol_keep));
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol_stream));
  auto ST = [&](float4* p, const float4& v) {
    asm volatile("st.global.L2::cache_hint.v4.f32 [%0], {%1, %2, %3, %4}, %5;" ::"l"(p),
                 "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w), "l"(pol_stream)
                 : "memory");
  };

  const int64_t n_dst = min(*n_dst_dev, n_dst_cap);
  const int64_t nwin = (n_dst + kRows - 1) / kRows;
  const int64_t G = (int64_t)gridDim.x * kWarps;
  const bool has_self = x_in != nullptr;
  const int rb4 = static_cast<int>(rb >> 4);
  const int gb4 = static_cast<int>(gb >> 4);

  // ---------------- producer state (window being issued)
  int64_t pw = (int64_t)blockIdx.x * kWarps + warp;
  int64_t pd0 = 0;
  int p_nr = 0;
  int32_t p_start = 0, p_end = 0, p_node = 0, p_eb = 0;
  int p_phase = 0;  // 1 = self batch next, 2 = edge batches
  auto load_window = [&]() -> bool {
    if (pw >= nwin) return false;
    pd0 = pw * kRows;
    p_nr = (n_dst - pd0 < kRows) ? static_cast<int>(n_dst - pd0) : kRows;
    p_start = lane < p_nr ? __ldg(indptr + pd0 + lane) : 0;
    p_end = __ldg(indptr + pd0 + p_nr);
    p_node = (has_self && lane < p_nr) ? __ldg(map + pd0 + lane) : 0;
    p_eb = __shfl_sync(0xffffffffu, p_start, 0);
    const int32_t nxt = __shfl_down_sync(0xffffffffu, p_start, 1);
    const int32_t my_end = lane + 1 < p_nr ? nxt : p_end;
    unsigned empty = __ballot_sync(0xffffffffu, lane < p_nr && my_end == p_start);
    while (empty) {  // rows without edges: H = 0 now
      const int r = __ffs(empty) - 1;
      empty &= empty - 1;
#pragma unroll
      for (int k = 0; k < NV; ++k) {
        const int c = lane + k * 32;
        if (c < f4) ST(out + (pd0 + r) * out_ld4 + c, make_float4(0.f, 0.f, 0.f, 0.f));
      }
    }
    p_phase = has_self ? 1 : 2;
    return true;
  };
  int64_t produced = 0, consumed = 0;
  bool more = load_window();

  auto produce = [&]() -> bool {
    while (more && p_phase == 2 && p_eb >= p_end) {
      pw += G;
      more = load_window();
    }
    if (!more) return false;
    const bool was_self = p_phase == 1;
    const int st = static_cast<int>(produced % stages);
    uint64_t* bar = bars + st;
    unsigned char* sl = slots + (size_t)st * stage_bytes;
    int cnt;
    int32_t g = 0;
    int2 m = make_int2(0, 0);
    if (was_self) {
      cnt = p_nr;
      g = p_node;
      p_phase = 2;
    } else {
      const int32_t e = p_eb + lane;
      cnt = min(kRows, p_end - p_eb);
      int r = 0;
#pragma unroll
      for (int step = kRows / 2; step >= 1; step >>= 1) {
        const int32_t s = __shfl_sync(0xffffffffu, p_start, (r + step) & 31);
        if (r + step < p_nr && s <= e) r += step;
      }
      const int32_t rs = __shfl_sync(0xffffffffu, p_start, r);
      const int32_t rn = __shfl_sync(0xffffffffu, p_start, (r + 1) & 31);
      const int32_t re = r + 1 < p_nr ? rn : p_end;
      if (lane < cnt) {
        const int32_t li = __ldg(idx + e);
        g = gid ? __ldg(gid + e) : __ldg(map + li);
        const int first =
            has_self ? static_cast<int>((__ldg(new_mask + (e >> 5)) >> (e & 31)) & 1u) : 0;
        m = make_int2(li, ((re - rs) << 8) | (first << 7) | ((e + 1 == re) << 6) | r);
      }
      p_eb += kRows;
    }
    if (lane < cnt) smeta[st * kRows + lane] = m;
    if (lane == 0) {
      hdr[st].d0 = pd0;
      hdr[st].cnt = cnt;
      hdr[st].self = was_self ? 1 : 0;
    }
    // rows of group q = lanes 4q..4q+3 (a short last group repeats its first row)
    const int ngroups = (cnt + 3) >> 2;
    int32_t rows[4];
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      const int src = 4 * (lane & 7) + t;
      const int32_t v = __shfl_sync(0xffffffffu, g, src & 31);
      const int32_t v0 = __shfl_sync(0xffffffffu, g, (4 * (lane & 7)) & 31);
      rows[t] = src < cnt ? v : v0;
    }
    __syncwarp();
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    if (lane == 0) mbar_arrive_expect_tx(bar, static_cast<uint32_t>(ngroups) * 4u * rb);
    __syncwarp();
    if (lane < ngroups)
      gather4(sl + (size_t)lane * gb, &xmap, rows[0], rows[1], rows[2], rows[3], bar, pol_keep);
    ++produced;
    return true;
  };

  float4 acc[NV];
#pragma unroll
  for (int k = 0; k < NV; ++k) acc[k] = make_float4(0.f, 0.f, 0.f, 0.f);
  for (;;) {
    while (produced - consumed < stages && produce()) {
    }
    if (consumed == produced) break;
    const int st = static_cast<int>(consumed % stages);
    mbar_wait(bars + st, static_cast<uint32_t>((consumed / stages) & 1));
    const BatchHdr h = hdr[st];
    const float4* sl = reinterpret_cast<const float4*>(slots + (size_t)st * stage_bytes);
    if (h.self) {
      for (int j = 0; j < h.cnt; ++j) {
        const float4* row = sl + (j >> 2) * gb4 + (j & 3) * rb4;
#pragma unroll
        for (int k = 0; k < NV; ++k) {
          const int c = lane + k * 32;
          if (c < f4) ST(x_in + (h.d0 + j) * x_in_ld4 + c, row[c]);
        }
      }
    } else {
      for (int j = 0; j < h.cnt; ++j) {
        const int2 m = smeta[st * kRows + j];
        const float4* row = sl + (j >> 2) * gb4 + (j & 3) * rb4;
#pragma unroll
        for (int k = 0; k < NV; ++k) {
          const int c = lane + k * 32;
          const float4 v = c < f4 ? row[c] : make_float4(0.f, 0.f, 0.f, 0.f);
          add4(acc[k], v);
          if ((m.y & 0x80) && c < f4) ST(x_in + (int64_t)m.x * x_in_ld4 + c, v);
        }
        if (m.y & 0x40) {  // last edge of dst row d0 + r: H = acc / deg, acc = 0
          const float fd = static_cast<float>(m.y >> 8);
          const int64_t d = h.d0 + (m.y & 0x3f);
#pragma unroll
          for (int k = 0; k < NV; ++k) {
            const int c = lane + k * 32;
            float4 o;
            o.x = __fdiv_rn(acc[k].x, fd);
            o.y = __fdiv_rn(acc[k].y, fd);
            o.z = __fdiv_rn(acc[k].z, fd);
            o.w = __fdiv_rn(acc[k].w, fd);
            if (c < f4) ST(out + d * out_ld4 + c, o);
            acc[k] = make_float4(0.f, 0.f, 0.f, 0.f);
          }
        }
      }
    }
    __syncwarp();
    ++consumed;
  }
}

}  // namespace cmb
