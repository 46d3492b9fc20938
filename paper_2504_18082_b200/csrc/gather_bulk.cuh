// gather_bulk.cuh -- the TMA bulk-copy form of the fused a4 + a5 kernel (included by
// features.cu; see the comment there for the arithmetic).
//
// Work decomposition: a warp walks windows of 32 consecutive dst rows (grid stride over
// windows).  A window becomes a sequence of BATCHES of at most 32 feature rows:
//   * one SELF batch (the window's own rows X[nodes[d]] -> X_in[d], a4 for dst rows), and
//   * EDGE batches: the window's edges [indptr[d0], indptr[d0+32]) in chunks of 32.
// Producer side (the same warp, running up to kStages batches ahead): the batch's index
// streams are read coalesced (lane k <-> edge k), every lane resolves its edge's dst row
// (binary search over the window's row starts held in lanes), whether it closes that row
// and whether it is the first occurrence of a new src node; lane 0 arms the stage's mbarrier
// with the batch's byte count and every lane issues one cp.async.bulk (TMA, SASS UBLKCP)
// global -> shared for its row.  Consumer side: wait on the stage's mbarrier, then fold the
// 32 rows from shared memory in edge (= CSR) order -- acc += row, X_in store on first
// occurrence, H = acc / deg (IEEE) on the last edge of a row -- exactly the oracle's fp32
// order.  kStages x 32 rows (x 400 B for F = 100: 51 KB) are in flight per warp without any
// register cost, which is what random 400-byte rows need (Little's law at ~6.5 TB/s).
#pragma once

namespace cmb {
namespace bulk {

constexpr int kWarps = 4;   // warps per block
constexpr int kStages = 4;  // batches in flight per warp
constexpr int kRows = 32;   // rows per batch

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
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes,
                                         uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
          "r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

struct BatchHdr {
  int64_t d0;   // first dst row of the window
  int32_t cnt;  // rows in the batch
  int32_t self; // 1 = SELF batch
};

constexpr size_t smem_bytes(uint32_t rb) {
  return (size_t)kWarps * kStages * kRows * rb +                 // row slots
         (size_t)kWarps * kStages * kRows * sizeof(int2) +       // per-slot {li, meta}
         (size_t)kWarps * kStages * sizeof(BatchHdr) +           // per-stage header
         (size_t)kWarps * kStages * sizeof(uint64_t);            // per-stage mbarrier
}

}  // namespace bulk

template <int NV>
__global__ void __launch_bounds__(bulk::kWarps * 32) k_gather_mean_bulk(
    const int32_t* __restrict__ indptr, const int32_t* __restrict__ idx,
    const int32_t* __restrict__ gid, const int64_t* __restrict__ n_dst_dev, int64_t n_dst_cap,
    const float* __restrict__ src, int64_t src_ld, const int32_t* __restrict__ map, int f4,
    uint32_t rb, float4* __restrict__ out, int64_t out_ld4, float4* __restrict__ x_in,
    int64_t x_in_ld4, const uint32_t* __restrict__ new_mask) {
  using namespace bulk;
  extern __shared__ __align__(128) unsigned char smem[];
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  unsigned char* slots = smem + (size_t)warp * kStages * kRows * rb;
  unsigned char* tail = smem + (size_t)kWarps * kStages * kRows * rb;
  int2* smeta = reinterpret_cast<int2*>(tail) + warp * kStages * kRows;
  BatchHdr* hdr = reinterpret_cast<BatchHdr*>(tail + kWarps * kStages * kRows * sizeof(int2)) +
                  warp * kStages;
  uint64_t* bars = reinterpret_cast<uint64_t*>(tail + kWarps * kStages * kRows * sizeof(int2) +
                                               kWarps * kStages * sizeof(BatchHdr)) +
                   warp * kStages;
  if (lane == 0) {
    for (int i = 0; i < kStages; ++i) mbar_init(bars + i, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncwarp();

  const int64_t n_dst = min(*n_dst_dev, n_dst_cap);
  const int64_t nwin = (n_dst + kRows - 1) / kRows;
  const int64_t G = (int64_t)gridDim.x * kWarps;
  const bool has_self = x_in != nullptr;
  const float4* rows4 = reinterpret_cast<const float4*>(slots);
  const int rb4 = static_cast<int>(rb >> 4);

  // ---------------- producer state (window being issued)
  int64_t pw = (int64_t)blockIdx.x * kWarps + warp;  // window index
  int64_t pd0 = 0;
  int p_nr = 0;
  int32_t p_start = 0, p_end = 0, p_node = 0, p_eb = 0;
  int p_phase = 0;  // 0 = load window, 1 = self batch next, 2 = edge batches
  auto load_window = [&]() -> bool {
    if (pw >= nwin) return false;
    pd0 = pw * kRows;
    p_nr = (n_dst - pd0 < kRows) ? static_cast<int>(n_dst - pd0) : kRows;
    p_start = lane < p_nr ? __ldg(indptr + pd0 + lane) : 0;
    p_end = __ldg(indptr + pd0 + p_nr);
    p_node = (has_self && lane < p_nr) ? __ldg(map + pd0 + lane) : 0;
    p_eb = __shfl_sync(0xffffffffu, p_start, 0);
    // rows without edges: H = 0 now (nothing to fold)
    const int32_t nxt = __shfl_down_sync(0xffffffffu, p_start, 1);
    const int32_t my_end = lane + 1 < p_nr ? nxt : p_end;
    unsigned empty = __ballot_sync(0xffffffffu, lane < p_nr && my_end == p_start);
    while (empty) {
      const int r = __ffs(empty) - 1;
      empty &= empty - 1;
#pragma unroll
      for (int k = 0; k < NV; ++k) {
        const int c = lane + k * 32;
        if (c < f4) out[(pd0 + r) * out_ld4 + c] = make_float4(0.f, 0.f, 0.f, 0.f);
      }
    }
    p_phase = has_self ? 1 : 2;
    return true;
  };
  int64_t produced = 0, consumed = 0;
  bool more = load_window();

  // issue the next batch into stage produced % kStages; false when no batch is left
  auto produce = [&](bool& was_self) -> bool {
    while (more && p_phase == 2 && p_eb >= p_end) {  // window done: next window
      pw += G;
      more = load_window();
    }
    if (!more) return false;
    was_self = p_phase == 1;
    const int st = static_cast<int>(produced % kStages);
    uint64_t* bar = bars + st;
    unsigned char* sl = slots + (size_t)st * kRows * rb;
    int cnt;
    int32_t g = 0;
    int2 m = make_int2(0, 0);
    if (p_phase == 1) {  // SELF batch
      cnt = p_nr;
      g = p_node;
      p_phase = 2;
    } else {             // EDGE batch
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
    __syncwarp();
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    if (lane == 0) mbar_arrive_expect_tx(bar, static_cast<uint32_t>(cnt) * rb);
    __syncwarp();
    if (lane < cnt) bulk_g2s(sl + (size_t)lane * rb, src + (int64_t)g * src_ld, rb, bar);
    ++produced;
    return true;
  };

  float4 acc[NV];
#pragma unroll
  for (int k = 0; k < NV; ++k) acc[k] = make_float4(0.f, 0.f, 0.f, 0.f);
  for (;;) {
    bool was_self = false;
    while (produced - consumed < kStages && produce(was_self)) {
    }
    if (consumed == produced) break;
    const int st = static_cast<int>(consumed % kStages);
    mbar_wait(bars + st, static_cast<uint32_t>((consumed / kStages) & 1));
    const BatchHdr h = hdr[st];
    const float4* sl = rows4 + (size_t)st * kRows * rb4;
    if (h.self) {
      for (int j = 0; j < h.cnt; ++j) {
#pragma unroll
        for (int k = 0; k < NV; ++k) {
          const int c = lane + k * 32;
          if (c < f4) x_in[(h.d0 + j) * x_in_ld4 + c] = sl[j * rb4 + c];
        }
      }
    } else {
      for (int j = 0; j < h.cnt; ++j) {
        const int2 m = smeta[st * kRows + j];
#pragma unroll
        for (int k = 0; k < NV; ++k) {
          const int c = lane + k * 32;
          const float4 v = c < f4 ? sl[j * rb4 + c] : make_float4(0.f, 0.f, 0.f, 0.f);
          add4(acc[k], v);
          if ((m.y & 0x80) && c < f4) x_in[(int64_t)m.x * x_in_ld4 + c] = v;
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
            if (c < f4) out[d * out_ld4 + c] = o;
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
