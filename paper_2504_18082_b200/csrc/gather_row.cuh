// gather_row.cuh -- the warp-per-row form of the fused a4 + a5 kernel (included by
// features.cu; arithmetic as in the comment of k_gather_mean_pipe).
//
// One warp per dst row (grid stride), lane c owning float4 column c of each 32-float4 chunk.  The edge ids of
// the row are held lane-parallel (lane j <-> edge j; a sampled block has deg <= 32) and were
// loaded one row ahead; the self row and up to DMAX edge rows are then issued back to back, so a
// row costs ONE memory round trip for deg <= DMAX (the 16-lane pipelined form needs
// ceil(deg / 2) + 1).  The sum runs in CSR order from +0 (the oracle's order); H = acc / deg
// uses the correctly rounded reciprocal y = RN(1/deg), computed once per row, and one FMA
// correction per element (q = RN(a*y), r = a - deg*q exact, RN(q + r*y) = RN(a/deg) -- the
// classical FMA division step), with __fdiv_rn kept for |a| outside [2^-100, 2^100] where the
// step's no-underflow / no-overflow premise could fail.  Warp-uniform control flow throughout
// (full-mask shuffles only).
#pragma once

namespace cmb {

__device__ __forceinline__ float div_small(float a, float d, float y) {
  const float aa = fabsf(a);
  if (!(aa >= 0x1p-100f && aa <= 0x1p100f)) return a == 0.f ? a / d : __fdiv_rn(a, d);
  const float q = __fmul_rn(a, y);
  const float r = __fmaf_rn(-d, q, a);
  return __fmaf_rn(r, y, q);
}

// Where feature row v lives.  DenseRows: one table in this GPU's HBM.  ShardedRows
// (NEXT-1): rows [r*S, (r+1)*S) in shard r, base[r] being this GPU's own shard or a peer's
// shard mapped into this process (CUDA IPC over NVLink), so the loads of remote rows travel
// over NVLink inside the kernel -- no staging copy, no separate collective.
struct DenseRows {
  const float4* base;
  uint32_t ld4;  // row stride in float4 (one IMAD.WIDE.U32 per row address)
  __device__ __forceinline__ const float4* row(int32_t v) const {
    return base + static_cast<uint64_t>(static_cast<uint32_t>(v)) * ld4;
  }
};
constexpr int kMaxShards = 8;
struct ShardedRows {
  const float4* base[kMaxShards];
  uint32_t ld4;
  uint64_t inv;  // ceil(2^32 / rows_per_shard): owner = (v * inv) >> 32, at most 1 too high
  uint32_t rows_per_shard;
  __device__ __forceinline__ const float4* row(int32_t v) const {
    const uint32_t u = static_cast<uint32_t>(v);
    uint32_t r = static_cast<uint32_t>((static_cast<uint64_t>(u) * inv) >> 32);
    if (static_cast<uint64_t>(r) * rows_per_shard > u) --r;
    return base[r] + static_cast<uint64_t>(u - r * rows_per_shard) * ld4;
  }
};

// The a4 + a5 operands of up to kMaxGatherBatches independent batches, walked as ONE sequence of
// dst rows (one launch per launch group instead of one per batch: no launch gap and no tail
// between the batches).  Batch j's rows are slots [pre_j, pre_{j+1}) of the walk, pre from the
// device counts n_dst_dev[j] (capped at n_dst_cap[j]).
constexpr int kMaxGatherBatches = CMB_MAX_BATCHES_PER_LAUNCH;
struct GatherSet {
  int nb;
  const int32_t* indptr[kMaxGatherBatches];  // hop L-1 block: [n_dst + 1]
  const int32_t* idx[kMaxGatherBatches];     // local src id per edge
  const int32_t* gid[kMaxGatherBatches];     // global src id per edge
  const int64_t* n_dst_dev[kMaxGatherBatches];
  int64_t n_dst_cap[kMaxGatherBatches];
  const int32_t* map[kMaxGatherBatches];     // nodes: row id of dst node d
  const uint32_t* mask[kMaxGatherBatches];   // first-occurrence bits per edge
  const int32_t* order[kMaxGatherBatches];   // visiting order of the dst rows, or NULL
  float4* out[kMaxGatherBatches];            // H
  int64_t out_ld4[kMaxGatherBatches];
  float4* x_in[kMaxGatherBatches];           // X_in
  int64_t x_in_ld4[kMaxGatherBatches];
};

template <int DMAX, int MINB, bool WIDE, class Rows>
__global__ void __launch_bounds__(256, MINB)
    k_gather_mean_row(const __grid_constant__ GatherSet S, const __grid_constant__ Rows rows,
                      int f4) {
  constexpr unsigned kFull = 0xffffffffu;
  const uint64_t pol_keep = policy_rows(), pol_stream = policy_evict_first();
  __shared__ int32_t pre[kMaxGatherBatches + 1];
  if (threadIdx.x == 0) {
    int32_t t = 0;
    pre[0] = 0;
    for (int j = 0; j < kMaxGatherBatches; ++j) {
      if (j < S.nb) t += static_cast<int32_t>(min(*S.n_dst_dev[j], S.n_dst_cap[j]));
      pre[j + 1] = t;
    }
  }
  __syncthreads();
  const int64_t n_dst = pre[kMaxGatherBatches];
  const int lane = threadIdx.x & 31;
  const int64_t W = static_cast<int64_t>(gridDim.x) * (blockDim.x >> 5);
  const float4 zero = make_float4(0.f, 0.f, 0.f, 0.f);

  // slot k of the walk: batch b, dst row d = order_b[k - pre_b] (a permutation of the batch's
  // rows: rows of nearby ids together, so the src rows they share are re-read while still in
  // L2) or k - pre_b
  struct A { int32_t e0, e1, self, d, b; };
  struct B { int32_t g, l, first; };
  auto loadA = [&](int64_t k) {
    A a{0, 0, 0, 0, 0};
    if (k < n_dst) {
      const int32_t kk = static_cast<int32_t>(k);
      int b = 0;
#pragma unroll
      for (int j = 1; j < kMaxGatherBatches; ++j) b += kk >= pre[j];
      const int32_t r = kk - pre[b];
      const int32_t d = S.order[b] ? __ldg(S.order[b] + r) : r;
      a.b = b;
      a.d = d;
      a.e0 = __ldg(S.indptr[b] + d);
      a.e1 = __ldg(S.indptr[b] + d + 1);
      a.self = __ldg(S.map[b] + d);
    }
    return a;
  };
  auto loadB = [&](const A& a) {
    B v{0, 0, 0};
    const int32_t e = a.e0 + lane;
    if (e < a.e1) {
      v.l = __ldg(S.idx[a.b] + e);
      v.g = __ldg(S.gid[a.b] + e);
      v.first = static_cast<int>((__ldg(S.mask[a.b] + (e >> 5)) >> (e & 31)) & 1u);
    }
    return v;
  };

  int64_t row = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  A ac = loadA(row);
  B bc = loadB(ac);
  A an = loadA(row + W);
  for (; row < n_dst; row += W) {
    const A aa = loadA(row + 2 * W);  // index pipeline: A two rows ahead, B one row ahead
    const B bn = loadB(an);
    const int deg = ac.e1 - ac.e0;
    const unsigned firsts = __ballot_sync(kFull, bc.first);
    float4* const x_in = S.x_in[ac.b];
    const int64_t x_in_ld4 = S.x_in_ld4[ac.b];
    // column chunks of 32 float4 (one for F <= 128; wide rows, e.g. F = 602, take several)
    for (int c0 = 0; c0 < (WIDE ? f4 : 1); c0 += 32) {
    const bool col = c0 + lane < f4;
    // every load is unconditional (no select or zeroing after it: a predicated or selected
    // load leaves a register move that waits on its scoreboard and holds the next load's
    // address back, splitting a row's loads over two round trips): lanes past F re-read the
    // row's last float4 (same request), slots past deg re-read the self row (an L2 hit); only
    // the first deg values are summed and only lanes < F/4 store
    const int cl = col ? c0 + lane : f4 - 1;
    const float4 sv = ldg4_hint(rows.row(ac.self) + cl, pol_keep);
    float4 acc = zero;
    for (int base = 0; base < deg; base += DMAX) {
      float4 v[DMAX];
#pragma unroll
      for (int j = 0; j < DMAX; ++j) {
        const int32_t g = __shfl_sync(kFull, bc.g, (base + j) & 31);
        v[j] = ldg4_hint(rows.row(base + j < deg ? g : ac.self) + cl, pol_keep);
      }
#pragma unroll
      for (int j = 0; j < DMAX; ++j) {
        if (base + j < deg) {
          add4(acc, v[j]);
          if ((firsts >> (base + j)) & 1u) {  // first occurrence of a new src node
            const int32_t l = __shfl_sync(kFull, bc.l, base + j);
            if (col)
              st4_hint(x_in + static_cast<int64_t>(l) * x_in_ld4 + c0 + lane, v[j], pol_stream);
          }
        }
      }
    }
    if (col) {
      float4 h = zero;
      if (deg > 0) {
        const float d = static_cast<float>(deg);
        const float y = __frcp_rn(d);
        h.x = div_small(acc.x, d, y);
        h.y = div_small(acc.y, d, y);
        h.z = div_small(acc.z, d, y);
        h.w = div_small(acc.w, d, y);
      }
      st4_hint(S.out[ac.b] + static_cast<int64_t>(ac.d) * S.out_ld4[ac.b] + c0 + lane, h,
               pol_stream);
      st4_hint(x_in + static_cast<int64_t>(ac.d) * x_in_ld4 + c0 + lane, sv, pol_stream);
    }
    }
    ac = an;
    bc = bn;
    an = aa;
  }
}

}  // namespace cmb
