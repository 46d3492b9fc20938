// gather_async.cuh -- the cp.async (LDGSTS) ring form of the fused a4 + a5 kernel (included by
// features.cu; arithmetic as in the comment of k_gather_mean_pipe).
//
// One warp per dst row at a time (grid stride over rows), lane c owning float4 column c
// (f4 <= 32).  A row is a sequence of ITEMS: its self row X[nodes[d]] then its deg edge rows
// X[src] in CSR order.  Every item is one 16-B cp.async per lane into a per-warp ring of KS
// shared-memory slots, so KS feature rows per warp are in flight without holding registers
// (the register-pipelined form keeps <= 3 rows per 16-lane group in flight and waits once per
// 2 edges).  The consumer side waits for the oldest item (cp.async.wait_group KS-1), folds it
// (self -> X_in[d]; edge -> acc += row, X_in store at a first occurrence; last item of the row
// -> H[d] = acc / deg), and refills the slot with the item KS ahead.  Each lane reads back only
// the bytes it copied itself; the per-slot item descriptor (warp-uniform) goes through shared
// memory, written by lane 0.  The index chain (indptr -> edge ids) runs two rows ahead of the
// issue side in registers, as in the pipelined form.
#pragma once

namespace cmb {
namespace asyncg {

constexpr int kWarps = 8;  // warps per block
constexpr int kSelf = 1, kFirst = 2, kLast = 4, kEnd = 8;

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, uint64_t pol) {
  const uint32_t s = static_cast<uint32_t>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.cg.shared.global.L2::cache_hint [%0], [%1], 16, %2;" ::"r"(s),
               "l"(gmem), "l"(pol)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() {
  asm volatile("cp.async.commit_group;" ::: "memory");
}
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

inline size_t smem_bytes(int ks, int f4) {
  return static_cast<size_t>(kWarps) * ks * (static_cast<size_t>(f4) * 16 + sizeof(int4));
}

}  // namespace asyncg

template <int KS>
__global__ void __launch_bounds__(asyncg::kWarps * 32)
    k_gather_mean_async(const int32_t* __restrict__ indptr, const int32_t* __restrict__ idx,
                        const int32_t* __restrict__ gid, const int64_t* __restrict__ n_dst_dev,
                        int64_t n_dst_cap, const float4* __restrict__ src, int64_t src_ld4,
                        const int32_t* __restrict__ map, int f4, float4* __restrict__ out,
                        int64_t out_ld4, float4* __restrict__ x_in, int64_t x_in_ld4,
                        const uint32_t* __restrict__ new_mask) {
  using namespace asyncg;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int lane = threadIdx.x & 31;
  const int wib = threadIdx.x >> 5;
  float4* ring = reinterpret_cast<float4*>(smem_raw) + static_cast<size_t>(wib) * KS * f4;
  int4* meta = reinterpret_cast<int4*>(reinterpret_cast<float4*>(smem_raw) +
                                       static_cast<size_t>(kWarps) * KS * f4) +
               wib * KS;
  const uint64_t pol_keep = policy_evict_last(), pol_stream = policy_evict_first();
  const int64_t n_dst = min(*n_dst_dev, n_dst_cap);
  const int64_t W = static_cast<int64_t>(gridDim.x) * kWarps;
  const bool col = lane < f4;

  struct A { int32_t e0, e1, self; };
  struct B { int32_t g, l, first; };
  auto loadA = [&](int64_t row) {
    A a{0, 0, 0};
    if (row < n_dst) {
      a.e0 = __ldg(indptr + row);
      a.e1 = __ldg(indptr + row + 1);
      a.self = __ldg(map + row);
    }
    return a;
  };
  auto loadB = [&](const A& a) {  // lane j <-> edge e0 + j (deg <= 32 on sampled blocks)
    B b{0, 0, 0};
    const int32_t e = a.e0 + lane;
    if (e < a.e1) {
      b.l = __ldg(idx + e);
      b.g = gid ? __ldg(gid + e) : __ldg(map + b.l);
      b.first = static_cast<int>((__ldg(new_mask + (e >> 5)) >> (e & 31)) & 1u);
    }
    return b;
  };

  // issue side: row ir, item ip (0 = self, 1..deg = edges)
  int64_t ir = blockIdx.x * static_cast<int64_t>(kWarps) + wib;
  A ca = loadA(ir), na = loadA(ir + W), nna = loadA(ir + 2 * W);
  B cb = loadB(ca), nb = loadB(na);
  int ip = 0;
  auto issue = [&](int slot) {
    if (ir < n_dst) {
      const int deg = ca.e1 - ca.e0;
      int32_t g;
      int4 m;
      if (ip == 0) {
        g = ca.self;
        m = make_int4(static_cast<int>(ir), kSelf | (deg == 0 ? kLast : 0), deg, 0);
      } else {
        const int j = ip - 1;
        g = __shfl_sync(0xffffffffu, cb.g, j);
        const int l = __shfl_sync(0xffffffffu, cb.l, j);
        const int fst = __shfl_sync(0xffffffffu, cb.first, j);
        m = make_int4(static_cast<int>(ir), (fst ? kFirst : 0) | (j == deg - 1 ? kLast : 0), deg,
                      l);
      }
      if (col) cp_async16(ring + slot * f4 + lane, src + static_cast<int64_t>(g) * src_ld4 + lane,
                          pol_keep);
      if (lane == 0) meta[slot] = m;
      if (++ip > deg) {  // next row: rotate the index pipeline
        ip = 0;
        ir += W;
        ca = na;
        cb = nb;
        na = nna;
        nb = loadB(na);
        nna = loadA(ir + 2 * W);
      }
    } else if (lane == 0) {
      meta[slot] = make_int4(0, kEnd, 0, 0);
    }
    cp_async_commit();
  };

#pragma unroll 1
  for (int s = 0; s < KS; ++s) issue(s);
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
  int cs = 0;
#pragma unroll 1
  for (;;) {
    cp_async_wait<KS - 1>();
    __syncwarp();
    const int4 m = meta[cs];
    if (m.y & kEnd) break;
    float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
    if (col) v = ring[cs * f4 + lane];
    const int64_t row = m.x;
    if (m.y & kSelf) {
      acc = make_float4(0.f, 0.f, 0.f, 0.f);
      if (x_in && col) st4_hint(x_in + row * x_in_ld4 + lane, v, pol_stream);
    } else {
      add4(acc, v);
      if (x_in && (m.y & kFirst) && col)
        st4_hint(x_in + static_cast<int64_t>(m.w) * x_in_ld4 + lane, v, pol_stream);
    }
    if ((m.y & kLast) && col) {
      float4 h = make_float4(0.f, 0.f, 0.f, 0.f);
      if (m.z > 0) {
        const float fd = static_cast<float>(m.z);
        h.x = __fdiv_rn(acc.x, fd);
        h.y = __fdiv_rn(acc.y, fd);
        h.z = __fdiv_rn(acc.z, fd);
        h.w = __fdiv_rn(acc.w, fd);
      }
      st4_hint(out + row * out_ld4 + lane, h, pol_stream);
    }
    __syncwarp();  // every lane has read meta[cs] before lane 0 rewrites it
    issue(cs);
    cs = cs + 1 == KS ? 0 : cs + 1;
  }
  cp_async_wait<0>();
}

}  // namespace cmb
