// sample_dev.cuh -- per-row helpers of a2 (biased fanout sampling).
//
// PAPER.md S4.2 P:683-691, S5 P:717: intra-community edges get unnormalised weight p,
// inter-community edges 1-p, and DGL's NeighborSampler draws `fanout` neighbours per node
// WITHOUT replacement (reading R1).  With two weight classes that law factorises exactly:
// the class sequence of successive draws is an urn (P(intra) = wi*ri / (wi*ri + wo*ro)),
// and given K intra picks the intra (inter) subset is uniform -> Floyd's subset sampler.
// So a row costs O(f) Philox draws whatever its degree.
#pragma once

#include "common.cuh"

#ifndef CMB_REC_EVICT_FIRST
#define CMB_REC_EVICT_FIRST 1  // the row-record loads L2 evict_first (50.8 vs 51.5 us per batch)
#endif

namespace cmb {
namespace smp {

constexpr uint32_t kEmpty = 0xFFFFFFFFu;

// A row split into its intra-community segment [lo, hi) and the rest (a0 bounds), with the
// eligible sizes under the Knob-2 weights (a zero-weight class is ineligible, reading R3).
struct RowInfo {
  int64_t rs, deg, ni_e, no_e;
  uint32_t lo, hi;
};

__device__ __forceinline__ RowInfo row_info(const DevGraph& g, int32_t v, uint32_t wi,
                                            uint32_t wo) {
  RowInfo r;
  uint32_t df = kRecDegSlow;
  if (g.rec) {  // one 16-byte load (graph.cu k_intra_bounds packs it)
#if CMB_REC_EVICT_FIRST  // read once per hop and row: do not displace the dedup maps
    uint4 q;
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    asm volatile("ld.global.nc.L2::cache_hint.v4.u32 {%0, %1, %2, %3}, [%4], %5;"
                 : "=r"(q.x), "=r"(q.y), "=r"(q.z), "=r"(q.w)
                 : "l"(g.rec + v), "l"(pol));
#else
    const uint4 q = __ldg(g.rec + v);
#endif
    df = q.y >> 8;
    r.rs = static_cast<int64_t>(q.x) | (static_cast<int64_t>(q.y & 0xFFu) << 32);
    r.deg = df;
    r.lo = q.z;
    r.hi = q.w;
  }
  if (df == kRecDegSlow) {  // no record, or a row too long for its degree field
    r.rs = __ldg(g.indptr + v);
    r.deg = __ldg(g.indptr + v + 1) - r.rs;
    const uint2 b = __ldg(g.bounds + v);
    r.lo = b.x;
    r.hi = b.y;
  }
  const int64_t ni = static_cast<int64_t>(r.hi) - r.lo;
  r.ni_e = wi ? ni : 0;
  r.no_e = wo ? r.deg - ni : 0;
  return r;
}

// the same for an id that may be out of [0, N) (a caller's root): such a row has no neighbours
// (the root insertion raised CMB_ERR_INVALID_INPUT)
__device__ __forceinline__ RowInfo row_info_checked(const DevGraph& g, int32_t v, uint32_t wi,
                                                    uint32_t wo) {
  if (static_cast<uint32_t>(v) >= static_cast<uint64_t>(g.n)) return RowInfo{0, 0, 0, 0, 0u, 0u};
  return row_info(g, v, wi, wo);
}

}  // namespace smp
}  // namespace cmb
