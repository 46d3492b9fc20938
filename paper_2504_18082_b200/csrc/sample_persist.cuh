// sample_persist.cuh -- the persistent cooperative schedule of a2 + a3 (included by sample.cu).
//
// One launch per batch, one block per SM (cooperative launch: all blocks co-resident), grid
// barriers between the phases of a hop.  Dedup uses a DIRECT map over node ids (one word per
// node in the workspace) instead of a hash table.  An entry is tag | value, the tag being a
// per-workspace batch counter in the word's top bits, so entries written by earlier batches
// read as empty and the map is never cleared between batches:
//     value = kFinal | id          node u has local id `id` (dst nodes, relabelled nodes)
//           = kMarkerTop - e       e = smallest edge position seen so far for new node u
// "First occurrence" is then ONE fire-and-forget atomicMax per edge (skipped when the entry
// already holds a winning value): a newer tag beats a stale entry, final ids beat markers,
// smaller e beats larger e.
// Map words (MapWord<W>): 32-bit (7-bit tag, 24-bit values: every id and edge position of the
// batch below 2^24 -- the BASELINE configs need <= 1.1M) whenever the batch's capacities allow,
// else 64-bit (32-bit tag, 31-bit values).  The 32-bit tag wraps after 127 batches: the batch
// that takes tag 1 clears the map first (one extra grid barrier every 127 batches).  Half the
// bytes per entry halves the map's footprint (9.8 instead of 19.6 MB per workspace on products),
// so the four maps of a launch group stay L2-resident across the gathers between two launches.
//
// Phases of hop h:
//  A  [relabel(h-1)] + count + prefix + positions/picks/marks
//     block b owns dst rows [b*R, (b+1)*R): row info cached in shared memory; counts; block scan;
//     single-pass cross-block prefix (publish own total, add the totals of blocks < b);
//     positions: the urn + Floyd draws of each row (one thread per row for f <= 16, G-lane
//     groups otherwise); each pick loads indices[pos] right away and marks its first occurrence
//     with atomicMax(map[u], tag | kMarkerTop - e)
//  C  flag + prefix + assign: first occurrences (map[u] == tag | kMarkerTop - e) get
//     id = n_h + global flag scan - 1: map[u] := tag | kFinal | id, nodes[id] := u.  With 32-bit
//     words the assign step also writes every edge's local id (own id, an earlier hop's id, or
//     the id of the node's first occurrence via the published block bases); with 64-bit words
//     the relabel indices[e] := id(map[u]) runs after the barrier, fused into hop h+1's A.
#pragma once

namespace cmb {
namespace pst {

using namespace smp;

constexpr int kMaxBlocks = 4096;
#ifndef CMB_ROW_CAP  // layout experiments only (tools/gpu_variant_ab.sh)
#define CMB_ROW_CAP 3072
#endif
constexpr int kRowCap = CMB_ROW_CAP;  // dst rows per block cached in shared memory
#ifndef CMB_ORDER_BITS  // layout experiments only
#define CMB_ORDER_BITS 12
#endif
constexpr int kOrderBits = CMB_ORDER_BITS;     // dst-order buckets: at most 2^12 node-id ranges
constexpr int kOrderBuckets = 1 << kOrderBits;

// the two map word layouts: tag in the top bits, then the final flag, then the value
template <class W>
struct MapWord;
template <>
struct MapWord<uint32_t> {
  using T = unsigned;
  static constexpr int kShift = 25;
  static constexpr unsigned kFinal = 1u << 24;
  static constexpr unsigned kMarkerTop = (1u << 24) - 1u;
  static constexpr unsigned kVal = (1u << 24) - 1u;
  static constexpr unsigned kTagMax = 127u;  // tags 1..127, then clear + wrap
};
template <>
struct MapWord<uint64_t> {
  using T = unsigned long long;
  static constexpr int kShift = 32;
  static constexpr unsigned long long kFinal = 0x80000000ull;
  static constexpr unsigned long long kMarkerTop = 0x7FFFFFFFull;
  static constexpr unsigned long long kVal = 0x7FFFFFFFull;
  static constexpr unsigned kTagMax = 0xFFFFFFFFu;  // never wraps in practice
};

// Accesses to the tagged dedup map are marked L2 evict_last: the maps of a launch group's
// workspaces (4 x 19.6 MB on products) then survive the gathers that stream ~2.4 GB through L2
// between two sampler launches, and a batch's first touches of map entries hit L2 instead of
// DRAM (sampler 81.0 -> 76.6 us per batch, gather 108.9 -> 109.4: 190.7 -> 186.9 us per step;
// evict_normal feature loads in the gather instead: 188.0).
__device__ __forceinline__ uint64_t map_pol() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ unsigned long long map_ld(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.global.cg.L2::cache_hint.u64 %0, [%1], %2;" : "=l"(v) : "l"(p), "l"(map_pol()));
  return v;
}
__device__ __forceinline__ unsigned map_ld(const unsigned* p) {
  unsigned v;
  asm volatile("ld.global.cg.L2::cache_hint.u32 %0, [%1], %2;" : "=r"(v) : "l"(p), "l"(map_pol()));
  return v;
}
__device__ __forceinline__ void map_st(unsigned long long* p, unsigned long long v) {
  asm volatile("st.global.L2::cache_hint.u64 [%0], %1, %2;" ::"l"(p), "l"(v), "l"(map_pol())
               : "memory");
}
__device__ __forceinline__ void map_st(unsigned* p, unsigned v) {
  asm volatile("st.global.L2::cache_hint.u32 [%0], %1, %2;" ::"l"(p), "r"(v), "l"(map_pol())
               : "memory");
}
// atomicMax without a result (a reduction), same policy
__device__ __forceinline__ void map_max(unsigned long long* p, unsigned long long v) {
  asm volatile("red.global.max.L2::cache_hint.u64 [%0], %1, %2;" ::"l"(p), "l"(v), "l"(map_pol())
               : "memory");
}
__device__ __forceinline__ void map_max(unsigned* p, unsigned v) {
  asm volatile("red.global.max.L2::cache_hint.u32 [%0], %1, %2;" ::"l"(p), "r"(v), "l"(map_pol())
               : "memory");
}
__device__ __forceinline__ unsigned long long map_exch(unsigned long long* p,
                                                       unsigned long long v) {
  unsigned long long o;
  asm volatile("atom.global.exch.L2::cache_hint.b64 %0, [%1], %2, %3;"
               : "=l"(o)
               : "l"(p), "l"(v), "l"(map_pol())
               : "memory");
  return o;
}
__device__ __forceinline__ unsigned map_exch(unsigned* p, unsigned v) {
  unsigned o;
  asm volatile("atom.global.exch.L2::cache_hint.b32 %0, [%1], %2, %3;"
               : "=r"(o)
               : "l"(p), "r"(v), "l"(map_pol())
               : "memory");
  return o;
}

// The picks' CSR loads (one random sector each, never reused within the batch) are marked L2
// evict_first, so they do not push the concurrently running batches' dedup maps (evict_last)
// out of L2: 54.4 -> 52.8 us per batch (CMB_PICK_EVICT_FIRST = 0 restores plain loads).
#ifndef CMB_PICK_EVICT_FIRST
#define CMB_PICK_EVICT_FIRST 1
#endif
__device__ __forceinline__ int32_t pick_ld(const int32_t* p) {
#if CMB_PICK_EVICT_FIRST
  int32_t v;
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  asm volatile("ld.global.nc.L2::cache_hint.s32 %0, [%1], %2;" : "=r"(v) : "l"(p), "l"(pol));
  return v;
#else
  return __ldg(p);
#endif
}

__device__ __forceinline__ uint64_t globaltimer() {
  uint64_t t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

// Several batches can share one launch: block b works on batch b % nb as virtual block
// b / nb of a virtual grid of the blocks with that residue (its own barrier, prefixes and
// map).  All phase code addresses blocks through vblk() / vgrid().
__shared__ int g_vblk, g_vgrid;
__device__ __forceinline__ int vblk() { return g_vblk; }
__device__ __forceinline__ int vgrid() { return g_vgrid; }

struct PArgs {
  DevGraph g;
  const int32_t* roots;
  int64_t n_roots;
  int L;
  int fan[CMB_MAX_HOPS];
  uint32_t wi, wo, k0, k1, batch;
  int32_t* nodes;
  int32_t* indptr[CMB_MAX_HOPS];
  int32_t* indices[CMB_MAX_HOPS];
  uint32_t* mask;
  int32_t* last_src;
  int64_t* sizes;
  void* map;                // [N] tagged direct dedup map (see above), MapWord<W>::T words
  unsigned* tag_ctr;        // [1] batches sampled with this workspace so far
  uint32_t* scan;           // [max e_cap] flag << 31 | block-local inclusive flag scan
  unsigned long long* pub;  // [3][kMaxBlocks] tagged block aggregates, last-hop block bases
  unsigned* bar;            // [0] arrivals, [1] generation
  uint64_t* prof;           // [kMaxBlocks][64] per-block %globaltimer at sub-step boundaries
  uint32_t* hist;           // [kOrderBuckets] dst rows of hop L-1 per bucket v >> order_shift
  uint32_t* rank;           // [n_cap[L-1]] a last-hop dst row's rank within its order bucket
  int32_t* order;           // optional [n_{L-1}]: the visiting order of the last hop's dst rows
  int order_shift;
  int32_t* status;
  int law;                  // Knob-2 law: 0 = successive weighted w/o replacement, 1 = slot
};

// Per-block sub-step timeline (profiling aid, one store per sub-step per block):
// thread 0 of every block records %globaltimer into prof[block][k], k counting the calls.
#define CMB_PROF(a, k)                                                               \
  do {                                                                               \
    if (threadIdx.x == 0 && (k) < 64)                                                \
      (a).prof[(size_t)vblk() * 64 + (k)] = globaltimer();                       \
    ++(k);                                                                           \
  } while (0)

__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned long long ld_relaxed64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_relaxed64(unsigned long long* p, unsigned long long v) {
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ void st_release64(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_acquire64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

// Generation-counting grid barrier (all blocks co-resident).
__device__ __forceinline__ void grid_barrier(unsigned* bar, unsigned& gen) {
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    const unsigned arrived = atomicAdd(bar, 1u);
    if (arrived == vgrid() - 1) {
      bar[0] = 0u;
      __threadfence();
      atomicAdd(bar + 1, 1u);
    } else {
      while (ld_acquire(bar + 1) == gen) {
      }
    }
    gen += 1u;
  }
  __syncthreads();
}

struct RowCache {
  int64_t rs[kRowCap];
  uint32_t deg[kRowCap];
  uint32_t lo[kRowCap];
  uint32_t hi[kRowCap];
  int32_t v[kRowCap];
  int32_t off[kRowCap];
};

template <int PB>
struct Smem {
  union {
    typename cub::BlockScan<int32_t, PB>::TempStorage scan;
    typename cub::BlockReduce<int32_t, PB>::TempStorage reduce;
  } cub;
  int32_t bc;
  int32_t next;  // positions step: the next unclaimed row chunk of the block
  RowCache rows;
};

// The tag of a published aggregate: this batch's map tag and the hop, so entries left by earlier
// batches or hops never match and the array needs no clearing between batches.
__device__ __forceinline__ unsigned pub_tag(unsigned ctr, int h) {
  return (ctr << 4) | static_cast<unsigned>(h + 1);
}

// Block b publishes its aggregate (tagged) and adds the aggregates of blocks [0, b) as they
// appear.  Every block publishes before it waits -> the wait always ends.  Only the numbers
// are exchanged, so relaxed accesses suffice.
template <int PB>
__device__ __forceinline__ int32_t publish_and_prefix(unsigned long long* pub, unsigned tag,
                                                      int32_t agg, Smem<PB>& sm) {
  if (threadIdx.x == 0)
    st_relaxed64(pub + vblk(), (static_cast<unsigned long long>(tag) << 32) |
                                       static_cast<uint32_t>(agg));
  int32_t s = 0;
  for (int j = threadIdx.x; j < (int)vblk(); j += PB) {
    unsigned long long v;
    while (((v = ld_relaxed64(pub + j)) >> 32) != tag) {
    }
    s += static_cast<int32_t>(v & 0xffffffffu);
  }
  const int32_t tot = cub::BlockReduce<int32_t, PB>(sm.cub.reduce).Sum(s);
  if (threadIdx.x == 0) sm.bc = tot;
  __syncthreads();
  const int32_t r = sm.bc;
  __syncthreads();
  return r;
}

__device__ __forceinline__ void range_of(int64_t n, int64_t align, int64_t& lo, int64_t& hi) {
  int64_t per = (n + vgrid() - 1) / vgrid();
  per = (per + align - 1) / align * align;
  lo = (int64_t)vblk() * per;
  if (lo > n) lo = n;
  hi = lo + per;
  if (hi > n) hi = n;
}

// relabel of hop h (all entries final): indices[e] := local id of its node
template <int PB, class W>
__device__ void phase_relabel(const PArgs& a, int h) {
  using M = MapWord<W>;
  using T = typename M::T;
  const T* map = static_cast<const T*>(a.map);
  const int64_t e_h = __ldcg(a.sizes + a.L + 1 + h);
  int32_t* gid = (h == a.L - 1) ? a.last_src : nullptr;
  int32_t* ind = a.indices[h];
  const int64_t stride = (int64_t)vgrid() * PB;
  for (int64_t e0 = vblk() * (int64_t)PB + threadIdx.x; e0 < e_h; e0 += 4 * stride) {
    int32_t u[4];
    T v[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) u[k] = e0 + k * stride < e_h ? __ldcg(ind + e0 + k * stride) : 0;
#pragma unroll
    for (int k = 0; k < 4; ++k) v[k] = e0 + k * stride < e_h ? map_ld(map + u[k]) : T(0);
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int64_t e = e0 + k * stride;
      if (e < e_h) {
        if (gid) gid[e] = u[k];
        ind[e] = static_cast<int32_t>(v[k] & M::kVal);
      }
    }
  }
}

// ---- the picks of one row: rank k (ascending position) at absolute CSR index p
// PickEmit: load the neighbour id right away, write it to the block and mark its first
// occurrence -- atomicMax(map[u], tag | kMarkerTop - e), a fire-and-forget reduction; final
// entries (roots, earlier hops) always beat markers, smaller e beats larger e.  The random CSR
// loads then overlap with the Philox work of the other rows of the phase instead of forming a
// pass of their own.  (Tried and removed: a separate coalesced picks pass through a pick-position
// array, 91 vs 84 us per batch; warp-deduplicating the marks with match_any, 88 vs 86 us.)
template <class W>
struct PickEmit {
  using M = MapWord<W>;
  using T = typename M::T;
  const int32_t* ind;
  int32_t* out;                // block indices of this row's first pick
  T* map;
  T tag;
  uint32_t e0;                 // absolute edge index of the row's first pick
  // (reading the entry first and skipping the reduction when it already holds a winning value,
  // against hub contention at p = 1, measured no better at MIX-0 / NORAND p = 1 and 1.9 us per
  // batch slower at RAND: removed)
  __device__ __forceinline__ void put(int k, int64_t p) const {
    const uint32_t u = static_cast<uint32_t>(pick_ld(ind + p));
    out[k] = static_cast<int32_t>(u);
    map_max(map + u, tag | (M::kMarkerTop - (e0 + static_cast<uint32_t>(k))));
  }
#ifndef CMB_PUT_ROW_MAX
#define CMB_PUT_ROW_MAX 10  // widest slot form whose picks are emitted as one batch (16: spills)
#endif
  // all picks of a row at once (thread-per-row form, FM <= 10): every neighbour load, then the
  // reductions -- one round trip per row instead of one per pick
  template <int FM>
  __device__ __forceinline__ void put_row(int tot, int64_t rs, const uint32_t (&pos)[FM]) const {
    if (tot <= 0) return;
    uint32_t u[FM], rk[FM];
#pragma unroll
    for (int s = 0; s < FM; ++s)
      u[s] = static_cast<uint32_t>(pick_ld(ind + rs + (s < tot ? pos[s] : pos[0])));
#pragma unroll
    for (int s = 0; s < FM; ++s) {
      uint32_t r = 0;
#pragma unroll
      for (int q = 0; q < FM; ++q) r += (q < tot) && pos[q] < pos[s];
      rk[s] = r;
      if (s < tot) out[r] = static_cast<int32_t>(u[s]);
    }
#pragma unroll
    for (int s = 0; s < FM; ++s)
      if (s < tot) map_max(map + u[s], tag | (M::kMarkerTop - (e0 + rk[s])));
  }
};

// take-all (reading R4): every eligible position, ascending; returns true if taken
template <class Emit>
__device__ __forceinline__ bool take_all(int64_t rs, int64_t deg, uint32_t lo, uint32_t hi,
                                         int64_t ni_e, int64_t no_e, int f, int lane, int G,
                                         const Emit& em) {
  if (f < ni_e + no_e) return false;
  if (ni_e && no_e) {
#pragma unroll 4
    for (int64_t q = lane; q < deg; q += G) em.put(static_cast<int>(q), rs + q);
  } else if (ni_e) {
#pragma unroll 4
    for (int64_t q = lane; q < ni_e; q += G) em.put(static_cast<int>(q), rs + lo + q);
  } else {
#pragma unroll 4
    for (int64_t q = lane; q < no_e; q += G)
      em.put(static_cast<int>(q), rs + (q < lo ? q : hi + (q - lo)));
  }
  return true;
}

// slot law (R23): picks of a row with f < m -- K_draw intra slots from the same words the
// positions step draws, then each class clipped (no refill)
__device__ __forceinline__ int32_t slot_count(int32_t v, int hop, int f, uint32_t wi,
                                              int64_t ni_e, int64_t no_e, uint32_t k0,
                                              uint32_t k1, uint32_t batch) {
  int kd = 0;
  for (int s = 0; s < f; ++s) {
    const PhiloxOut w = philox4x32_10(static_cast<uint32_t>(s), static_cast<uint32_t>(v),
                                      (kTagSample << 24) | static_cast<uint32_t>(hop), batch,
                                      k0, k1);
    kd += (lo64(w) >> 48) < wi;
  }
  const int64_t K = kd < ni_e ? kd : ni_e;
  const int64_t kb = f - kd < no_e ? f - kd : no_e;
  return static_cast<int32_t>(K + kb);
}

// G lanes per row (f <= G): lane s owns Philox slot s
template <int G, class Emit>
__device__ __forceinline__ void row_positions_group(int32_t v, int64_t rs, int64_t deg,
                                                    uint32_t lo, uint32_t hi, int hop, int f,
                                                    uint32_t wi, uint32_t wo, uint32_t k0,
                                                    uint32_t k1, uint32_t batch, int lane,
                                                    unsigned gmask, const Emit& em, int law) {
  const int64_t ni = static_cast<int64_t>(hi) - lo;
  const int64_t ni_e = wi ? ni : 0, no_e = wo ? deg - ni : 0;
  if (take_all(rs, deg, lo, hi, ni_e, no_e, f, lane, G, em)) return;
  PhiloxOut w{0u, 0u, 0u, 0u};
  if (lane < f)
    w = philox4x32_10(static_cast<uint32_t>(lane), static_cast<uint32_t>(v),
                      (kTagSample << 24) | static_cast<uint32_t>(hop), batch, k0, k1);
  const uint64_t u01 = lo64(w), u23 = hi64(w);
  int K = 0, kb;
  if (law == 1) {  // slot law: K_draw intra slots, each class clipped, no refill
    const int kd = __popc(__ballot_sync(gmask, lane < f && (u01 >> 48) < wi));
    K = kd < ni_e ? kd : static_cast<int>(ni_e);
    kb = f - kd < no_e ? f - kd : static_cast<int>(no_e);
  } else {
    uint64_t ri = static_cast<uint64_t>(ni_e), ro = static_cast<uint64_t>(no_e);
    for (int s = 0; s < f; ++s) {
      const uint64_t x = __shfl_sync(gmask, u01, s, G);
      const uint64_t wri = wi * ri;
      if (__umul64hi(x, wri + wo * ro) < wri) {
        ++K;
        --ri;
      } else {
        --ro;
      }
    }
    kb = f - K;
  }
  const int tot = K + kb;  // picks of this row (f under law A)
  const bool in = lane < K;
  const uint64_t n_cls = in ? static_cast<uint64_t>(ni_e) : static_cast<uint64_t>(no_e);
  const int k_cls = in ? K : kb;
  const int t = in ? lane : lane - K;
  const uint32_t j = static_cast<uint32_t>(n_cls - static_cast<uint64_t>(k_cls) + t);
  const uint32_t rr = static_cast<uint32_t>(__umul64hi(u23, static_cast<uint64_t>(j) + 1u));
  uint32_t sel = kEmpty;
  for (int s = 0; s < tot; ++s) {
    const uint32_t rs_ = __shfl_sync(gmask, rr, s, G);
    const bool same_cls = (lane < K) == (s < K);
    const unsigned hit = __ballot_sync(gmask, lane < s && same_cls && sel == rs_);
    if (lane == s) sel = hit ? j : rr;
  }
  uint32_t pos = in ? lo + sel : (sel < lo ? sel : hi + (sel - lo));
  if (lane >= tot) pos = kEmpty;
  int rank = 0;
  for (int s = 0; s < tot; ++s) rank += __shfl_sync(gmask, pos, s, G) < pos;
  if (lane < tot) em.put(rank, rs + pos);
}

// one thread per row (f <= FM): the same draws with every loop statically unrolled over FM
// slots (register arrays, predicated on s < f) -- no shuffles, 32 rows per warp.
// (32-bit row quantities: a row's degree is below N < 2^31; fewer registers, fewer spills)
template <int FM, class Emit>
__device__ __forceinline__ void row_positions_thread(int32_t v, int64_t rs, uint32_t deg,
                                                     uint32_t lo, uint32_t hi, int hop, int f,
                                                     uint32_t wi, uint32_t wo, uint32_t k0,
                                                     uint32_t k1, uint32_t batch,
                                                     const Emit& em, int law) {
  const uint32_t ni = hi - lo;
  const uint32_t ni_e = wi ? ni : 0u, no_e = wo ? deg - ni : 0u;
  if (take_all(rs, deg, lo, hi, ni_e, no_e, f, 0, 1, em)) return;
  uint64_t r23[FM];
  uint32_t ri = ni_e, ro = no_e;
  int K = 0, kd = 0;
  const uint32_t c2 = (kTagSample << 24) | static_cast<uint32_t>(hop);
#pragma unroll
  for (int s = 0; s < FM; ++s) {  // urn over f successive draws; keep r23 of each slot
    r23[s] = 0;
    if (s < f) {
      const PhiloxOut w = philox4x32_10(static_cast<uint32_t>(s), static_cast<uint32_t>(v), c2,
                                        batch, k0, k1);
      r23[s] = hi64(w);
      kd += (lo64(w) >> 48) < wi;  // slot law: slot s intra iff unif(r01, 65536) < P16
      const uint64_t wri = static_cast<uint64_t>(wi) * ri;
      if (__umul64hi(lo64(w), wri + static_cast<uint64_t>(wo) * ro) < wri) {
        ++K;
        --ri;
      } else {
        --ro;
      }
    }
  }
  int kb = f - K;
  if (law == 1) {
    K = kd < static_cast<int64_t>(ni_e) ? kd : static_cast<int>(ni_e);
    kb = f - kd < static_cast<int64_t>(no_e) ? f - kd : static_cast<int>(no_e);
  }
  const int tot = K + kb;  // picks of this row (f under law A)
  uint32_t pos[FM];
#pragma unroll
  for (int s = 0; s < FM; ++s) {  // Floyd: slots [0,K) intra subset, [K,K+kb) inter subset
    pos[s] = kEmpty;
    if (s < tot) {
      const bool in = s < K;
      const uint32_t n_cls = in ? ni_e : no_e;
      const int k_cls = in ? K : kb;
      const int t = in ? s : s - K;
      const uint32_t j = n_cls - static_cast<uint32_t>(k_cls) + static_cast<uint32_t>(t);
      const uint32_t r = static_cast<uint32_t>(__umul64hi(r23[s], static_cast<uint64_t>(j) + 1u));
      bool hit = false;
#pragma unroll
      for (int q = 0; q < s; ++q) hit |= ((q < K) == in) && pos[q] == r;
      pos[s] = hit ? j : r;
    }
  }
#pragma unroll
  for (int s = 0; s < FM; ++s) {  // class offsets -> row positions
    if (s < tot) {
      const uint32_t q = pos[s];
      pos[s] = s < K ? lo + q : (q < lo ? q : hi + (q - lo));
    }
  }
  if constexpr (FM <= CMB_PUT_ROW_MAX) {
    em.template put_row<FM>(tot, rs, pos);  // ascending emit by rank, loads batched
  } else {
#pragma unroll
    for (int s = 0; s < FM; ++s) {  // ascending emit by rank
      if (s < tot) {
        int rank = 0;
#pragma unroll
        for (int q = 0; q < FM; ++q) rank += (q < tot) && pos[q] < pos[s];
        em.put(rank, rs + pos[s]);
      }
    }
  }
}

template <int PB, int G, class W>
__device__ void phase_count_sample(const PArgs& a, int h, Smem<PB>& sm, int& pk,
                                   typename MapWord<W>::T tag, unsigned ctr) {
  using T = typename MapWord<W>::T;
  const int64_t n_h = h == 0 ? a.n_roots : __ldcg(a.sizes + h);
  const int32_t* dst = h == 0 ? a.roots : a.nodes;
  const int f = a.fan[h];
  int64_t lo, hi;
  range_of(n_h, 1, lo, hi);
  RowCache& rc = sm.rows;
  if (threadIdx.x == 0) sm.next = 0;  // read after publish_and_prefix's barrier
  // (1) counts, block scan, cached row info.  A thread owns RPT consecutive rows per round: their
  // ids, then their row records and the dst-order histogram atomics are issued before any is
  // used (one block scan per PB * RPT rows); rows in (thread, row) order = row order
#ifndef CMB_COUNT_RPT  // layout experiments only
#define CMB_COUNT_RPT 1
#endif
  constexpr int RPT = CMB_COUNT_RPT;
  const bool place = a.order && h == a.L - 1;
  int32_t run = 0;
  for (int64_t t0 = lo; t0 < hi; t0 += static_cast<int64_t>(PB) * RPT) {
    const int64_t i0 = t0 + static_cast<int64_t>(threadIdx.x) * RPT;
    int32_t v[RPT];
#pragma unroll
    for (int q = 0; q < RPT; ++q) v[q] = i0 + q < hi ? __ldcg(dst + i0 + q) : 0;
    RowInfo r[RPT];
#pragma unroll
    for (int q = 0; q < RPT; ++q)
      r[q] = i0 + q < hi ? row_info_checked(a.g, v[q], a.wi, a.wo) : RowInfo{0, 0, 0, 0, 0u, 0u};
    uint32_t rk[RPT];
#pragma unroll
    for (int q = 0; q < RPT; ++q)  // the row's rank in its bucket (an out-of-range root, flagged,
      rk[q] = place && i0 + q < hi   // counts in bucket 0)
                  ? atomicAdd(a.hist + (static_cast<uint32_t>(v[q]) < static_cast<uint64_t>(a.g.n)
                                            ? static_cast<uint32_t>(v[q]) >> a.order_shift
                                            : 0u),
                              1u)
                  : 0u;
    int32_t c[RPT], sum = 0;
#pragma unroll
    for (int q = 0; q < RPT; ++q) {
      const int64_t m = r[q].ni_e + r[q].no_e;
      c[q] = static_cast<int32_t>(m < f ? m : f);
      if (a.law == 1 && f < m)
        c[q] = slot_count(v[q], h, f, a.wi, r[q].ni_e, r[q].no_e, a.k0, a.k1, a.batch);
      sum += c[q];
    }
    int32_t ex, agg;
    cub::BlockScan<int32_t, PB>(sm.cub.scan).ExclusiveSum(sum, ex, agg);
    __syncthreads();
    int32_t off = run + ex;
#pragma unroll
    for (int q = 0; q < RPT; ++q) {
      const int64_t i = i0 + q;
      if (i < hi) {
        const int64_t k = i - lo;
        a.indptr[h][i] = off;
        if (place) a.rank[i] = rk[q];
        if (k < kRowCap) {
          rc.rs[k] = r[q].rs;
          rc.deg[k] = static_cast<uint32_t>(r[q].deg);
          rc.lo[k] = r[q].lo;
          rc.hi[k] = r[q].hi;
          rc.v[k] = v[q];
          rc.off[k] = off;
        }
      }
      off += c[q];
    }
    run += agg;
  }
  CMB_PROF(a, pk);
  const int32_t base = publish_and_prefix<PB>(a.pub, pub_tag(ctr, h), run, sm);
  CMB_PROF(a, pk);
  if (vblk() == vgrid() - 1 && threadIdx.x == 0) {
    a.indptr[h][n_h] = base + run;
    a.sizes[a.L + 1 + h] = base + run;
  }
  // (2) positions
  auto fetch = [&](int64_t i, int32_t& v, int64_t& rs, int64_t& deg, uint32_t& rlo,
                   uint32_t& rhi, int32_t& off) {
    const int64_t k = i - lo;
    if (k < kRowCap) {
      v = rc.v[k];
      rs = rc.rs[k];
      deg = rc.deg[k];
      rlo = rc.lo[k];
      rhi = rc.hi[k];
      off = rc.off[k];
    } else {
      v = __ldcg(dst + i);
      const RowInfo r = row_info_checked(a.g, v, a.wi, a.wo);
      rs = r.rs;
      deg = r.deg;
      rlo = r.lo;
      rhi = r.hi;
      off = __ldcg(a.indptr[h] + i);
    }
  };
  // thread per row when the block has many rows (every thread busy); G-lane groups when the
  // rows are few (small hops: spread each row's f draws over lanes instead)
#ifndef CMB_SAMPLER_ROWS_PER_THREAD  // rows per thread above which a thread takes a whole row
#define CMB_SAMPLER_ROWS_PER_THREAD 0  // (layout experiments only; 0: whenever G-lane groups
#endif                                 // would need more than one pass over the block's rows)
  if (f <= 16 && (hi - lo) * G > PB && (hi - lo) > static_cast<int64_t>(PB) * CMB_SAMPLER_ROWS_PER_THREAD) {
    auto row = [&](int32_t i) {
      int32_t v, off;
      int64_t rs, deg;
      uint32_t rlo, rhi;
      fetch(i, v, rs, deg, rlo, rhi, off);
      a.indptr[h][i] = base + off;
      const uint32_t e0 = static_cast<uint32_t>(base + off);
      const PickEmit<W> em{a.g.indices, a.indices[h] + e0, static_cast<T*>(a.map), tag, e0};
      // the slot arrays are sized to the fanout: an unrolled slot a row does not use still
      // issues its (predicated) Philox rounds -- exact sizes for the per-row fanouts of the
      // BASELINE configs' big hops (5, 10) cut the sampler 3.5 % on products (f = 5 was an
      // 8-slot form); other fanouts round up to 8 or 16 slots (more exact sizes spill)
      switch (f) {
#define CMB_ROWPOS(FM_)                                                                      \
    row_positions_thread<FM_>(v, rs, static_cast<uint32_t>(deg), rlo, rhi, h, f, a.wi, a.wo,   \
                              a.k0, a.k1, a.batch, em,                                       \
                              a.law);                                                        \
    break;
        case 5: CMB_ROWPOS(5)
        case 10: CMB_ROWPOS(10)
        default:
          if (f <= 8) {
            CMB_ROWPOS(8)
          }
          CMB_ROWPOS(16)
#undef CMB_ROWPOS
      }
    };
    // warps claim 32-row chunks from a block counter: a warp whose rows come back early takes
    // more, so the block's barrier after this step waits less for its slowest warp (a static
    // stride over the rows: 168.6 vs 166.5 us per step on products at 6 batches per launch)
    const int32_t nrows = static_cast<int32_t>(hi - lo);
    const int wl = threadIdx.x & 31;
    for (;;) {
      int32_t c0 = 0;
      if (wl == 0) c0 = atomicAdd(&sm.next, 32);
      c0 = __shfl_sync(0xffffffffu, c0, 0);
      if (c0 >= nrows) break;
      const int32_t i = static_cast<int32_t>(lo) + c0 + wl;
      if (i < hi) row(i);
    }
  } else {
    const int lane = threadIdx.x & (G - 1);
    const int wl = threadIdx.x & 31;
    const unsigned gmask = (G == 32) ? 0xffffffffu : (((1u << G) - 1u) << (wl & ~(G - 1)));
    for (int64_t i = lo + threadIdx.x / G; i < hi; i += PB / G) {
      int32_t v, off;
      int64_t rs, deg;
      uint32_t rlo, rhi;
      fetch(i, v, rs, deg, rlo, rhi, off);
      if (lane == 0) a.indptr[h][i] = base + off;
      const uint32_t e0 = static_cast<uint32_t>(base + off);
      row_positions_group<G>(v, rs, deg, rlo, rhi, h, f, a.wi, a.wo, a.k0, a.k1, a.batch, lane,
                             gmask,
                             PickEmit<W>{a.g.indices, a.indices[h] + e0, static_cast<T*>(a.map),
                                         tag, e0},
                             a.law);
    }
  }
  __syncthreads();
  CMB_PROF(a, pk);
}

// 8 consecutive int32 of p starting at e0 (a multiple of 8), entries at or past n read as 0:
// two 16-byte loads when the run is whole and 16-byte aligned, else scalar loads
__device__ __forceinline__ void ld8(const int32_t* p, int64_t e0, int64_t n, int32_t (&v)[8]) {
  if (e0 + 8 <= n && (reinterpret_cast<uintptr_t>(p + e0) & 15) == 0) {
    const int4 x = __ldcg(reinterpret_cast<const int4*>(p + e0));
    const int4 y = __ldcg(reinterpret_cast<const int4*>(p + e0) + 1);
    v[0] = x.x; v[1] = x.y; v[2] = x.z; v[3] = x.w;
    v[4] = y.x; v[5] = y.y; v[6] = y.z; v[7] = y.w;
  } else {
#pragma unroll
    for (int k = 0; k < 8; ++k) v[k] = e0 + k < n ? __ldcg(p + e0 + k) : 0;
  }
}
__device__ __forceinline__ void st8(int32_t* p, int64_t e0, int64_t n, const int32_t (&v)[8]) {
  if (e0 + 8 <= n && (reinterpret_cast<uintptr_t>(p + e0) & 15) == 0) {
    reinterpret_cast<int4*>(p + e0)[0] = make_int4(v[0], v[1], v[2], v[3]);
    reinterpret_cast<int4*>(p + e0)[1] = make_int4(v[4], v[5], v[6], v[7]);
  } else {
#pragma unroll
    for (int k = 0; k < 8; ++k)
      if (e0 + k < n) p[e0 + k] = v[k];
  }
}

// The visiting order of the last hop's dst rows (blocks.dst_order): after the grid barrier
// that follows the count step every bucket count is final; each block scans the counts and
// places its own dst rows (the count step's row range) at bucket offset + the rank the count
// step's histogram atomic returned (no second atomic: 12.8 -> see DESIGN.md).
template <int PB>
__device__ void place_dst_rows(const PArgs& a, int h, int64_t n_h, Smem<PB>& sm) {
  static_assert(kOrderBuckets % PB == 0, "buckets per thread");
  constexpr int BPT = kOrderBuckets / PB;
  uint32_t* off = reinterpret_cast<uint32_t*>(&sm.rows);  // the row cache is free in this phase
  uint32_t c[BPT];
  int32_t s = 0;
#pragma unroll
  for (int q = 0; q < BPT; ++q) {
    c[q] = __ldcg(a.hist + threadIdx.x * BPT + q);
    s += static_cast<int32_t>(c[q]);
  }
  int32_t ex;
  cub::BlockScan<int32_t, PB>(sm.cub.scan).ExclusiveSum(s, ex);
#pragma unroll
  for (int q = 0; q < BPT; ++q) {
    off[threadIdx.x * BPT + q] = static_cast<uint32_t>(ex);
    ex += static_cast<int32_t>(c[q]);
  }
  __syncthreads();
  const int32_t* dst = h == 0 ? a.roots : a.nodes;
  int64_t lo, hi;
  range_of(n_h, 1, lo, hi);
  constexpr int U = 4;  // rows per thread per round: their loads in flight together
  for (int64_t i0 = lo + threadIdx.x; i0 < hi; i0 += static_cast<int64_t>(U) * PB) {
    uint32_t b[U], pos[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t i = i0 + static_cast<int64_t>(u) * PB;
      const uint32_t v = i < hi ? static_cast<uint32_t>(__ldcg(dst + i)) : 0u;
      b[u] = v < static_cast<uint64_t>(a.g.n) ? v >> a.order_shift : 0u;
      pos[u] = i < hi ? __ldcg(a.rank + i) : 0u;
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t i = i0 + static_cast<int64_t>(u) * PB;
      if (i < hi) a.order[off[b[u]] + pos[u]] = static_cast<int32_t>(i);
    }
  }
  __syncthreads();
}

// flags + prefix + assign
template <int PB, class W>
__device__ void phase_flag_assign(const PArgs& a, int h, Smem<PB>& sm, int& pk,
                                  typename MapWord<W>::T tag, unsigned ctr, bool fuse) {
  using M = MapWord<W>;
  using T = typename M::T;
  T* map = static_cast<T*>(a.map);
  const int64_t n_h = h == 0 ? a.n_roots : __ldcg(a.sizes + h);
  const int64_t e_h = __ldcg(a.sizes + a.L + 1 + h);
  int64_t lo, hi;
  range_of(e_h, 32, lo, hi);
  // fuse (last hop, 32-bit words): the relabel of this hop is done here, not in a pass after one
  // more grid barrier.  Every edge's entry is final after the marks: its own marker (a first
  // occurrence), a final id (a node of an earlier hop) or the marker of the first occurrence w.
  // The scan word then records that: flag << 31 | count, 1 << 30 | id, or w; the assign loop
  // turns w into id(w) = n_h + base(block of w) + count(w) - 1 from the blocks' published bases.
  unsigned long long* bases = a.pub + 2 * kMaxBlocks;
  uint32_t* mask = (h == a.L - 1) ? a.mask : nullptr;
  const int32_t* nbr = a.indices[h];
  if (a.order && h == a.L - 1) {
    place_dst_rows<PB>(a, h, n_h, sm);
    CMB_PROF(a, pk);  // (timeline: the last hop's "place" sub-step)
  }
  // a thread owns EPT consecutive edges per round (the block's range is 32-aligned, so 32 / EPT
  // threads fill one new-src mask word): their ids in vector loads, all EPT map lookups in
  // flight, one block scan per PB * EPT edges
#ifndef CMB_FLAG_EPT  // layout experiments only: 8 or 16
#define CMB_FLAG_EPT 8
#endif
  constexpr int EPT = CMB_FLAG_EPT;
  static_assert(EPT == 8 || EPT == 16, "edges per thread in the flag step");
  int32_t run = 0;
  for (int64_t c0 = lo; c0 < hi; c0 += static_cast<int64_t>(PB) * EPT) {
    const int64_t e0 = c0 + static_cast<int64_t>(threadIdx.x) * EPT;
    int32_t u[EPT];
#pragma unroll
    for (int q = 0; q < EPT; q += 8)
      ld8(nbr, e0 + q, hi, *reinterpret_cast<int32_t(*)[8]>(u + q));
    T mv[EPT];
#pragma unroll
    for (int k = 0; k < EPT; ++k) mv[k] = map_ld(map + u[k]);  // past hi: u = 0, harmless
    uint32_t fl = 0;
#pragma unroll
    for (int k = 0; k < EPT; ++k)
      fl |= (e0 + k < hi && mv[k] == (tag | (M::kMarkerTop - static_cast<uint32_t>(e0 + k))))
                ? (1u << k) : 0u;
    int32_t ex, agg;
    cub::BlockScan<int32_t, PB>(sm.cub.scan).ExclusiveSum(__popc(fl), ex, agg);
    __syncthreads();
    int32_t sc[EPT];
    int32_t acc = run + ex;
#pragma unroll
    for (int k = 0; k < EPT; ++k) {  // flag << 31 | block-local inclusive flag count
      acc += (fl >> k) & 1u;
      sc[k] = static_cast<int32_t>(((fl >> k) & 1u) << 31 | static_cast<uint32_t>(acc));
      if (fuse && !((fl >> k) & 1u))  // not a first occurrence: the node's id, or its first edge
        sc[k] = static_cast<int32_t>(
            (mv[k] & M::kFinal) ? (1u << 30) | static_cast<uint32_t>(mv[k] & M::kVal)
                                : M::kMarkerTop - static_cast<uint32_t>(mv[k] & M::kVal));
    }
#pragma unroll
    for (int q = 0; q < EPT; q += 8)
      st8(reinterpret_cast<int32_t*>(a.scan), e0 + q, hi,
          *reinterpret_cast<const int32_t(*)[8]>(sc + q));
    if (mask) {  // edges e0 .. e0+EPT-1 are bits EPT * (thread % (32 / EPT)) .. of word e0 / 32
      constexpr int TPW = 32 / EPT;
      uint32_t w = fl << (EPT * (threadIdx.x & (TPW - 1)));
#pragma unroll
      for (int o = 1; o < TPW; o <<= 1) w |= __shfl_xor_sync(0xffffffffu, w, o);
      if ((threadIdx.x & (TPW - 1)) == 0 && e0 < hi) mask[e0 >> 5] = w;
    }
    run += agg;
  }
  CMB_PROF(a, pk);
  if (fuse) __threadfence();  // this thread's scan words before the block's base (below)
  const int32_t base =
      publish_and_prefix<PB>(a.pub + kMaxBlocks, pub_tag(ctr, h), run, sm);
  CMB_PROF(a, pk);
  if (vblk() == vgrid() - 1 && threadIdx.x == 0) a.sizes[h + 1] = n_h + base + run;
  if (fuse) {
    if (threadIdx.x == 0)  // the block's base, tagged like the aggregates (no clearing needed)
      st_release64(bases + vblk(), (static_cast<unsigned long long>(pub_tag(ctr, h)) << 32) |
                                       static_cast<uint32_t>(base));
    int64_t per = (e_h + vgrid() - 1) / vgrid();  // range_of's block size
    per = (per + 31) / 32 * 32;
    int32_t* ind = a.indices[h];
    // a node's first occurrence w precedes every other edge of it, so its block is this block
    // or an earlier one: collect the bases of blocks 0 .. vblk() once (each published right
    // after that block's prefix, which all aggregates this block already saw allow), then the
    // edges' id lookups are independent loads -- no per-edge wait
    uint32_t* sbase = reinterpret_cast<uint32_t*>(&sm.rows);  // the row cache is free here
    const unsigned want = pub_tag(ctr, h);
    for (int j = threadIdx.x; j <= vblk(); j += PB) {
      if (j == vblk()) {
        sbase[j] = static_cast<uint32_t>(base);
      } else {
        unsigned long long v;
        while (((v = ld_acquire64(bases + j)) >> 32) != want) {
        }
        sbase[j] = static_cast<uint32_t>(v);
      }
    }
    __syncthreads();  // (the acquires above order every thread's scan reads below)
    for (int64_t e0 = lo + static_cast<int64_t>(threadIdx.x) * 8; e0 < hi;
         e0 += static_cast<int64_t>(PB) * 8) {
      int32_t sc[8], u[8], id[8];
      ld8(reinterpret_cast<const int32_t*>(a.scan), e0, hi, sc);
      ld8(nbr, e0, hi, u);
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const uint32_t c = static_cast<uint32_t>(sc[k]);
        if (c >> 31) {  // a first occurrence -> the next local id
          id[k] = static_cast<int32_t>(n_h + base + (c & 0x7fffffffu) - 1);
          if (e0 + k < hi) {
            a.nodes[id[k]] = u[k];
            if (h < a.L - 1)  // the next hop's marks must see the node's final id
              map_st(map + u[k], tag | M::kFinal | static_cast<uint32_t>(id[k]));
          }
        } else if (c >> 30) {  // a node of an earlier hop
          id[k] = static_cast<int32_t>(c & 0x3fffffffu);
        } else if (e0 + k >= hi) {
          id[k] = 0;
        } else {  // the id given to edge c, the node's first occurrence (maybe another block's)
          const uint32_t cw = static_cast<uint32_t>(__ldcg(a.scan + c)) & 0x7fffffffu;
          id[k] = static_cast<int32_t>(n_h + static_cast<int64_t>(sbase[c / per]) + cw - 1);
        }
      }
      st8(ind, e0, hi, id);
      if (h == a.L - 1) st8(a.last_src, e0, hi, u);
    }
    return;
  }
  for (int64_t e0 = lo + static_cast<int64_t>(threadIdx.x) * 8; e0 < hi;
       e0 += static_cast<int64_t>(PB) * 8) {
    int32_t sc[8], u[8];
    ld8(reinterpret_cast<const int32_t*>(a.scan), e0, hi, sc);
    ld8(nbr, e0, hi, u);
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      if (sc[k] < 0) {  // flag bit 31: a first occurrence -> the next local id
        const uint32_t id =
            static_cast<uint32_t>(n_h + base + (static_cast<uint32_t>(sc[k]) & 0x7fffffffu) - 1);
        a.nodes[id] = u[k];
        map_st(map + u[k], tag | M::kFinal | id);
      }
    }
  }
}

constexpr int kMaxNB = CMB_MAX_BATCHES_PER_LAUNCH;  // batches per launch
struct PMulti {
  int nb;
  PArgs a[kMaxNB];
};

template <int PB, class W>
__device__ __forceinline__ void run_batch(const PArgs& a) {
  using M = MapWord<W>;
  using T = typename M::T;
  T* map = static_cast<T*>(a.map);
  extern __shared__ __align__(16) unsigned char smem_raw[];
  Smem<PB>& sm = *reinterpret_cast<Smem<PB>*>(smem_raw);
  __shared__ unsigned gen_s, ctr_s, width_s;
  constexpr unsigned kWidth = sizeof(T);
  if (threadIdx.x == 0) {
    gen_s = ld_acquire(a.bar + 1);
    ctr_s = __ldcg(a.tag_ctr) + 1u;  // this batch's counter (published by block 0 below)
    width_s = __ldcg(a.tag_ctr + 1);  // map word bytes of the workspace's last batch (0: none)
  }
  __syncthreads();
  unsigned gen = gen_s;
  const unsigned ctr = ctr_s;
  // map tag 1..kTagMax; the batch that (re)starts at tag 1 clears the map first, so no entry of
  // an earlier cycle can beat this cycle's markers (the workspace starts zeroed: counter 0), and
  // so does a batch whose map width differs from the previous batch's on this workspace
  const unsigned tagv = (ctr - 1u) % M::kTagMax + 1u;
  const T tag = static_cast<T>(tagv) << M::kShift;
  int pk = 0;
  if ((tagv == 1u && ctr > 1u) || (width_s != 0u && width_s != kWidth)) {
    const int64_t n = a.g.n;
    for (int64_t i = vblk() * (int64_t)PB + threadIdx.x; i < n; i += (int64_t)vgrid() * PB)
      map[i] = T(0);
    grid_barrier(a.bar, gen);
  }
  // the dst-order buckets start empty: cleared here, before the grid barrier that precedes the
  // last hop's count step (one more barrier when that count step is hop 0's)
  if (a.order && vblk() == 0)
    for (int i = threadIdx.x; i < kOrderBuckets; i += PB) a.hist[i] = 0u;
  if (a.order && a.L == 1) grid_barrier(a.bar, gen);
  CMB_PROF(a, pk);
  for (int64_t i = vblk() * (int64_t)PB + threadIdx.x; i < a.n_roots;
       i += (int64_t)vgrid() * PB) {
    const uint32_t u = static_cast<uint32_t>(a.roots[i]);
    if (u >= static_cast<uint64_t>(a.g.n)) {  // out of range: error; the row samples nothing and
      raise_status(a.status, CMB_ERR_INVALID_INPUT);  // node 0 stands in for it in the outputs, so
      a.nodes[i] = 0;                                 // every later read stays inside the graph
      continue;
    }
    a.nodes[i] = static_cast<int32_t>(u);
    const T old = map_exch(map + u, tag | M::kFinal | static_cast<uint32_t>(i));
    // duplicate root <=> the entry already holds a final id of THIS batch (a marker of this
    // batch -- hop-0 picks run concurrently -- is not a duplicate: the final id replaces it)
    if ((old >> M::kShift) == tagv && (old & M::kFinal))
      raise_status(a.status, CMB_ERR_INVALID_INPUT);
  }
  if (vblk() == 0 && threadIdx.x == 0) a.sizes[0] = a.n_roots;
  for (int h = 0; h < a.L; ++h) {
    // (32-bit words: every hop relabels inside its own assign step, so no pass here)
    if (h > 0 && sizeof(T) != 4) phase_relabel<PB, W>(a, h - 1);
    CMB_PROF(a, pk);                                  // +0 relabel(h-1)
    const int f = a.fan[h];
#if defined(CMB_SAMPLER_G8)
    if (f <= 8) phase_count_sample<PB, 8, W>(a, h, sm, pk, tag, ctr);
    else
#endif
    if (f <= 16) phase_count_sample<PB, 16, W>(a, h, sm, pk, tag, ctr);
    else phase_count_sample<PB, 32, W>(a, h, sm, pk, tag, ctr);  // +1 count, +2 prefix, +3 positions
    CMB_PROF(a, pk);                                  // +4 picks + marks
    grid_barrier(a.bar, gen);
    CMB_PROF(a, pk);                                  // +5 barrier (marks final)
    if (h == 0 && vblk() == 0 && threadIdx.x == 0) {  // all blocks have read them
      a.tag_ctr[0] = ctr;
      a.tag_ctr[1] = kWidth;
    }
    // with 32-bit words every hop relabels inside its assign step (no relabel pass; the last
    // hop needs no barrier after it)
    const bool fuse = sizeof(T) == 4;
    phase_flag_assign<PB, W>(a, h, sm, pk, tag, ctr, fuse);  // +6 flag scan, +7 prefix
    CMB_PROF(a, pk);                                  // +8 assign (+ relabel if fused)
    if (fuse && h == a.L - 1) break;
    grid_barrier(a.bar, gen);
    CMB_PROF(a, pk);                                  // +9 barrier
  }
  if (sizeof(T) != 4) phase_relabel<PB, W>(a, a.L - 1);
  CMB_PROF(a, pk);
}

template <int PB, class W>
__global__ void __launch_bounds__(PB, 1024 / PB)
    k_sample_persistent(const __grid_constant__ PMulti m) {
  const int nb = m.nb;
  const int grp = blockIdx.x % nb;
  if (threadIdx.x == 0) {
    g_vblk = blockIdx.x / nb;
    g_vgrid = (gridDim.x - grp + nb - 1) / nb;
  }
  __syncthreads();
  run_batch<PB, W>(m.a[grp]);
}

template <int PB>
constexpr size_t smem_bytes() {
  return sizeof(Smem<PB>);
}

}  // namespace pst
}  // namespace cmb
