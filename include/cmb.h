/*
 * cmb.h -- C ABI of the B200-native COMM-RAND mini-batch hot path
 * (arXiv 2504.18082, "community-structure-aware randomized mini-batching").
 *
 * One mini-batch step (Alg. 1) is:
 *   a0 cmb_load_graph            community offsets + per-row intra segment (once per graph)
 *   a1 cmb_order_roots           Knob-1 root order (Table 1; S4.1 P:653-680), once per epoch
 *   a2+a3 cmb_sample_blocks      Knob-2 biased fanout sampling (S4.2 P:683-691) + dedup/relabel
 *                                into per-hop blocks ("Build sub-graph S_i")
 *   a4 cmb_gather_features       input-feature rows of the sub-graph
 *   a5 cmb_sage_mean_aggregate   GraphSAGE mean aggregation of the input-side block
 *   a4+a5 cmb_gather_aggregate   both in one pass over the feature table
 *   NEXT-4 cmb_sage_layer_forward  a4+a5 fused with the first GraphSAGE layer (tcgen05 bf16 GEMM)
 *
 * Conventions (all entry points):
 *  - extern "C", plain pointers and sizes; "device" = CUDA global memory of the
 *    current device, "host" = ordinary host memory.
 *  - Every device buffer is OWNED BY THE CALLER (allocate it with any CUDA
 *    allocator, e.g. PyTorch's caching allocator).  The library never allocates
 *    or frees device memory; workspaces are sized by the *_workspace_bytes
 *    queries and must be 256-byte aligned.
 *  - Work is enqueued asynchronously on `stream` (a cudaStream_t, NULL = the
 *    legacy default stream).  Buffers must stay valid until it completes.
 *    No entry point except cmb_load_graph(validate=1) and cmb_get_device_status
 *    synchronises; sizes produced on the device stay on the device, so a whole
 *    batch can be enqueued (or graph-captured) without host round trips.
 *  - Errors: host-checkable errors are returned immediately.  Conditions only
 *    the device can see (capacity overflow, a full hash table, invalid input
 *    data) set a sticky status word inside the workspace, read with
 *    cmb_get_device_status.  No call aborts or traps; no exception crosses the
 *    ABI; cmb_last_error_message() holds a thread-local detail string.
 *  - Requires a compute capability 10.0 device (B200, sm_100a) and returns
 *    CMB_ERR_UNSUPPORTED_DEVICE otherwise.
 *  - Randomness: Philox4x32-10 (Salmon et al., SC'11), key = seed, counter =
 *    (slot, node-or-community id, (tag << 24) | hop, batch-or-epoch)
 *    (reading R11); tags 1 = sampling, 2 = root key, 3 = community key.
 *    Every result is a pure function of (graph, seed, batch/epoch, knobs).
 */
#ifndef CMB_H_
#define CMB_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#if defined(__GNUC__)
#define CMB_API __attribute__((visibility("default")))
#else
#define CMB_API
#endif

#define CMB_VERSION_MAJOR 0
#define CMB_VERSION_MINOR 1
#define CMB_MAX_HOPS 8
#define CMB_MAX_FANOUT 32

typedef enum {
  CMB_OK = 0,
  CMB_ERR_INVALID_ARGUMENT = 1,      /* null pointer, bad size/knob, misaligned buffer      */
  CMB_ERR_INVALID_GRAPH = 2,         /* CSR row unsorted / duplicate / id out of range      */
  CMB_ERR_NOT_COMMUNITY_ORDERED = 3, /* community ids not non-decreasing / gap / out of range */
  CMB_ERR_CAPACITY = 4,              /* output or workspace capacity too small               */
  CMB_ERR_CUDA = 5,                  /* a CUDA runtime call failed (see last_error_message)  */
  CMB_ERR_UNSUPPORTED_DEVICE = 6,    /* current device is not compute capability 10.x        */
  CMB_ERR_INVALID_INPUT = 7          /* device-detected bad input (duplicate / unsorted ids) */
} cmb_status;

/* Knob-1 root partitioning policies (Table 1). */
typedef enum {
  CMB_ROOTS_RAND = 0,   /* RAND-ROOTS: uniform shuffle of the training set               */
  CMB_ROOTS_NORAND = 1, /* NORAND-ROOTS: no shuffle; static across epochs                */
  CMB_ROOTS_COMM = 2,   /* COMM-RAND-MIX-k%: shuffle communities as blocks, group k% of
                           the training-set communities into super-blocks, shuffle the
                           nodes inside each super-block (k = mix_fraction)              */
  CMB_ROOTS_COMM_STATIC = 3 /* COMM-RAND-MIX-k% with STATIC super-blocks of k% ADJACENT
                           training-set communities (id order; SURVEY.md 8(f) NEXT-2 (ii),
                           reading R24): the super-blocks are shuffled as units each epoch,
                           the nodes inside each super-block shuffled                    */
} cmb_roots_mode;

typedef struct cmb_graph cmb_graph; /* opaque host handle; holds borrowed device pointers */

/* Graph description (a0).  The graph must be community-ordered:
 * community c owns a contiguous id range, i.e. community[] is non-decreasing and
 * every id in [0, num_communities) occurs.  Rows are strictly ascending (simple
 * graph), ids < num_nodes; the graph is expected to be symmetric but the
 * path does not rely on it. */
typedef struct {
  int64_t num_nodes;        /* N                                                        */
  int64_t num_edges;        /* nnz = number of CSR entries                              */
  const int64_t* indptr;    /* device [N+1]                                             */
  const int32_t* indices;   /* device [nnz]                                             */
  const int32_t* community; /* device [N]                                               */
  int32_t num_communities;  /* C >= 1                                                   */
  const float* features;    /* device [N * feat_ld] row-major fp32, or NULL (sample-only) */
  int32_t feat_dim;         /* F (columns used)                                         */
  int64_t feat_ld;          /* row stride in floats, >= F                               */
  void* workspace;          /* device, >= cmb_graph_workspace_bytes(N, C), lives as long as the handle */
  size_t workspace_bytes;
  int32_t validate;         /* 1: check CSR + community order on the device and synchronise */
} cmb_graph_desc;

/* Bytes of graph workspace: community offsets int32[C+1] + per-row intra segment
 * uint32x2[N] + a packed 16-byte row record per node (row start, degree and intra segment,
 * so the sampler reads one random sector per row instead of two or three) + status word. */
CMB_API size_t cmb_graph_workspace_bytes(int64_t num_nodes, int32_t num_communities);

/* a0: builds the per-row intra-community segment [lo, hi) of every row (the
 * neighbours u of v with community[u] == community[v] are contiguous in a
 * sorted row of a community-ordered graph; reading R5) and returns a handle.
 * With validate = 1 it synchronises `stream` and returns CMB_ERR_INVALID_GRAPH /
 * CMB_ERR_NOT_COMMUNITY_ORDERED for bad input. */
CMB_API cmb_status cmb_load_graph(const cmb_graph_desc* desc, void* stream, cmb_graph** out);
CMB_API cmb_status cmb_free_graph(cmb_graph* g); /* frees the host handle only */
/* Device pointers of the a0 products (for tests / tools): cbeg int32[C+1],
 * bounds uint32[2N] = (lo, hi) per row. */
CMB_API cmb_status cmb_graph_arrays(const cmb_graph* g, const int32_t** cbeg, const uint32_t** bounds);

/* ------------------------------------------------------------------ a1 */
CMB_API size_t cmb_order_roots_workspace_bytes(int64_t n_train, int32_t num_communities);
/* Root order for one epoch (Knob-1).  train_ids: device int32[n_train], ascending
 * and unique (the training set).  out_order: device int32[n_train], a permutation
 * of train_ids.  Batches are consecutive batch_size slices of out_order, the last
 * one partial (reading R21).
 *   RAND:   sorted by (key(v), v), key(v) = 64-bit Philox(0, v, 2<<24, epoch)
 *   NORAND: train_ids unchanged
 *   COMM:   C_tr = distinct communities of the training set (ascending); they are
 *           shuffled (sorted by (ckey(c), c)); consecutive runs of
 *           S = max(1, floor(mix_fraction * C_tr + 0.5)) of them form super-blocks;
 *           nodes are sorted by (super-block, key(v), v).  mix_fraction = 0 is
 *           COMM-RAND-MIX-0%, 1 reproduces RAND bit for bit (readings R9, R10).
 *   COMM_STATIC: the C_tr communities in ascending id order, j = 0..C_tr-1, form
 *           super-blocks b = j / S (adjacent, fixed across epochs); super-blocks are
 *           ranked by (sbkey(b), b), sbkey(b) = 64-bit Philox(1, b, 3<<24, epoch), and
 *           nodes sorted by (super-block rank, key(v), v) (reading R24).
 * mix_fraction in [0, 1].  Non-ascending train_ids set CMB_ERR_INVALID_INPUT in
 * the workspace status word. */
CMB_API cmb_status cmb_order_roots(const cmb_graph* g, const int32_t* train_ids, int64_t n_train,
                           cmb_roots_mode mode, double mix_fraction, uint64_t seed, uint32_t epoch,
                           int32_t* out_order, void* workspace, size_t workspace_bytes,
                           void* stream);

/* ------------------------------------------------------------------ a2 + a3 */
/* Per-batch sub-graph in HOP order: hop h expands dst nodes nodes[0:n_h) and its
 * block has src nodes nodes[0:n_{h+1}) (the dst list is the src prefix, reading
 * R7; DGL's block index is L-1-h).  New src nodes are appended in order of first
 * occurrence over (dst index, row position) (reading R8).  All buffers device. */
typedef struct {
  int32_t* nodes;                      /* [nodes_cap] global ids; nodes[0:n_L) = input nodes  */
  int64_t nodes_cap;
  int32_t* indptr[CMB_MAX_HOPS];       /* hop h: [n_cap[h] + 1]; entries beyond n_h equal e_h */
  int32_t* indices[CMB_MAX_HOPS];      /* hop h: [e_cap[h]] local src ids in [0, n_{h+1})     */
  int64_t indices_cap[CMB_MAX_HOPS];
  uint32_t* new_src_mask;              /* optional (NULL): [(e_cap[L-1]+31)/32] words; bit e set
                                          iff edge e of hop L-1 is the first occurrence of a src
                                          node that is not a dst node (used by cmb_gather_aggregate) */
  int32_t* last_src_ids;               /* optional (NULL): [e_cap[L-1]] global id of the src node of
                                          every edge of hop L-1 (= nodes[indices[L-1][e]]; lets
                                          cmb_gather_aggregate skip the relabel-map lookup)      */
  int64_t* sizes;                      /* [2L+1]: n_0..n_L then e_0..e_{L-1}                  */
  int32_t* dst_order;                  /* optional (NULL): [n_cap[L-1]] the sampler writes a
                                          permutation of [0, n_{L-1}) grouping the dst rows of
                                          hop L-1 by node-id bucket (v >> s, at most 4096
                                          buckets; order inside a bucket unspecified) and the
                                          a4 + a5 calls visit the rows in that order, so rows
                                          of one community, which share most of their src rows
                                          (P:683-691), are processed together and re-read those
                                          rows from L2.  Results do not depend
                                          on it: every output row is the same, byte for byte. */
} cmb_blocks;

/* Capacity bounds (host): n_cap[0] = n_roots, e_cap[h] = n_cap[h] * f_h,
 * n_cap[h+1] = min(num_nodes, n_cap[h] + e_cap[h]).  n_cap has n_hops+1 entries. */
CMB_API void cmb_blocks_capacity(int64_t n_roots, const int32_t* fanouts, int32_t n_hops,
                         int64_t num_nodes, int64_t* n_cap, int64_t* e_cap);
/* Bytes of sampler workspace for batches of up to n_roots roots: device, 256-B aligned,
 * zero-filled ONCE by the caller and then owned by the sampler (no per-batch memset): grid
 * barrier words, tagged block aggregates, a batch counter and a direct dedup map of one word per
 * node -- 32-bit words (7-bit batch tag: the batch that wraps the tag clears the map) when every
 * local id and edge position of a batch of this capacity is below 2^24, else 64-bit words.  A
 * workspace may serve batches of either width (a width change clears the map); one launch
 * uses one width for all its batches, so a workspace sized for the narrow width must not be
 * combined with a batch that needs the wide one (CMB_ERR_INVALID_ARGUMENT). */
CMB_API size_t cmb_sample_workspace_bytes(int64_t n_roots, const int32_t* fanouts, int32_t n_hops,
                                  int64_t num_nodes);
/* Samples an n_hops-hop sub-graph from `roots` (device int32[n_roots], distinct).
 * fanouts: HOST int32[n_hops] in hop order (fanouts[0] expands the roots; reading
 * R6), each in [1, CMB_MAX_FANOUT].  p_intra in [0, 1] (Knob-2; the paper's range
 * is [0.5, 1]): every intra-community edge of the expanded node has weight
 * P16 = floor(p*65536 + 0.5), every other edge 65536 - P16, and each row draws
 * min(f, #positive-weight neighbours) distinct neighbours by successive weighted
 * sampling without replacement (DGL NeighborSampler(prob=...); readings
 * R1-R4, R13).  batch_id keys the RNG (use epoch * n_batches + b).  Blocks in
 * `out` must have at least the cmb_blocks_capacity capacities. */
CMB_API cmb_status cmb_sample_blocks(const cmb_graph* g, const int32_t* roots, int64_t n_roots,
                             const int32_t* fanouts, int32_t n_hops, double p_intra, uint64_t seed,
                             uint32_t batch_id, cmb_blocks* out, void* workspace,
                             size_t workspace_bytes, void* stream);

/* Knob-2 laws.  CMB_LAW_A (default of cmb_sample_blocks): successive weighted sampling without
 * replacement with per-edge weights P16 / 65536 - P16 (DGL NeighborSampler(prob=...);
 * reading R1).  CMB_LAW_SLOT (reading R23, the north_star's literal
 * "takes an intra-community neighbour with probability p_intra"): take-all first; else each of
 * the f slots is intra iff unif(r01(W_s), 65536) < P16, the K_draw intra slots take
 * min(K_draw, ni_e) distinct intra neighbours and the rest min(f - K_draw, no_e) distinct inter
 * ones (no refill: a row may return fewer than f picks), with the same Philox words and Floyd
 * steps as law A. */
typedef enum { CMB_LAW_A = 0, CMB_LAW_SLOT = 1 } cmb_sample_law;

/* cmb_sample_blocks under an explicit law (CMB_INVALID_ARGUMENT for an unknown law). */
CMB_API cmb_status cmb_sample_blocks_law(const cmb_graph* g, const int32_t* roots, int64_t n_roots,
                                         const int32_t* fanouts, int32_t n_hops, double p_intra,
                                         int32_t law, uint64_t seed, uint32_t batch_id,
                                         cmb_blocks* out, void* workspace, size_t workspace_bytes,
                                         void* stream);

/* Several independent batches in ONE launch (up to CMB_MAX_BATCHES_PER_LAUNCH): the SMs are
 * split evenly between the batches, which run the same phases concurrently, so the latency-
 * bound phases of small hops overlap across batches.  Each batch has its own roots, batch id,
 * output blocks and workspace (workspaces must be distinct); results are identical to
 * calling cmb_sample_blocks once per batch. */
#ifndef CMB_MAX_BATCHES_PER_LAUNCH
#define CMB_MAX_BATCHES_PER_LAUNCH 8
#endif
typedef struct {
  const int32_t* roots; /* device int32[n_roots], distinct */
  int64_t n_roots;
  uint32_t batch_id;
  cmb_blocks* out;
  void* workspace;
  size_t workspace_bytes;
} cmb_batch;
CMB_API cmb_status cmb_sample_blocks_multi(const cmb_graph* g, const cmb_batch* batches,
                                           int32_t n_batches, const int32_t* fanouts,
                                           int32_t n_hops, double p_intra, int32_t law,
                                           uint64_t seed, void* stream);

/* ------------------------------------------------------------------ a4 / a5 */
/* a4: out[i, 0:F] = features[node_ids[i], 0:F] for i < *n_dev (device count; rows
 * beyond it up to n_cap are untouched).  Bit-exact copy.  out_ld >= F floats. */
CMB_API cmb_status cmb_gather_features(const cmb_graph* g, const int32_t* node_ids, const int64_t* n_dev,
                               int64_t n_cap, float* out, int64_t out_ld, void* stream);

/* a5: H[d, j] = (sum over e in [indptr[d], indptr[d+1]) in CSR order of
 * src[row(e), j]) / deg_d, fp32 accumulation and IEEE division; H[d] = 0 for an
 * empty row (reading R12: neighbours only).  row(e) = indices[e], or
 * src_map[indices[e]] when src_map != NULL (the fused form reading the feature
 * table directly).  d < *n_dst_dev (device count) <= n_dst_cap. */
CMB_API cmb_status cmb_sage_mean_aggregate(const int32_t* indptr, const int32_t* indices,
                                   const int64_t* n_dst_dev, int64_t n_dst_cap, const float* src,
                                   int64_t src_ld, const int32_t* src_map, int32_t feat_dim,
                                   float* out, int64_t out_ld, void* stream);

/* a4 + a5 in one pass over the feature table for the input-side block (hop L-1):
 * writes X_in[i] = features[nodes[i]] for every i < n_L and H = mean aggregate of
 * hop L-1 (same arithmetic as cmb_sage_mean_aggregate).  Each feature row is
 * read once per reference; X_in rows of new src nodes are written at their first
 * occurrence (blocks->new_src_mask must have been filled by cmb_sample_blocks). */
CMB_API cmb_status cmb_gather_aggregate(const cmb_graph* g, const cmb_blocks* blocks, int32_t n_hops,
                                int64_t n_last_dst_cap, int64_t nodes_cap, float* x_in,
                                int64_t x_in_ld, float* h_out, int64_t h_ld, void* stream);

/* ------------------------------------------------------------------ a6: row-sharded features */
/* Rank r of `world` owns feature rows [r*S, min(N, (r+1)*S)), S = rows_per_shard (north_star:
 * "for papers100M-scale inputs the feature table is row-sharded, with an NCCL all-to-all over
 * NVLink for remote rows").  The exchange of one batch is: cmb_shard_plan on the requesting
 * rank, all-to-all of counts and ids (NCCL, host side), cmb_gather_rows on every owner,
 * all-to-all of the rows back, cmb_scatter_rows -> X_in byte-identical to cmb_gather_features
 * on a replicated table. */
CMB_API size_t cmb_shard_plan_workspace_bytes(int64_t n_cap);
/* Stable bucketing of nodes[0:*n_dev) by owner = id / rows_per_shard: counts (device int64
 * [world]), send_ids (device int32 [n_cap], owner-major, original order within an owner) and
 * perm (device int32 [n_cap], the X_in row of each send slot).  An id whose owner is >= world
 * sets CMB_ERR_INVALID_INPUT in the workspace status. */
CMB_API cmb_status cmb_shard_plan(const int32_t* nodes, const int64_t* n_dev, int64_t n_cap,
                                  int64_t rows_per_shard, int32_t world, int64_t* counts,
                                  int32_t* send_ids, int32_t* perm, void* workspace,
                                  size_t workspace_bytes, void* stream);
/* Row gather from a (shard of a) feature table whose first row is global row `row0`:
 * out[i, 0:F] = x[(ids[i] - row0) * ld + 0:F] for i < *n_dev <= n_cap.  Bit-exact copy. */
CMB_API cmb_status cmb_gather_rows(const float* x, int64_t ld, int64_t row0, int32_t feat_dim,
                                   const int32_t* ids, const int64_t* n_dev, int64_t n_cap,
                                   float* out, int64_t out_ld, void* stream);
/* out[perm[k], 0:F] = rows[k, 0:F] for k < *n_dev <= n_cap. */
CMB_API cmb_status cmb_scatter_rows(const float* rows, int64_t rows_ld, const int32_t* perm,
                                    const int64_t* n_dev, int64_t n_cap, int32_t feat_dim,
                                    float* out, int64_t out_ld, void* stream);

/* ------------------------------------------------------------------ NEXT-2 (iii): reorder */
/* Community reordering of a graph that is NOT community-ordered (
 * reading R25): new ids sort the nodes by (community, old id); perm[new] = old,
 * inv[old] = new; row i of the output is old row perm[i] renamed through inv and sorted;
 * community_out[i] = community[perm[i]] (non-decreasing, ready for cmb_load_graph).  All
 * arrays are device, caller-allocated: perm / inv / community_out [N], indptr_out [N+1],
 * indices_out [nnz].  N < 2^31; nnz of any size (above 2^31 - 1 entries the rows are sorted in
 * chunks of <= 2^30 entries, whose boundaries are read back to the host once: the call then
 * synchronises the stream; a single row must stay below 2^30 entries).  Feature rows and train
 * ids follow the permutation (e.g. cmb_gather_rows with perm; train_new = sort(inv[train])). */
CMB_API size_t cmb_community_order_workspace_bytes(int64_t num_nodes, int64_t nnz);
CMB_API cmb_status cmb_community_order(const int64_t* indptr, const int32_t* indices,
                                       const int32_t* community, int64_t num_nodes, int64_t nnz,
                                       int32_t num_communities, int32_t* perm, int32_t* inv,
                                       int64_t* indptr_out, int32_t* indices_out,
                                       int32_t* community_out, void* workspace,
                                       size_t workspace_bytes, void* stream);

/* ------------------------------------------------------------------ step executor */
/* Where cmb_step_group writes the a4 + a5 outputs of one batch (see cmb_gather_aggregate). */
typedef struct {
  float* x_in;
  int64_t x_in_ld;
  float* h_out;
  int64_t h_ld;
  int64_t n_last_dst_cap; /* n_cap[L-1] of the batch's blocks */
  int64_t nodes_cap;      /* n_cap[L]                         */
} cmb_batch_features;
/* a4 + a5 of n_batches (<= CMB_MAX_BATCHES_PER_LAUNCH) sampled batches in ONE launch: exactly
 * cmb_gather_aggregate of each (same outputs, byte for byte), their dst rows walked as one
 * sequence so the batches share the launch (no gap and no tail between them).  blocks[j] and
 * feats[j] as cmb_gather_aggregate's arguments; every batch needs new_src_mask and
 * last_src_ids, 16-B aligned output rows and a 16-B aligned feature table. */
CMB_API cmb_status cmb_gather_aggregate_multi(const cmb_graph* g, const cmb_blocks* const* blocks,
                                              const cmb_batch_features* feats, int32_t n_batches,
                                              int32_t n_hops, void* stream);
/* One launch group of the step, enqueued by ONE call: cmb_sample_blocks_multi over the
 * n_batches batches, then cmb_gather_aggregate_multi over them (same results as
 * cmb_gather_aggregate of each).  events: NULL, or 2 + 2 * n_batches cudaEvent_t (entries may be
 * NULL) recorded on `stream` before/after the sampler launch and around the gather launch:
 * events[2], events[3] bracket it, events[4 ..] are recorded at its end (so per-batch gather
 * times sum to the launch's). */
CMB_API cmb_status cmb_step_group(const cmb_graph* g, const cmb_batch* batches,
                                  const cmb_batch_features* feats, int32_t n_batches,
                                  const int32_t* fanouts, int32_t n_hops, double p_intra,
                                  int32_t law, uint64_t seed, void* const* events, void* stream);

/* ------------------------------------------------------------------ NEXT-3: HBM feature cache */
/* SURVEY.md 8(f) NEXT-3; the paper's software-cache setting (S6.5.1: a GPU cache of
 * node features with LRU replacement in front of UVA reads of a host-resident table).  The
 * feature table stays in pinned host memory (host_x must be device-accessible, e.g.
 * cudaHostAlloc'ed: UVA); `capacity` rows of it are cached in HBM (cache_rows, device,
 * capacity x cache_ld floats).  Replacement is CLOCK (second chance, an LRU approximation);
 * rows referenced by the current batch are never evicted during it.  All buffers are caller
 * owned; the descriptor is plain data. */
typedef struct {
  void* workspace;            /* device, cmb_feature_cache_bytes(), 256-B aligned          */
  size_t workspace_bytes;
  int64_t num_nodes;          /* N of the graph                                           */
  int64_t capacity;           /* cached rows; >= max_rows                                 */
  int64_t max_rows;           /* >= nodes_cap of every batch (unique input rows, n_L cap)  */
  int64_t max_edges;          /* >= indices_cap[L-1] of every batch                       */
  const float* host_x;        /* device-accessible host table [N x host_ld]               */
  int64_t host_ld;
  float* cache_rows;          /* device [capacity x cache_ld]                              */
  int64_t cache_ld;           /* multiple of 4 floats                                     */
} cmb_feature_cache;
CMB_API size_t cmb_feature_cache_bytes(int64_t num_nodes, int64_t capacity, int64_t max_rows,
                                       int64_t max_edges);
/* Empties the cache (every directory entry invalid). */
CMB_API cmb_status cmb_feature_cache_init(void* workspace, size_t workspace_bytes,
                                          int64_t num_nodes, int64_t capacity, int64_t max_rows,
                                          int64_t max_edges, void* stream);
/* a4 + a5 of a sampled batch through the cache: misses are copied from host_x into the cache,
 * then the fused gather + aggregate reads every row from HBM.  Results are byte-identical to
 * cmb_gather_aggregate on the host table.  batch_tag: distinct for consecutive calls, never
 * 0xFFFFFFFF.  stats: NULL or device int64[2], incremented by (rows of the batch, misses). */
CMB_API cmb_status cmb_cache_gather_aggregate(const cmb_graph* g, const cmb_blocks* blocks,
                                              int32_t n_hops, int64_t n_last_dst_cap,
                                              int64_t nodes_cap, const cmb_feature_cache* cache,
                                              int32_t feat_dim, uint32_t batch_tag, float* x_in,
                                              int64_t x_in_ld, float* h_out, int64_t h_ld,
                                              int64_t* stats, void* stream);

/* ------------------------------------------------------------------ NEXT-1: one-sided gather */
/* the same a4 + a5 as cmb_gather_aggregate, but feature row v is read
 * from shards[v / rows_per_shard] at row v % rows_per_shard (row stride shard_ld floats):
 * with the peers' shards mapped into this process (cmb_ipc_open) the kernel reads remote rows
 * over NVLink itself -- the exchange is fused into the gather, no staging and no all-to-all.
 * shards: HOST array of `world` (<= 8) device pointers, 16-B aligned; rows_per_shard * world
 * must cover num_nodes; feat_dim columns are gathered.  Results are byte-identical to
 * cmb_gather_aggregate on the concatenated table.  blocks->new_src_mask and last_src_ids are
 * required (filled by cmb_sample_blocks). */
CMB_API cmb_status cmb_gather_aggregate_sharded(const cmb_graph* g, const cmb_blocks* blocks,
                                                int32_t n_hops, int64_t n_last_dst_cap,
                                                int64_t nodes_cap, const float* const* shards,
                                                int32_t world, int64_t rows_per_shard,
                                                int64_t shard_ld, int32_t feat_dim, float* x_in,
                                                int64_t x_in_ld, float* h_out, int64_t h_ld,
                                                void* stream);
/* CUDA IPC export of the allocation holding dev_ptr: writes the 64-byte handle to `handle`
 * (caller-owned, >= 64 bytes) and dev_ptr's byte offset inside the allocation. */
CMB_API cmb_status cmb_ipc_export(const void* dev_ptr, void* handle, uint64_t* offset);
/* Maps a peer process's exported allocation: *dev_ptr = mapped base + offset, *base = the
 * mapped base (pass it to cmb_ipc_close).  Fails (CMB_ERR_CUDA) in the exporting process. */
CMB_API cmb_status cmb_ipc_open(const void* handle, uint64_t offset, void** dev_ptr, void** base);
CMB_API cmb_status cmb_ipc_close(void* base);

/* ------------------------------------------------------------------ NEXT-4: first SAGE layer */
/* SURVEY.md 8(f) NEXT-4, reading R26: the input-side GraphSAGE-mean layer of the
 * model the paper trains (Eq. (1), in the GraphSAGE form of its footnote,
 * P:501; 3-layer GraphSAGE, hidden dim 256), fused with a4 + a5:
 *     Y[d, :] = sigma( X[nodes[d]] W_self + H[d] W_neigh + bias ),   d < n_{L-1},
 * H = the a5 mean of hop L-1 (neighbours only, R12), sigma = ReLU if relu else identity.
 * Operands are rounded to bf16, products accumulate in fp32 on the tensor cores (tcgen05, TMEM);
 * H and X_in are never written.  Accuracy: |Y - exact| <= 2^-7 * (|X_dst||W_self| + |H||W_neigh|
 * + |b|) (+ 2^-8 |Y| for a bf16 output), see R26.
 *
 * cmb_sage_weights_bytes: size of the packed weight image for feat_dim F (1..128) and out_dim Fo
 * (16..256, a multiple of 16); 0 if unsupported.
 * cmb_sage_pack_weights: w_self, w_neigh = device fp32 [F x Fo] row-major (Y = X W); writes the
 * bf16 image (device, caller-owned, 16-B aligned, >= cmb_sage_weights_bytes) in the tensor
 * cores' K-major 128-byte-swizzled operand layout.  Pack once per weight update.
 * cmb_sage_layer_forward: reads the feature table of g (feat_dim <= 128, ld % 4 == 0) through
 * blocks (filled by cmb_sample_blocks; last_src_ids required), w_img (packed for g's F and
 * out_dim), bias (device fp32 [Fo] or NULL); writes out (device, fp32 if out_bf16 == 0 else
 * bf16, row stride out_ld elements >= Fo, rows 16-B aligned) for d < the device count
 * n_{L-1} <= n_last_dst_cap.  One persistent CTA per SM (~197 KB shared memory, 256 TMEM
 * columns).  Host-checkable errors return CMB_ERR_INVALID_ARGUMENT. */
CMB_API size_t cmb_sage_weights_bytes(int32_t feat_dim, int32_t out_dim);
CMB_API cmb_status cmb_sage_pack_weights(const float* w_self, const float* w_neigh,
                                         int32_t feat_dim, int32_t out_dim, void* w_img,
                                         size_t w_img_bytes, void* stream);
CMB_API cmb_status cmb_sage_layer_forward(const cmb_graph* g, const cmb_blocks* blocks,
                                          int32_t n_hops, int64_t n_last_dst_cap,
                                          const void* w_img, const float* bias, int32_t out_dim,
                                          int32_t relu, int32_t out_bf16, void* out,
                                          int64_t out_ld, void* stream);

/* NEXT-4 GCN variant (reading R28): Y = sigma(A' X_in W + bias) on the input-side block,
 * A' = (D + I)^-1 (A + I) (row-normalised adjacency with a self loop, Eq. (1)), fused
 * with the gather like cmb_sage_layer_forward (same arguments and limits; one weight matrix
 * w = device fp32 [F x Fo] row-major, packed by cmb_gcn_pack_weights into a half-size image). */
CMB_API size_t cmb_gcn_weights_bytes(int32_t feat_dim, int32_t out_dim);
CMB_API cmb_status cmb_gcn_pack_weights(const float* w, int32_t feat_dim, int32_t out_dim,
                                        void* w_img, size_t w_img_bytes, void* stream);
CMB_API cmb_status cmb_gcn_layer_forward(const cmb_graph* g, const cmb_blocks* blocks,
                                         int32_t n_hops, int64_t n_last_dst_cap,
                                         const void* w_img, const float* bias, int32_t out_dim,
                                         int32_t relu, int32_t out_bf16, void* out,
                                         int64_t out_ld, void* stream);
/* Its weight gradients (reading R35; the chain rule on Eq. (1)):
 * dZ = dY * 1[Y > 0] (y = the forward's bf16 output, or NULL for an identity layer),
 * dW = (A' X_in)^T dZ -> dw fp32 [F x Fo] row-major, db = sum_d dZ[d] -> db fp32 [Fo].  The
 * aggregate rows are rebuilt from the feature table exactly as the forward builds them (bf16),
 * the products accumulate in fp32 on the tensor cores per CTA and the CTA partials are summed
 * in fp64 in a fixed order (deterministic).  Arguments, limits and workspace
 * (cmb_sage_backward_workspace_bytes) as cmb_sage_layer_backward. */
CMB_API cmb_status cmb_gcn_layer_backward(const cmb_graph* g, const cmb_blocks* blocks,
                                          int32_t n_hops, int64_t n_last_dst_cap, const void* dy,
                                          int64_t dy_ld, int32_t dy_f32, const void* y,
                                          int64_t y_ld, int32_t out_dim, float* dw, float* db,
                                          void* workspace, size_t workspace_bytes, void* stream);

/* NEXT-4 for wide feature rows (F > 128: Reddit's F = 602), where the fused layer
 * cannot keep K = 2F resident: the same layer (reading R26) and weight gradients (reading R27)
 * computed from the a4 + a5 outputs of cmb_gather_aggregate, x_dst = X_in (rows < n = n_dev[0]
 * <= n_rows_cap, ld x_ld) and h = H (ld h_ld), fp32 device.  Operands are rounded to bf16 (as in
 * the fused layer, same bounds), the two dense products run as cuBLASLt bf16 GEMMs with fp32
 * accumulation (the library's only library GEMM), packing / bias / ReLU / mask / dW unpack /
 * fixed-order db are this library's kernels.
 *   cmb_sage_dense_pack_weights: w_self, w_neigh fp32 [F x Fo] row-major -> the bf16 image
 *     (cmb_sage_dense_weights_bytes; Fo a multiple of 8).
 *   cmb_sage_dense_forward: out[r] = sigma(x_dst[r] W_self + h[r] W_neigh + bias) for r < n
 *     (bf16 or fp32, ld out_ld), rows n .. n_rows_cap zero.
 *   cmb_sage_dense_backward: dZ = dY * 1[Y > 0] (y = the forward's bf16 output; NULL = identity),
 *     dw fp32 [2][F][Fo] = (X_dst^T dZ, H^T dZ), db fp32 [Fo] = sum_r dZ[r] (fp64, fixed order).
 * workspace: cmb_sage_dense_workspace_bytes(n_rows_cap, F, Fo) bytes, 256-B aligned, caller owned
 * (it holds the bf16 operand image, the fp32 product, dZ and cuBLASLt's scratch). */
CMB_API size_t cmb_sage_dense_weights_bytes(int32_t feat_dim, int32_t out_dim);
CMB_API size_t cmb_sage_dense_workspace_bytes(int64_t n_rows_cap, int32_t feat_dim,
                                              int32_t out_dim);
CMB_API cmb_status cmb_sage_dense_pack_weights(const float* w_self, const float* w_neigh,
                                               int32_t feat_dim, int32_t out_dim, void* w_img,
                                               size_t w_img_bytes, void* stream);
CMB_API cmb_status cmb_sage_dense_forward(const float* x_dst, int64_t x_ld, const float* h,
                                          int64_t h_ld, const int64_t* n_dev, int64_t n_rows_cap,
                                          int32_t feat_dim, const void* w_img, const float* bias,
                                          int32_t out_dim, int32_t relu, int32_t out_bf16,
                                          void* out, int64_t out_ld, void* workspace,
                                          size_t workspace_bytes, void* stream);
CMB_API cmb_status cmb_sage_dense_backward(const float* x_dst, int64_t x_ld, const float* h,
                                           int64_t h_ld, const int64_t* n_dev,
                                           int64_t n_rows_cap, int32_t feat_dim, const void* dy,
                                           int64_t dy_ld, int32_t dy_f32, const void* y,
                                           int64_t y_ld, int32_t out_dim, float* dw, float* db,
                                           void* workspace, size_t workspace_bytes, void* stream);

/* NEXT-4 hidden layers (reading R29): layer l >= 2 of the model on hop h = L - l:
 *     Y[d] = sigma( Yp[d] W_self + mean_{e in row d of hop h} Yp[indices[h][e]] W_neigh + b ),
 * d < n_h (device count blocks->sizes[h] <= n_dst_cap).  y_prev: device bf16 [n_{h+1} x in_dim]
 * (the previous layer's output, row = local src id of hop h), row stride y_prev_ld (multiple of
 * 8, 16-B aligned); in_dim in {64, 128, 192, 256}; w_img packed by cmb_sage_hidden_pack_weights
 * (w_self, w_neigh device fp32 [in_dim x out_dim]); out as for cmb_sage_layer_forward.  bf16
 * operands, fp32 accumulation; the mean is summed in fp32 in CSR order. */
CMB_API size_t cmb_sage_hidden_weights_bytes(int32_t in_dim, int32_t out_dim);
CMB_API cmb_status cmb_sage_hidden_pack_weights(const float* w_self, const float* w_neigh,
                                                int32_t in_dim, int32_t out_dim, void* w_img,
                                                size_t w_img_bytes, void* stream);
CMB_API cmb_status cmb_sage_hidden_forward(const cmb_blocks* blocks, int32_t hop,
                                           int64_t n_dst_cap, const void* y_prev,
                                           int64_t y_prev_ld, int32_t in_dim, const void* w_img,
                                           const float* bias, int32_t out_dim, int32_t relu,
                                           int32_t out_bf16, void* out, int64_t out_ld,
                                           void* stream);

/* NEXT-4 aggregation backward (reading R30, the "transposed-block scatter-add"):
 *     dX[indices[e], :] += dH[d, :] / deg_d   for every edge e of row d < *n_dst_dev,
 * i.e. dX += M^T dH for the mean H = M X of cmb_sage_mean_aggregate.  ADDS into dx (zero it, or
 * pass a buffer that already holds the self path's gradient).  dh: device fp32 [n_dst x ld];
 * dx: device fp32 [n_src x ld]; rows 16-B aligned (ld % 4 == 0); columns >= feat_dim untouched.
 * fp32 vector reductions in no fixed order: |error| <= (c_s + 2) 2^-24 (M^T |dH|)[s]. */
CMB_API cmb_status cmb_sage_mean_backward(const int32_t* indptr, const int32_t* indices,
                                          const int64_t* n_dst_dev, int64_t n_dst_cap,
                                          const float* dh, int64_t dh_ld, int32_t feat_dim,
                                          float* dx, int64_t dx_ld, void* stream);

/* NEXT-4 backward (reading R27): weight gradients of the same layer for one batch,
 *     dZ = dY * 1[Y > 0] (y != NULL; y = NULL: dZ = dY),
 *     dW_self = X_dst^T dZ,  dW_neigh = H^T dZ,  db = sum_d dZ[d, :],
 * with [X_dst | H] recomputed from the feature table exactly as the forward builds it (bf16
 * operands, fp32 accumulation on the tensor cores per CTA, fp64 sum of the per-CTA partials:
 * deterministic).  dy: device [n_{L-1} x out_dim], bf16 (dy_f32 = 0) or fp32 (dy_f32 = 1:
 * e.g. cmb_sage_hidden_input_grad's dX, rounded to bf16 as it is staged); y: device bf16; row
 * strides dy_ld / y_ld elements (16-B aligned rows).  dw: device fp32 [2 x F x out_dim] (dW_self then dW_neigh,
 * row-major like the forward's W); db: device fp32 [out_dim].  out_dim: a power of two in
 * [16, 256]; F <= 128.  workspace: device, >= cmb_sage_backward_workspace_bytes (partials).
 * Accuracy: |dW - exact| <= 2^-7 * |A|^T |dZ|, |db - exact| <= 2^-12 * sum |dZ| (R27). */
CMB_API size_t cmb_sage_backward_workspace_bytes(int32_t feat_dim, int32_t out_dim);
CMB_API cmb_status cmb_sage_layer_backward(const cmb_graph* g, const cmb_blocks* blocks,
                                           int32_t n_hops, int64_t n_last_dst_cap,
                                           const void* dy, int64_t dy_ld, int32_t dy_f32,
                                           const void* y, int64_t y_ld, int32_t out_dim,
                                           float* dw, float* db,
                                           void* workspace, size_t workspace_bytes, void* stream);

/* NEXT-4 forward with the A tile saved for the backward ("saved operand"):
 * cmb_sage_layer_forward that also writes every 128-row tile's operand image [X_dst | H] (bf16,
 * the tensor cores' K-major 128-B-swizzled layout, rows past n_{L-1} zero) to a_save with the TMA
 * engine while the MMAs run; cmb_sage_layer_backward_saved then loads those images (one bulk
 * copy per tile) instead of re-gathering the feature rows -- same arithmetic, same results, bit
 * for bit.  a_save: device, >= cmb_sage_saved_a_bytes(F, n_last_dst_cap) bytes (64 KB per tile
 * at F <= 128), 16-B aligned, caller-owned; valid until the next forward on it.  The SAGE form
 * only (not GCN). */
CMB_API size_t cmb_sage_saved_a_bytes(int32_t feat_dim, int64_t n_last_dst_cap);
CMB_API cmb_status cmb_sage_layer_forward_save(const cmb_graph* g, const cmb_blocks* blocks,
                                               int32_t n_hops, int64_t n_last_dst_cap,
                                               const void* w_img, const float* bias,
                                               int32_t out_dim, int32_t relu, int32_t out_bf16,
                                               void* out, int64_t out_ld, void* a_save,
                                               size_t a_save_bytes, void* stream);
CMB_API cmb_status cmb_sage_layer_backward_saved(const cmb_graph* g, const cmb_blocks* blocks,
                                                 int32_t n_hops, int64_t n_last_dst_cap,
                                                 const void* a_saved, size_t a_saved_bytes,
                                                 const void* dy, int64_t dy_ld, int32_t dy_f32,
                                                 const void* y, int64_t y_ld, int32_t out_dim,
                                                 float* dw, float* db, void* workspace,
                                                 size_t workspace_bytes, void* stream);

/* NEXT-4 hidden-layer backward (reading R31 = R27 applied to the R29 layer): weight
 * gradients of a layer >= 2 on hop `hop` of the blocks, whose input is the previous layer's
 * bf16 output y_prev (rows = local src ids of the hop, the dst rows d < n_hop its prefix):
 *     dZ = dY * 1[Y > 0] (y != NULL; y = NULL: dZ = dY),
 *     dW_self = y_prev[0:n_dst]^T dZ,  dW_neigh = H^T dZ,  db = sum_d dZ[d, :],
 * H = the neighbour means exactly as cmb_sage_hidden_forward builds them (fp32 sum in CSR order
 * times RN(1/deg), rounded to bf16).  bf16 operands, fp32 accumulation per CTA on the tensor
 * cores, fp64 sum of the per-CTA partials (deterministic).  y_prev: device bf16 [n_src x ld]
 * (ld % 8 == 0, ld >= in_dim, 16-B aligned); dy: device [n_dst x ld], bf16 or (dy_f32 = 1) fp32
 * rounded to bf16 as it is staged; y: device bf16 [n_dst x ld] (16-B aligned rows, ld >= out_dim); dw: device fp32 [2 x in_dim x out_dim] (dW_self then dW_neigh, row-major like W);
 * db: device fp32 [out_dim].  in_dim in {64, 128, 192, 256}; out_dim a power of two in
 * [16, 256].  workspace: device, >= cmb_sage_hidden_backward_workspace_bytes (partials; the
 * library never allocates).  n_dst = min(sizes[hop], n_dst_cap).  dz_out (optional, NULL to
 * skip): device bf16 [n_dst x dz_ld] receives the masked dZ (bit-exact dY * 1[Y > 0]), the
 * operand of cmb_sage_hidden_input_grad -- written by the same kernel, no extra pass.
 * Host-checked errors return CMB_ERR_INVALID_ARGUMENT before any launch.
 * Accuracy: |dW - exact| <= 2^-7 * |A|^T |dZ|, |db - exact| <= 2^-12 * sum |dZ| (R31). */
CMB_API size_t cmb_sage_hidden_backward_workspace_bytes(int32_t in_dim, int32_t out_dim);
CMB_API cmb_status cmb_sage_hidden_backward(const cmb_blocks* blocks, int32_t hop,
                                            int64_t n_dst_cap, const void* y_prev,
                                            int64_t y_prev_ld, int32_t in_dim, const void* dy,
                                            int64_t dy_ld, int32_t dy_f32, const void* y,
                                            int64_t y_ld,
                                            int32_t out_dim, float* dw, float* db,
                                            void* workspace, size_t workspace_bytes,
                                            void* dz_out, int64_t dz_ld, void* stream);

/* NEXT-4 hidden-layer input gradient (reading R32): the gradient that flows into the
 * layer's input Yp (the previous layer's output) through both of its paths,
 *     dX = P^T (dZ W_self^T) + M^T (dZ W_neigh^T),
 * P = the dst-prefix selection (dX[d] gets dZ[d] W_self^T for d < n_dst) and M^T = the
 * transposed-block scatter of cmb_sage_mean_backward (dX[idx[e]] += dH[d] / deg_d).  Three
 * launches: the tensor-core layer kernel in its self-only form twice (A = dZ, B = the packed
 * W_self^T, then W_neigh^T; fp32 out: dX rows < n_dst, dH), then the scatter into dX.
 * wt_img: cmb_sage_hidden_pack_weights_t of the layer's W_self, W_neigh ([in_dim x out_dim]
 * fp32 row-major, as for the forward), cmb_sage_hidden_weights_t_bytes bytes.
 * dz: device bf16 [n_dst x dz_ld], dz_ld >= out_dim rounded up to 64, columns out_dim.. zero
 * (cmb_sage_hidden_backward's dz_out).  dx: device fp32 [n_src_cap x dx_ld], OVERWRITTEN (zeroed
 * first); dh: device fp32 scratch [n_dst_cap x dh_ld].  ld % 4 == 0, 16-B aligned.
 * in_dim in [16, 256] a multiple of 16; out_dim in [1, 256].
 * Accuracy: |dX - exact| <= 2^-7 * (P^T |dZ||W_self|^T + M^T |dZ||W_neigh|^T) (R32). */
CMB_API size_t cmb_sage_hidden_weights_t_bytes(int32_t in_dim, int32_t out_dim);
CMB_API cmb_status cmb_sage_hidden_pack_weights_t(const float* w_self, const float* w_neigh,
                                                  int32_t in_dim, int32_t out_dim, void* wt_img,
                                                  size_t wt_img_bytes, void* stream);
CMB_API cmb_status cmb_sage_hidden_input_grad(const cmb_blocks* blocks, int32_t hop,
                                              int64_t n_dst_cap, int64_t n_src_cap,
                                              const void* dz, int64_t dz_ld, int32_t out_dim,
                                              const void* wt_img, int32_t in_dim, float* dx,
                                              int64_t dx_ld, float* dh, int64_t dh_ld,
                                              void* stream);

/* NEXT-4 loss (reading R33; "minimizing the loss between the labels
 * ... and the node embeddings of the last layer"): softmax cross-entropy of the last layer's
 * logits, mean over the batch's n = min(*n_dev, n_cap) roots (the prefix of `nodes`):
 *     *loss = (1/n) sum_i [ logsumexp(Y[i, 0:C]) - Y[i, label_i] ],  label_i = node_labels[nodes[i]],
 *     dY[i, c] = (softmax(Y[i])_c - 1[c == label_i]) / n  (bf16; columns C .. dy_cols-1 = 0).
 * logits: device fp32 [n x ld]; node_labels: device int32 [N]; nodes: the batch's node list
 * (device); n_dev: device int64 (cmb_blocks sizes[0]); dy: device bf16 [n x dy_ld]; loss:
 * device fp64 scalar (per-root terms in row_loss, device fp64 scratch [n_cap], summed in a fixed
 * order by a second launch: deterministic); dy_cols <= 256; status: device int32 word or
 * NULL, set to CMB_ERR_INVALID_ARGUMENT if a label is outside [0, C) (that row is skipped).
 * 1 <= C <= 256.  Accuracy (fp32 softmax): |dY - exact| <= 2^-8 |dY| + 2^-20 / n,
 * |loss - exact| <= 2^-20 * mean_i (|max_c Y[i, c]| + 1). */
CMB_API cmb_status cmb_softmax_xent(const float* logits, int64_t ld, const int32_t* node_labels,
                                    const int32_t* nodes, const int64_t* n_dev, int64_t n_cap,
                                    int32_t num_classes, void* dy, int64_t dy_ld, int32_t dy_cols,
                                    double* loss, double* row_loss, int32_t* status,
                                    void* stream);

/* NEXT-4 optimizer step (reading R34; DGL's GraphSAGE defaults, lr 1e-3,
 * weight decay 5e-4 -- Adam in that example): on n fp32 parameters (flat, device, 16-B aligned,
 * n % 4 == 0), with the step's gradient g and the moment buffers m, v (zero before step 1):
 *     g' = g + wd w;  m = b1 m + (1 - b1) g';  v = b2 v + (1 - b2) g'^2;
 *     w -= lr (m / (1 - b1^step)) / (sqrt(v / (1 - b2^step)) + eps).
 * Hyper-parameters in fp64: 1 - beta and the bias corrections are formed in fp64 and rounded
 * once (1 - 0.999f would be off by 1.3e-5).  Updates w, m, v in place.  fp32 arithmetic: |w - exact| <= 2^-22 |w| + 2^-18 lr (|u| + 1),
 * u the exact update direction. */
CMB_API cmb_status cmb_adam_step(float* w, const float* g, float* m, float* v, int64_t n,
                                 double lr, double beta1, double beta2, double eps,
                                 double weight_decay, int32_t step, void* stream);

/* One GraphSAGE layer's slice of the flat parameter buffer and its bf16 operand images, for
 * cmb_adam_step_pack: parameters [offset, offset + 2 in_dim out_dim + out_dim) of the buffer are
 * [W_self | W_neigh | b] (row-major [in_dim x out_dim] each); img: the forward weight image
 * (cmb_sage_pack_weights / cmb_sage_hidden_pack_weights layout, kh = ceil(in_dim / 64));
 * img_t: NULL or the transposed image of cmb_sage_hidden_pack_weights_t (kt = ceil(out_dim/64)).
 * dense = 1: img is a cmb_sage_dense_pack_weights image instead (wide first layer, in_dim may
 * exceed 256; img_t must be NULL). */
typedef struct {
  int64_t offset;
  int32_t in_dim, out_dim;
  void* img;
  void* img_t;
  int32_t dense;
} cmb_layer_pack;

/* cmb_adam_step fused with the repack of the updated weights: every W element is written, as
 * bf16, into its layer's forward image and (img_t != NULL) its transposed image in the same pass
 * -- one launch instead of one Adam launch plus one packer launch per image.  The images'
 * padding (columns >= in_dim / out_dim) must already be zero (it is never written).  n_layers
 * <= 8; layers must tile [0, n) in order. */
CMB_API cmb_status cmb_adam_step_pack(float* w, const float* g, float* m, float* v, int64_t n,
                                      double lr, double beta1, double beta2, double eps,
                                      double weight_decay, int32_t step,
                                      const cmb_layer_pack* layers, int32_t n_layers,
                                      void* stream);
/* The same with the step number on the DEVICE: `step` (device int32) is advanced by one on the
 * stream, then read by the update, which forms the bias corrections from it in fp64 -- nothing
 * step-dependent is baked into the launches, so a captured CUDA graph of a whole training step
 * can be replayed (GraphSAGE.train_step(graph=True)).  Same arithmetic as cmb_adam_step_pack. */
CMB_API cmb_status cmb_adam_step_pack_dev(float* w, const float* g, float* m, float* v,
                                          int64_t n, double lr, double beta1, double beta2,
                                          double eps, double weight_decay, int32_t* step,
                                          const cmb_layer_pack* layers, int32_t n_layers,
                                          void* stream);

/* ------------------------------------------------------------------ status */
/* Synchronises `stream`, returns (and clears) the sticky device status word of a
 * graph / order / sample workspace. */
CMB_API cmb_status cmb_get_device_status(void* workspace, void* stream);
CMB_API const char* cmb_status_string(cmb_status s);
CMB_API const char* cmb_last_error_message(void);
CMB_API int cmb_version(void); /* major * 100 + minor */

#ifdef __cplusplus
}
#endif
#endif /* CMB_H_ */
