/*
 * jz_knn.h -- C ABI of the B200-native jz-tree exact kNN hot path.
 *
 * Problem ("N separate source and query points ... float32",
 * L453 "query points equal to the source points", L454 "periodic wrapping in
 * the distance calculation"; BASELINE.json north_star): given N points in 3-D
 * (FP32), an optional periodic box and k, return for every point the k nearest
 * points (itself included) as global indices and squared distances, ordered by
 * (d2, index) ascending. The result is the unique exact answer under the
 * canonical FP32 distance (R1-R3):
 *     t_d = RN(q_d - s_d); periodic: t_d >= L_d/2 -> RN(t_d - L_d),
 *                                    t_d < -L_d/2 -> RN(t_d + L_d);
 *     d2  = fmaf(t_z, t_z, fmaf(t_y, t_y, t_x * t_x)).
 *
 * Method (§2-§3): Morton (z-order) sort with 21-bit-per-axis keys,
 * plane-based tree hierarchy, dual tree walk NodeToNode per plane
 * (Alg. 1-3) and LeafToLeaf. All steps run in sm_100a
 * CUDA kernels; there is no CPU fallback.
 *
 * Conventions
 *  - Pointers are CUDA DEVICE pointers unless marked (host).
 *  - Calls are ordered on the given stream (jz_stream_t == cudaStream_t; NULL =
 *    legacy default stream). build/query synchronise the stream internally a few
 *    times to read data-dependent sizes; outputs are complete when they return.
 *  - Every int-returning call returns JZ_OK (0) or an error code; on error no
 *    output is written and jz_last_error() returns a thread-local message.
 *  - Thread safety: one index must not be used by two threads at once; distinct
 *    indices are independent.
 */
#ifndef JZ_KNN_H
#define JZ_KNN_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#if defined(__GNUC__)
#define JZ_API __attribute__((visibility("default")))
#else
#define JZ_API
#endif

typedef struct CUstream_st *jz_stream_t; /* same type as cudaStream_t */
typedef struct jz_knn_index jz_knn_index;  /* opaque; owns all its device memory */
typedef struct jz_comm jz_comm;            /* opaque communicator of the multi-GPU path (one rank per GPU) */
typedef struct jz_comm_world jz_comm_world; /* opaque in-process world of logical ranks (tests) */

enum {
  JZ_OK = 0,
  JZ_EINVAL = 2,    /* bad argument (n < 1, k < 1, k > number of sources, bad box, bad order, NULL pointer) */
  JZ_EDATA = 3,     /* NaN / Inf coordinate, or periodic coordinate outside [0, L) */
  JZ_ECAPACITY = 4, /* reserved: internal capacities grow on demand */
  JZ_ECUDA = 5,     /* CUDA runtime error (message in jz_last_error) */
  JZ_ENCCL = 6,     /* NCCL error, or libnccl.so.2 not loadable (message in jz_last_error) */
  JZ_ENOMEM = 7     /* device allocation failed */
};

enum { JZ_ORDER_INPUT = 0, JZ_ORDER_Z = 1 };

enum {
  JZ_FLAG_FRAME = 1u << 0,         /* use frame_origin / frame_extent for the Morton keys (multi-GPU: one global frame) */
  JZ_FLAG_NO_EARLY_EXIT = 1u << 1, /* disable the sorted-r_low early exit (pruning-safety tests) */
  JZ_FLAG_NO_SEGSORT = 1u << 2,    /* do not sort interaction segments by r_low (implies no early exit) */
  JZ_FLAG_QBOX_DIAG = 1u << 3      /* jz_knn_query_boxes: R_max = AABB diagonal of the smallest ancestor
                                      holding k points instead of the NodeToNode walk (no walk, but far
                                      looser on clustered data: measured 7x more ghosts) */
};

/* Tree / walk parameters. Zero fields take the defaults (nmax0 see DESIGN.md §6). */
typedef struct {
  int32_t nmax0;   /* N_max^(0), leaf capacity; 0 => 80 (paper: 48, tuned for its kernels). Range 1..128 */
  int32_t coarsen; /* c, N_max^(p) = N_max^(0) c^p; 0 => 16 (paper: 8, tuned for its kernels). >= 2 */
  int32_t ntarget; /* N_target: build plane p >= 1 iff 2N / N_max^(p) >= N_target; 0 => 30 (paper: ~1000) */
  int32_t ngr;     /* NGR, top nodes per super node; 0 => 32 */
  uint32_t flags;  /* JZ_FLAG_* */
  float frame_origin[3]; /* with JZ_FLAG_FRAME: key frame origin (open boundary) */
  float frame_extent;    /* with JZ_FLAG_FRAME: key frame edge length (> 0) */
  int32_t reg_fmax;      /* regularisation f_max: 0 => off; > 0 => every plane also splits
                            the gaps whose Morton level exceeds lvl_max^(p), 2^lvl_max <= f_max V_90%^(p)
                            (paper: f_max ~ 50). Structure only: results are identical either way. */
  int32_t reserved[3];
} jz_knn_params;

/*
 * Build the tree over n points.
 *   pos   [n][3] float, xyz row-major (device). The index copies what it needs;
 *         pos may be freed once the call returns.
 *   box   (host) [3] periodic box lengths L_d > 0, or NULL for open boundaries.
 *         Periodic coordinates must satisfy 0 <= x_d < L_d (else JZ_EDATA).
 *   p     (host) parameters or NULL for defaults.
 *   out   (host) receives the new index (caller frees with jz_knn_free).
 * Global index of point i = i. All n points are queries.
 */
JZ_API int jz_knn_build(const float *pos, int64_t n, const float *box, const jz_knn_params *p, jz_stream_t s,
                 jz_knn_index **out);

/*
 * Build over points that carry their global index: pts4[i] = {x, y, z, bits(gidx)}
 * (device, float4, gidx an int32 stored bitwise in .w). Point types (PAPER.md L272-279
 * "Multiple point types": one tree built jointly over all types, then type-specific
 * z-ordered arrays with per-type leaf splits):
 *   - query  iff its input position i < n_query (row i of the result);
 *   - source iff gidx >= 0 (a neighbour candidate, reported as gidx).
 * Points [n_query, n) with gidx >= 0 are sources only (multi-GPU ghosts, DESIGN.md
 * "Multi-GPU"); points with gidx < 0 are queries only. Node counts of the walk count
 * sources. jz_knn_rows() returns n_query.
 */
JZ_API int jz_knn_build_xyzg(const float *pts4, int64_t n, int64_t n_query, const float *box, const jz_knn_params *p,
                      jz_stream_t s, jz_knn_index **out);

/*
 * Separate query points ("query the tree using a set of query points
 * x_query distinct from the source points x"):
 *   src [n_src][3], qry [n_qry][3] float (device, may be freed after the call).
 * Builds the joint tree (L276-279) over both sets. Row i of jz_knn_query answers
 * qry[i]; indices refer to src. n_src >= 1, n_qry >= 0, n_src + n_qry <= 2^31 - 2;
 * periodic: all coordinates in [0, L) (JZ_EDATA otherwise). With JZ_ORDER_Z,
 * out_row_gidx[r] = the query's row i.
 */
JZ_API int jz_knn_build_xq(const float *src, int64_t n_src, const float *qry, int64_t n_qry, const float *box,
                    const jz_knn_params *p, jz_stream_t s, jz_knn_index **out);

/* Number of result rows the index produces (host out). */
JZ_API int jz_knn_rows(const jz_knn_index *ix, int64_t *m);

/*
 * k nearest neighbours of every query point.
 *   k        1 <= k <= number of sources. k > k_max = 32 runs ceil(k/32) LeafToLeaf
 *            passes, pass c keeping only pairs after the last (d2, index) of pass c-1
 *            ("call the kernel multiple times if k > k_max, filtering
 *            additionally by a minimum radius R_min (and an equality breaking index
 *            offset)").
 *   order    JZ_ORDER_INPUT: row i belongs to query point i (input position; for
 *            jz_knn_build_xyzg: the i-th query point of pts4).
 *            JZ_ORDER_Z: rows in Morton order; out_row_gidx[r] names the point (its
 *            gidx if it is also a source, else its query row).
 *   out_idx  [m][k] int32 global indices (device)
 *   out_d2   [m][k] float canonical squared distances (device)
 *   out_row_gidx [m] int32 (device) or NULL; required for JZ_ORDER_Z.
 * The index is reusable for several queries (construction never depends on k).
 */
JZ_API int jz_knn_query(jz_knn_index *ix, int k, int order, int32_t *out_idx, float *out_d2, int32_t *out_row_gidx,
                 jz_stream_t s);

/* Release the index (synchronises its stream). NULL-safe. */
JZ_API void jz_knn_free(jz_knn_index *ix);

/*
 * End-to-end convenience on HOST buffers: copies pos_host to the device, builds,
 * queries, copies the rows back (input order), frees. pos_host [n][3],
 * idx_host [n][k], d2_host [n][k], 1 <= k <= n; pinned host memory gives full PCIe speed.
 */
JZ_API int jz_knn_search_host(const float *pos_host, int64_t n, const float *box, const jz_knn_params *p, int k,
                       int32_t *idx_host, float *d2_host, jz_stream_t s);

/*
 * End to end on HOST buffers with the rows in z order (the multi-GPU paper output form)
 * and streamed: LeafToLeaf runs in 16 chunks of work items (contiguous z-order row ranges) and
 * each finished chunk is copied to the host on a second stream while the next one runs, so the
 * device-to-host transfer overlaps the walk (k > 32: one copy at the end). Row r of idx_host /
 * d2_host [n][k] belongs to input point row_gidx_host[r] ([n]). Same errors as above.
 */
JZ_API int jz_knn_search_host_z(const float *pos_host, int64_t n, const float *box, const jz_knn_params *p, int k,
                                int32_t *idx_host, float *d2_host, int32_t *row_gidx_host, jz_stream_t s);

/*
 * Per-stage device timings (ms) of the last build + query on this index, for the
 * phase breakdown of PAPER.md Fig. knnsteps:
 *   [0] frame+validate [1] sort [2] tree build [3] node-to-node walk [4] leaf-to-leaf [5] total.
 * Also reports the number of (query, source) distance evaluations of the last query
 * in *evals (host, may be NULL). Timing is off unless JZ_TIMING=1 in the environment
 * or jz_set_timing(1) was called.
 */
JZ_API int jz_knn_stage_times(const jz_knn_index *ix, float out_ms[6], int64_t *evals);
JZ_API void jz_set_timing(int on);

/* Counters of the last query (host out[9]): [0] distance evaluations, [1] top-k insertions,
 * [2] number of leaves, [3] number of tree planes, LeafToLeaf: [4] candidate-log appends,
 * [5] top-k merge rounds (per warp), [6] log compactions (per warp), [7] leaves staged (per
 * warp), [8] 32-query work items. */
JZ_API int jz_knn_stats(const jz_knn_index *ix, int64_t out[9]);

/* Number of kernels this library has launched in the process so far. */
JZ_API int64_t jz_launch_count(void);

/* Thread-local description of the last error. */
JZ_API const char *jz_last_error(void);

/* ---------------------------------------------------------------------------
 * Multi-GPU exact kNN (§3.3 L388-393 distributed kNN; L112-114 sample-
 * splitter Morton-range partition; L458 z-order output).
 * One process (or thread) per rank, each with its own device and stream. Every
 * call below is COLLECTIVE: all ranks of the communicator must make it, in the
 * same order. The exchanges run inside the library on a jz_comm.
 * ------------------------------------------------------------------------- */

/* NCCL bootstrap, step 1 (rank 0 only): a 128-byte NCCL unique id (host) that the
 * caller broadcasts to the other ranks (e.g. with torch.distributed). libnccl.so.2
 * is opened at run time (dlopen); JZ_ENCCL if it cannot be loaded. */
JZ_API int jz_comm_unique_id(uint8_t id[128]);

/* NCCL bootstrap, step 2 (every rank): communicator of nranks (1..32) ranks on the
 * CURRENT CUDA device (ncclCommInitRank). *out is owned by the caller (jz_comm_free),
 * must outlive every index built on it. JZ_EINVAL on bad arguments, JZ_ENCCL from NCCL. */
JZ_API int jz_comm_init(const uint8_t id[128], int nranks, int rank, jz_comm **out);

/* In-process world of nranks (1..32) logical ranks sharing one device (tests and
 * single-GPU rehearsals of the multi-GPU path): each logical rank runs in its own
 * host thread with its own stream and gets its communicator from jz_comm_init_local.
 * Exchanges are device-to-device copies between the ranks' buffers. */
JZ_API int jz_comm_local_world(int nranks, jz_comm_world **out);

/* Communicator of logical rank `rank` of world w (w must outlive it). */
JZ_API int jz_comm_init_local(jz_comm_world *w, int rank, jz_comm **out);

/* rank and size (host) of a communicator. */
JZ_API int jz_comm_rank_size(const jz_comm *c, int32_t *rank, int32_t *size);

/* Release a communicator (NULL-safe; not collective for local worlds). */
JZ_API void jz_comm_free(jz_comm *c);

/* Release a local world after every communicator of it was freed (NULL-safe). */
JZ_API void jz_comm_world_free(jz_comm_world *w);

/* Distributed build (collective). This rank passes its slice of the global input:
 * pos [n][3] float32 (device; n may be 0), global ids gidx_base .. gidx_base+n-1 (the
 * slices of the ranks need not be contiguous for JZ_ORDER_Z; JZ_ORDER_INPUT needs
 * the slices contiguous and in rank order). Steps inside: validation (JZ_EDATA as
 * jz_knn_build) and one global key frame (open boundary: all-reduced bounding box,
 * P:L133), N_samp = min(1000, 16384 / R) keys sampled per rank, all-gathered,
 * sorted identically on every rank, R - 1 quantile splitters; Morton-range partition
 * (a key equal to a splitter goes to the upper rank), all-to-all-v of float4 {x, y, z,
 * bits(gidx)} rows; local tree over the received points. *out: an index of
 * this rank's received points, bound to comm (which must outlive it); free it with
 * jz_knn_free. JZ_EINVAL: no points on any rank, bad box or arguments. */
JZ_API int jz_knn_build_dist(jz_comm *comm, const float *pos, int64_t n, int64_t gidx_base, const float *box,
                             const jz_knn_params *p, jz_stream_t s, jz_knn_index **out);

/* Rows (host) that jz_knn_query_dist writes on this rank: JZ_ORDER_Z = the points
 * this rank received in the partition; JZ_ORDER_INPUT = n of its own input slice. */
JZ_API int jz_knn_rows_dist(const jz_knn_index *ix, int order, int64_t *m);

/* Distributed query (collective), exact for any 1 <= k <= total points: rows ordered
 * (d2, global index), self included, bit-identical to the single-GPU jz_knn_query
 * over the union. Steps inside: (1) walk over the local points: exact
 * local rows whose k-th d2 bounds the global k-th d2; (2) query boxes = the nodes of
 * the finest plane with <= 4096 nodes, radius^2 = the largest local k-th d2 inside,
 * all-gathered; (3) each rank sends every point within a peer box's radius (exact
 * point-box bound) with an all-to-all-v, and the boxes some point reached are
 * all-reduced; (4) only the queries of reached boxes are walked again over local +
 * ghost points and their rows replaced (P:L388-393 remote data). JZ_ORDER_Z: rows
 * [m][k] (m = jz_knn_rows_dist) in z order of this rank's points, out_row_gidx [m]
 * their global ids. JZ_ORDER_INPUT: rows [n][k] of the own input slice in
 * input order (reverse all-to-all-v); out_row_gidx optional.
 * out_idx int32 global ids, out_d2 float32 canonical d2 (device, caller-owned). */
JZ_API int jz_knn_query_dist(jz_knn_index *ix, int k, int order, int32_t *out_idx, float *out_d2,
                             int32_t *out_row_gidx, jz_stream_t s);

/* Counters / wall times (host) of this rank's last distributed build + query:
 * counts = {local points, ghost points received, queries walked twice, query boxes};
 * ms = {frame + partition, local build, local walk, boxes + ghosts + second walk,
 * reverse exchange, device-busy time of this logical rank accumulated since its
 * communicator was created (worlds made with JZ_LOCAL_SERIAL=1 run the ranks' device
 * work one rank at a time, so this is the uncontended per-rank time; 0 for NCCL)}. */
JZ_API int jz_knn_dist_stats(const jz_knn_index *ix, int64_t counts[4], double ms[6]);

/* ---------------------------------------------------------------------------
 * Multi-GPU stage entry points (per-rank compute on device buffers, used by
 * jz_knn_build_dist / jz_knn_query_dist and exposed for tests and tools).
 * ------------------------------------------------------------------------- */

/* Morton keys of n points in a given frame (origin[3], extent; periodic: pass the
 * box as origin 0 / extent per axis via box != NULL). keys: [n] uint64 (device). */
JZ_API int jz_morton_keys(const float *pos, int64_t n, const float *box, const float *origin, float extent,
                   uint64_t *keys, jz_stream_t s);

/* For each point, the destination rank r such that splitters[r-1] <= key < splitters[r]
 * (splitters sorted, nsplit = R - 1 entries), plus per-rank counts.
 *   dest [n] int32 (device), counts [R] int64 (device, overwritten). */
JZ_API int jz_bucket_by_splitters(const uint64_t *keys, int64_t n, const uint64_t *splitters, int32_t nsplit,
                           int32_t *dest, int64_t *counts, jz_stream_t s);

/* Stable pack of pos (xyz) + global index base+i into float4 rows grouped by dest rank:
 * out4 [n][4] (device), offsets [R] (device, exclusive prefix of counts). */
JZ_API int jz_pack_by_rank(const float *pos, int64_t n, int64_t gidx_base, const int32_t *dest, const int64_t *offsets,
                    int32_t nranks, float *out4, jz_stream_t s);

/* Number of nodes of a plane (plane < 0: the top plane; 0: leaves). */
JZ_API int jz_knn_plane_nodes(const jz_knn_index *ix, int plane, int64_t *nnodes);

/* Query boxes for ghost selection: for each node of `plane` (< 0: top plane), its AABB
 * and the largest R_max^2 of its leaves; R_max^2 bounds the canonical k-th neighbour d2
 * of every contained query point: FindRmax down to the leaf plane; with
 * JZ_FLAG_QBOX_DIAG the AABB diagonal (self d_up^2, exact R8 bound) of the smallest
 * ancestor-or-self node holding >= k points (no walk, looser).
 * boxes [nnodes][8] floats {lo.x, lo.y, lo.z, r2, hi.x, hi.y, hi.z, bits(rank)} (device). */
JZ_API int jz_knn_query_boxes(jz_knn_index *ix, int k, int plane, int rank, float *boxes, jz_stream_t s);

/* Ghost selection: mask[i] (i in the index's sorted point order) gets bit r set when a
 * query box of rank r != self_rank can reach point i (exact box bound d_low^2 <= r2,
 * leaf granularity). counts [nranks] int64 (device) = points flagged per rank.
 * boxes [nbox][8] as produced by jz_knn_query_boxes (all-gathered). nranks <= 32. */
JZ_API int jz_knn_select_ghosts(jz_knn_index *ix, const float *boxes, int64_t nbox, int self_rank, int32_t nranks,
                         int32_t *mask, int64_t *counts, jz_stream_t s);

/* Pack the flagged points (float4 {x, y, z, bits(gidx)}) by destination rank into
 * out4 at offsets [nranks] (device, exclusive prefix of the counts). */
JZ_API int jz_knn_pack_ghosts(jz_knn_index *ix, const int32_t *mask, int32_t nranks, const int64_t *offsets, float *out4,
                       jz_stream_t s);

/* F4 -- friends-of-friends (§5) on an index built over points that are both
 * sources and queries (jz_knn_build; JZ_EINVAL otherwise). Groups are the connected components
 * of the graph with an edge between two points iff their canonical FP32 d2 (as for kNN) is
 * <= RN32(r_link * r_link) (R21). The walk is the kNN dual walk with a fixed radius;
 * links go to a union-find over z positions with atomic compare-and-swap.
 *   labels [n] int32 (device, caller-owned): label of input row i = the smallest input index of
 *          its group (unique, so bit-comparable).
 *   *ngroups (host, may be NULL): number of groups with >= min_count points (paper 20).
 * The catalogue of those groups stays in the index until the next jz_fof / jz_knn_free.
 * Synchronises s. */
JZ_API int jz_fof(jz_knn_index *ix, float r_link, int32_t min_count, int32_t *labels, int64_t *ngroups, jz_stream_t s);
/* Copy the catalogue (device arrays of >= ngroups entries; JZ_ECAPACITY if cap < ngroups), in the
 * paper's group order (z order of each group's first point): label int32, count int32,
 * centre of mass float64 [g][3] (periodic: wrapped into [0, L)), inertia radius float64 (rms
 * distance to the centre). FP64 sums in nondeterministic order: last-bit differences between
 * runs. */
JZ_API int jz_fof_catalogue(const jz_knn_index *ix, int64_t cap, int32_t *label, int32_t *count, double *com,
                            double *rad, jz_stream_t s);

/* Group order of the last jz_fof: order [n] (device) = input rows in group order -- a
 * stable sort of the points by their group's root, so the groups (all groups, singletons
 * included) appear in z order of their roots and each group is a contiguous block internally in
 * z order. group_beg [ngroups_all + 1] (device, optional, caller sizes it n + 1) = start of each
 * block in order[], group_beg[ngroups_all] = n; *ngroups_all (host, optional). JZ_EINVAL before
 * any jz_fof on this index. Synchronises s. */
JZ_API int jz_fof_group_order(const jz_knn_index *ix, int32_t *order, int32_t *group_beg, int64_t *ngroups_all,
                              jz_stream_t s);

/* F2 -- multi-GPU rows in input order ("final reordering step": the
 * reverse all-to-all of the result). Step 1 (sender): the z-ordered rows of this rank
 * (idx [m][k] int32, d2 [m][k] float32, row_gidx [m] int32, from jz_knn_query with
 * JZ_ORDER_Z) are grouped by dest [m] int32 (the rank owning row_gidx: jz_bucket_by_splitters
 * with the input-slice bounds as splitters) at offsets [nranks] int64 (exclusive prefix of
 * the per-rank counts) into out [m][2k+1] int32 words: k indices, k d2 bit patterns, gidx.
 * All pointers device; the order inside a destination group is unspecified.
 * Step 2 (receiver, after the all-to-all-v): rows [m][2k+1] are written to out_idx /
 * out_d2 [n][k] at row gidx - gidx_base. JZ_EDATA if a gidx lies outside
 * [gidx_base, gidx_base + n) (nothing is guaranteed about the outputs then). Synchronises s. */
JZ_API int jz_pack_rows(const int32_t *idx, const float *d2, const int32_t *row_gidx, int64_t m, int32_t k,
                        const int32_t *dest, const int64_t *offsets, int32_t nranks, int32_t *out, jz_stream_t s);
JZ_API int jz_scatter_rows(const int32_t *rows, int64_t m, int32_t k, int64_t gidx_base, int64_t n, int32_t *out_idx,
                           float *out_d2, jz_stream_t s);

/* Introspection for stage tests (copies to HOST memory dst, returns bytes needed or -1):
 * what 0 sorted keys u64[n], 1 sorted float4 points [n], 2 perm i32[n] (sorted -> input),
 * 3 plane `plane` beg i32[nnodes+1], 4 plane boxes (32 B per node), 5 plane count (int64). */
JZ_API int64_t jz_knn_debug_copy(const jz_knn_index *ix, int what, int plane, void *dst, int64_t cap);

#ifdef __cplusplus
}
#endif
#endif /* JZ_KNN_H */
