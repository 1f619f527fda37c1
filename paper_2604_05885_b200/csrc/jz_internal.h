// jz_internal.h -- host-side structures of the CUDA path (index, planes, interaction lists).
#pragma once
#include <cstdint>
#include <functional>
#include <string>
#include <vector>

#include "../../include/jz_knn.h"
#include "jz_common.cuh"

typedef jz_knn_params jz_knn_params_t;



namespace jz {

// One tree plane (a set of nodes partitioning the points).
//   p = 0 (leaves): beg[i] = first point of leaf i (spl^(0)), beg[nnodes] = N.
//   p >= 1       : beg[i] = first child (a node of plane p-1) of node i (spl^(p) as positions
//                  in plane p-1's split array, P:L224 / Fig. 3 spl^(1) = {0,2,4,5}).
struct Plane {
  int64_t nnodes = 0;
  int64_t nmax = 0;
  int32_t *beg = nullptr;     // [nnodes + 1] (device)
  int32_t *leafspl = nullptr; // [nnodes + 1] index into the leaf split array (device); p = 0: identity
  NodeBox *box = nullptr;     // [nnodes] (device)
  int lvl_max = -1;           // regularisation level bound of the plane, -1 = off
};

struct Stage {
  cudaEvent_t ev[8] = {};
  bool on = false;
};

}  // namespace jz

// the index behind the C ABI's opaque jz_knn_index (jz_api.cu; multi-GPU fields: jz_dist.cu)
struct jz_knn_index {
  cudaStream_t st = nullptr;
  int64_t n = 0, n_query = 0, n_src = 0;
  jz::Dom D{};
  jz_knn_params prm{};
  float4 *pts = nullptr;     // all points, z order (.w = gidx; < 0: query-only point)
  uint64_t *keys = nullptr;
  int32_t *perm = nullptr;   // z position -> input position
  // type-separated views: alias pts / leaf beg / perm when every point is both
  float4 *spts = nullptr, *qpts = nullptr;
  int32_t *sbeg = nullptr, *qbeg = nullptr, *qin = nullptr;
  bool own_s = false, own_q = false;
  bool input_ids = false;  // point ids are input positions 0..n-1 (jz_knn_build): needed by jz_fof
  std::vector<jz::Plane> planes;
  cudaEvent_t ev[8] = {};
  bool timing = false;
  float times[6] = {0, 0, 0, 0, 0, 0};
  long long evals = 0, inserts = 0;
  long long walk[5] = {0, 0, 0, 0, 0};  // entries, warp-passed leaves, staged leaves, flush rounds, work items
  unsigned long long *d_evals = nullptr;
  // friends-of-friends catalogue of the last jz_fof call (device; group order = root z-order)
  int64_t fof_ngroups = 0;
  int32_t *fof_label = nullptr, *fof_count = nullptr;
  double *fof_com = nullptr, *fof_rad = nullptr;
  int32_t *fof_root = nullptr;  // [n] root z position of each z position (last jz_fof; group order)
  // multi-GPU (jz_knn_build_dist): this rank's part of a distributed index (jz_dist.cu)
  jz_comm *comm = nullptr;
  int64_t n_own = 0, gidx_base = 0;  // this rank's input slice: global ids [gidx_base, gidx_base + n_own)
  bool has_box = false;
  float box[3] = {0, 0, 0};
  jz_knn_params prm_frame{};         // params with the global key frame (open boundary: JZ_FLAG_FRAME)
  bool empty = false;                // no local points after the partition (no tree)
  double dist_ms[8] = {0, 0, 0, 0, 0, 0, 0, 0};  // phase wall times of the last build / query
  int64_t dist_cnt[4] = {0, 0, 0, 0};          // local points, ghosts received, re-queried, boxes
};

namespace jz {

// build (jz_sort.cu)
void compute_frame(const float *pos, int64_t n, int stride, const Dom &D, const jz_knn_params_t &prm, Frame *frame,
                   cudaStream_t st);
void sort_points(const float *pos, int64_t n, int stride, int gidx_mode, int64_t gidx_base, const Frame &frame,
                 uint64_t *keys_out, int32_t *perm_out, float4 *pts_out, cudaStream_t st);
void morton_keys(const float *pos, int64_t n, const Frame &f, uint64_t *keys, cudaStream_t st);
// stable LSD sort of 32-bit (key, value) pairs (one-sweep passes; in and out buffers distinct)
void sort_pairs_u32(const uint32_t *keys, const uint32_t *vals, int64_t n, uint32_t *keys_out, uint32_t *vals_out,
                    cudaStream_t st);
void local_bbox(const float *pos, int64_t n, int stride, const Dom &D, float lo[3], float hi[3], cudaStream_t st);

// tree (jz_build.cu)
void build_planes(const uint64_t *keys, const float4 *pts, int64_t n, const jz_knn_params_t &prm,
                  std::vector<Plane> &planes, cudaStream_t st);
void free_planes(std::vector<Plane> &planes, cudaStream_t st);

// walk (jz_walk.cu)
struct IList {
  int64_t nrecv = 0, total = 0;
  int64_t *ispl = nullptr;  // [nrecv + 1]
  int32_t *isrc = nullptr;  // [total]
  float *rlow = nullptr;    // [total]  squared lower bound d_low^2 of the (receiver, source) pair
  void release(cudaStream_t st);
};
// Walk the plane hierarchy from the super nodes down to plane `stop` (Alg. 1
// lines 1-5): returns the interaction list whose receivers are the nodes of plane `stop`
// and R_max^2 of those nodes (caller frees). If stop > top plane (only possible for a
// one-plane tree and stop = 1), the receivers are the super nodes: *superbeg (first top
// node of each super node, caller frees) is set, the list is the dense one and
// *rmax2 = nullptr (= +inf).
// qbeg (optional): query leaf starts when the queries are a subset of the points -- receivers
// without queries get no list.
// fixed_r2 >= 0: fixed-radius walk (friends-of-friends): no FindRmax, every node's radius^2 is
// fixed_r2, so the lists hold the pairs with d_low^2 <= fixed_r2.
void walk_to(const std::vector<Plane> &planes, const Dom &D, int k, int ngr, unsigned flags, int stop, IList &il,
             float **rmax2, int32_t **superbeg, cudaStream_t st, float fixed_r2 = -1.f,
             const int32_t *qbeg = nullptr);

// friends-of-friends walk with node links (§5): lists of plane-1 receivers
// (pairs of nodes neither too far nor fully linked) and the point-level union-find start par[npts]
// (points of linked leaves point to the first point of their group's root leaf)
void fof_walk(const std::vector<Plane> &planes, const Dom &D, int ngr, float b2, IList &out_il,
              int32_t **superbeg_out, int32_t *par, int64_t npts, cudaStream_t st);

// leaf-to-leaf (jz_leaf.cu)
struct LeafArgs {
  const float4 *spts;       // source points (z order)
  const int32_t *sbeg;      // [nleaf+1] first source of each leaf
  const float4 *qpts;       // query points (z order); .w = gidx, or the input row of a query-only point
  const int32_t *qbeg;      // [nleaf+1] first query of each leaf
  const int32_t *qin;       // [nq] input row of each query
  const NodeBox *leaf_box;  // [nleaf]
  int64_t nleaf;
  const int32_t *par_leaf;  // [npar+1] first leaf of each receiving parent
  const NodeBox *par_box;   // [npar] or nullptr
  int64_t npar;
  const IList *il;          // receivers = parents
  const float *rmax2;       // [npar] or nullptr
  int k;                    // any k >= 1: ceil(k / kMaxK) kernel passes
  int order;
  unsigned flags;
  int32_t *out_idx;
  float *out_d2;
  int32_t *out_row_gidx;
  unsigned long long *evals;  // device counter (may be nullptr)
  // optional chunked launch (JZ_ORDER_Z streaming): after chunk c, on_rows(q_lo, q_hi) is called
  // with the finished z-order query rows [q_lo, q_hi); nq = number of queries
  int chunks = 1;
  int64_t nq = 0;
  std::function<void(int64_t, int64_t)> on_rows;
};
void leaf_to_leaf(const LeafArgs &a, const Dom &D, cudaStream_t st);

// friends-of-friends leaf stage (jz_leaf.cu): links every pair of points with canonical
// d2 <= b2 in the union-find array par (sorted positions; roots = smallest position)
void fof_leaf(const LeafArgs &a, const Dom &D, float b2, int32_t *par, cudaStream_t st);

// read-only view of an index for the multi-GPU stage kernels (jz_dist.cu)
struct IndexView {
  int64_t n;
  const float4 *pts;
  const std::vector<Plane> *planes;
  Dom D;
  int ngr;
  unsigned flags;
};
IndexView view_of(const jz_knn_index *ix);

// A1-A8 build of an index (jz_api.cu): stride 3 (xyz) or 4 (xyzg with gidx_mode = 1)
jz_knn_index *build_impl(const float *pos, int64_t n, int stride, int gidx_mode, int64_t n_query, const float *box,
                         const jz_knn_params *p, cudaStream_t st);

// text returned by jz_last_error() (thread-local)
void set_last_error(const std::string &m);

}  // namespace jz
