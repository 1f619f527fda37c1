// jz_api.cu -- C ABI (include/jz_knn.h) and host orchestration of the hot path.
//
//   jz_knn_build  : A1 frame/validate -> A2/A3 encode + radix sort + gather -> A4-A8 planes
//   jz_knn_query  : A9/A10 walk to the leaf plane -> A11/A12 LeafToLeaf with fused output
// (Alg. 1). Device memory comes from the stream-ordered pool
// (cudaMallocAsync), so repeated build/query calls reuse memory without device syncs.
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "jz_common.cuh"
#include "jz_internal.h"

struct jz_knn_index {
  cudaStream_t st = nullptr;
  int64_t n = 0, n_query = 0;
  jz::Dom D{};
  jz_knn_params prm{};
  float4 *pts = nullptr;
  uint64_t *keys = nullptr;
  int32_t *perm = nullptr;
  int32_t *zrow = nullptr;
  std::vector<jz::Plane> planes;
  cudaEvent_t ev[8] = {};
  bool timing = false;
  float times[6] = {0, 0, 0, 0, 0, 0};
  long long evals = 0, inserts = 0;
  long long walk[5] = {0, 0, 0, 0, 0};  // entries, warp-passed leaves, staged leaves, flush rounds, work items
  unsigned long long *d_evals = nullptr;
};

#include <atomic>

namespace jz {
static std::atomic<long long> g_launches{0};
void count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }
IndexView view_of(const jz_knn_index *ix) {
  return IndexView{ix->n, ix->pts, &ix->planes, ix->D, ix->prm.ngr, ix->prm.flags};
}
}  // namespace jz

namespace {
thread_local std::string g_err;
int g_timing = -1;

int fail(int code, const std::string &m) {
  g_err = m;
  return code;
}

bool timing_enabled() {
  if (g_timing < 0) {
    const char *e = getenv("JZ_TIMING");
    g_timing = (e && e[0] == '1') ? 1 : 0;
  }
  return g_timing == 1;
}

void init_pool() {
  static bool done = false;
  if (done) return;
  done = true;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return;
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
    uint64_t thr = UINT64_MAX;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
  }
}

jz_knn_params normalize(const jz_knn_params *p) {
  jz_knn_params r;
  memset(&r, 0, sizeof(r));
  if (p) r = *p;
  if (r.nmax0 <= 0) r.nmax0 = 128;  // larger leaves amortise the walk (paper default 48)
  if (r.coarsen <= 0) r.coarsen = 8;
  if (r.ntarget <= 0) r.ntarget = 1000;
  if (r.ngr <= 0) r.ngr = 32;
  return r;
}

jz::Dom make_dom(const float *box) {
  jz::Dom D;
  memset(&D, 0, sizeof(D));
  if (box) {
    D.periodic = 1;
    for (int d = 0; d < 3; ++d) {
      D.L[d] = box[d];
      D.h[d] = 0.5f * box[d];
    }
  }
  return D;
}

void check_box(const float *box) {
  if (!box) return;
  for (int d = 0; d < 3; ++d)
    if (!(box[d] > 0.f) || !std::isfinite(box[d])) throw jz::Error(JZ_EINVAL, "periodic box lengths must be finite and > 0");
}

void rec(jz_knn_index *ix, int i) {
  if (ix->timing) JZ_CUDA(cudaEventRecord(ix->ev[i], ix->st));
}

__global__ void k_zrow_flags(const int32_t *__restrict__ perm, int64_t n, int64_t nq, int32_t *__restrict__ f) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    f[i] = perm[i] < nq;
}
__global__ void k_i64_to_i32(const int64_t *__restrict__ a, int64_t n, int32_t *__restrict__ b) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    b[i] = (int32_t)a[i];
}

jz_knn_index *build_impl(const float *pos, int64_t n, int stride, int gidx_mode, int64_t n_query, const float *box,
                         const jz_knn_params *p, cudaStream_t st) {
  if (!pos) throw jz::Error(JZ_EINVAL, "pos is NULL");
  if (n < 1 || n > (int64_t)INT32_MAX - 1) throw jz::Error(JZ_EINVAL, "n must be in [1, 2^31 - 2]");
  if (n_query < 0 || n_query > n) throw jz::Error(JZ_EINVAL, "n_query must be in [0, n]");
  check_box(box);
  jz_knn_params prm = normalize(p);
  if (prm.nmax0 > jz::kMaxLeaf) throw jz::Error(JZ_EINVAL, "nmax0 must be <= 128");
  if (prm.coarsen < 2) throw jz::Error(JZ_EINVAL, "coarsen must be >= 2");
  if ((prm.flags & JZ_FLAG_FRAME) && !(prm.frame_extent > 0.f)) throw jz::Error(JZ_EINVAL, "frame_extent must be > 0");
  init_pool();
  auto *ix = new jz_knn_index();
  ix->st = st;
  ix->n = n;
  ix->n_query = n_query;
  ix->D = make_dom(box);
  ix->prm = prm;
  ix->timing = timing_enabled();
  try {
    if (ix->timing)
      for (auto &e : ix->ev) JZ_CUDA(cudaEventCreate(&e));
    rec(ix, 0);
    jz::Frame frame;
    jz::compute_frame(pos, n, stride, ix->D, prm, &frame, st);
    rec(ix, 1);
    JZ_CUDA(cudaMallocAsync(&ix->pts, n * sizeof(float4), st));
    JZ_CUDA(cudaMallocAsync(&ix->keys, n * sizeof(uint64_t), st));
    JZ_CUDA(cudaMallocAsync(&ix->perm, n * sizeof(int32_t), st));
    jz::sort_points(pos, n, stride, gidx_mode, 0, frame, ix->keys, ix->perm, ix->pts, st);
    rec(ix, 2);
    jz::build_planes(ix->keys, ix->pts, n, prm, ix->planes, st);
    if (n_query < n) {  // z-order row of each query (ghost-carrying builds)
      int32_t *f = nullptr;
      int64_t *ps = nullptr;
      JZ_CUDA(cudaMallocAsync(&f, n * sizeof(int32_t), st));
      JZ_CUDA(cudaMallocAsync(&ps, (n + 1) * sizeof(int64_t), st));
      JZ_CUDA(cudaMallocAsync(&ix->zrow, n * sizeof(int32_t), st));
      k_zrow_flags<<<jz::grid_for(n, 256), 256, 0, st>>>(ix->perm, n, n_query, f);
      JZ_LAUNCH_CHECK();
      jz::exclusive_scan_i32_to_i64(f, ps, n, st);
      k_i64_to_i32<<<jz::grid_for(n, 256), 256, 0, st>>>(ps, n, ix->zrow);
      JZ_LAUNCH_CHECK();
      JZ_CUDA(cudaFreeAsync(f, st));
      JZ_CUDA(cudaFreeAsync(ps, st));
    }
    rec(ix, 3);
    if (ix->timing) {
      JZ_CUDA(cudaEventSynchronize(ix->ev[3]));
      cudaEventElapsedTime(&ix->times[0], ix->ev[0], ix->ev[1]);
      cudaEventElapsedTime(&ix->times[1], ix->ev[1], ix->ev[2]);
      cudaEventElapsedTime(&ix->times[2], ix->ev[2], ix->ev[3]);
    }
    JZ_CUDA(cudaStreamSynchronize(st));
  } catch (...) {
    jz_knn_free(ix);
    throw;
  }
  return ix;
}

}  // namespace

extern "C" {

const char *jz_last_error(void) { return g_err.c_str(); }

void jz_set_timing(int on) { g_timing = on ? 1 : 0; }

int64_t jz_launch_count(void) { return (int64_t)jz::g_launches.load(); }

#define JZ_API_BEGIN try {
#define JZ_API_END                                                  \
  }                                                                 \
  catch (const jz::Error &e) {                                      \
    return fail(e.code, e.what());                                  \
  }                                                                 \
  catch (const std::exception &e) {                                 \
    return fail(JZ_ECUDA, e.what());                                \
  }

int jz_knn_build(const float *pos, int64_t n, const float *box, const jz_knn_params *p, jz_stream_t s,
                 jz_knn_index **out) {
  JZ_API_BEGIN
  if (!out) return fail(JZ_EINVAL, "out is NULL");
  *out = build_impl(pos, n, 3, 0, n, box, p, (cudaStream_t)s);
  return JZ_OK;
  JZ_API_END
}

int jz_knn_build_xyzg(const float *pts4, int64_t n, int64_t n_query, const float *box, const jz_knn_params *p,
                      jz_stream_t s, jz_knn_index **out) {
  JZ_API_BEGIN
  if (!out) return fail(JZ_EINVAL, "out is NULL");
  *out = build_impl(pts4, n, 4, 1, n_query, box, p, (cudaStream_t)s);
  return JZ_OK;
  JZ_API_END
}

int jz_knn_rows(const jz_knn_index *ix, int64_t *m) {
  if (!ix || !m) return fail(JZ_EINVAL, "NULL argument");
  *m = ix->n_query;
  return JZ_OK;
}

int jz_knn_query(jz_knn_index *ix, int k, int order, int32_t *out_idx, float *out_d2, int32_t *out_row_gidx,
                 jz_stream_t s) {
  JZ_API_BEGIN
  if (!ix || !out_idx || !out_d2) return fail(JZ_EINVAL, "NULL argument");
  if (k < 1 || k > jz::kMaxK) return fail(JZ_EINVAL, "k must be in [1, 32]");
  if (k > ix->n) return fail(JZ_EINVAL, "k must not exceed the number of points");
  if (order != JZ_ORDER_INPUT && order != JZ_ORDER_Z) return fail(JZ_EINVAL, "bad order");
  if (order == JZ_ORDER_Z && !out_row_gidx) return fail(JZ_EINVAL, "JZ_ORDER_Z needs out_row_gidx");
  cudaStream_t st = (cudaStream_t)s;
  ix->st = st;
  if (ix->n_query == 0) return JZ_OK;
  rec(ix, 4);
  jz::IList il;
  float *rmax2 = nullptr;
  int32_t *superbeg = nullptr;
  // walk down to plane 1: its nodes are the receiving parents of LeafToLeaf (jz_leaf.cu)
  jz::walk_to(ix->planes, ix->D, k, ix->prm.ngr, ix->prm.flags, 1, il, &rmax2, &superbeg, st);
  rec(ix, 5);
  if (!ix->d_evals) JZ_CUDA(cudaMallocAsync(&ix->d_evals, 16 * sizeof(unsigned long long), st));
  JZ_CUDA(cudaMemsetAsync(ix->d_evals, 0, 16 * sizeof(unsigned long long), st));
  const bool one_plane = ix->planes.size() == 1;
  jz::LeafArgs la;
  la.pts = ix->pts;
  la.leaf_beg = ix->planes[0].beg;
  la.leaf_box = ix->planes[0].box;
  la.par_leaf = one_plane ? superbeg : ix->planes[1].beg;
  la.par_box = one_plane ? nullptr : ix->planes[1].box;
  la.npar = il.nrecv;
  la.il = &il;
  la.rmax2 = rmax2;
  la.perm = ix->perm;
  la.zrow = ix->zrow;
  la.n_query = ix->n_query;
  la.k = k;
  la.order = order;
  la.flags = ix->prm.flags;
  la.out_idx = out_idx;
  la.out_d2 = out_d2;
  la.out_row_gidx = out_row_gidx;
  la.evals = ix->d_evals;
  jz::leaf_to_leaf(la, ix->D, st);
  rec(ix, 6);
  il.release(st);
  if (rmax2) JZ_CUDA(cudaFreeAsync(rmax2, st));
  if (superbeg) JZ_CUDA(cudaFreeAsync(superbeg, st));
  unsigned long long ev[16] = {};
  JZ_CUDA(cudaMemcpyAsync(ev, ix->d_evals, sizeof(ev), cudaMemcpyDeviceToHost, st));
  JZ_CUDA(cudaStreamSynchronize(st));
  ix->evals = (long long)ev[0];
  ix->inserts = (long long)ev[1];
  for (int i = 0; i < 5; ++i) ix->walk[i] = (long long)ev[2 + i];

  if (ix->timing) {
    cudaEventElapsedTime(&ix->times[3], ix->ev[4], ix->ev[5]);
    cudaEventElapsedTime(&ix->times[4], ix->ev[5], ix->ev[6]);
    ix->times[5] = ix->times[0] + ix->times[1] + ix->times[2] + ix->times[3] + ix->times[4];
  }
  return JZ_OK;
  JZ_API_END
}

void jz_knn_free(jz_knn_index *ix) {
  if (!ix) return;
  cudaStream_t st = ix->st;
  jz::free_planes(ix->planes, st);
  if (ix->pts) cudaFreeAsync(ix->pts, st);
  if (ix->keys) cudaFreeAsync(ix->keys, st);
  if (ix->perm) cudaFreeAsync(ix->perm, st);
  if (ix->zrow) cudaFreeAsync(ix->zrow, st);
  if (ix->d_evals) cudaFreeAsync(ix->d_evals, st);
  cudaStreamSynchronize(st);
  for (auto &e : ix->ev)
    if (e) cudaEventDestroy(e);
  delete ix;
}

int jz_knn_search_host(const float *pos_host, int64_t n, const float *box, const jz_knn_params *p, int k,
                       int32_t *idx_host, float *d2_host, jz_stream_t s) {
  JZ_API_BEGIN
  if (!pos_host || !idx_host || !d2_host) return fail(JZ_EINVAL, "NULL argument");
  if (n < 1) return fail(JZ_EINVAL, "n must be >= 1");
  if (k < 1 || k > jz::kMaxK || k > n) return fail(JZ_EINVAL, "k must be in [1, min(32, n)]");
  cudaStream_t st = (cudaStream_t)s;
  init_pool();
  float *dpos = nullptr;
  int32_t *didx = nullptr;
  float *dd2 = nullptr;
  JZ_CUDA(cudaMallocAsync(&dpos, n * 3 * sizeof(float), st));
  JZ_CUDA(cudaMemcpyAsync(dpos, pos_host, n * 3 * sizeof(float), cudaMemcpyHostToDevice, st));
  jz_knn_index *ix = nullptr;
  int rc = jz_knn_build(dpos, n, box, p, s, &ix);
  if (rc != JZ_OK) {
    cudaFreeAsync(dpos, st);
    return rc;
  }
  JZ_CUDA(cudaFreeAsync(dpos, st));
  JZ_CUDA(cudaMallocAsync(&didx, n * k * sizeof(int32_t), st));
  JZ_CUDA(cudaMallocAsync(&dd2, n * k * sizeof(float), st));
  rc = jz_knn_query(ix, k, JZ_ORDER_INPUT, didx, dd2, nullptr, s);
  jz_knn_free(ix);
  if (rc == JZ_OK) {
    JZ_CUDA(cudaMemcpyAsync(idx_host, didx, n * k * sizeof(int32_t), cudaMemcpyDeviceToHost, st));
    JZ_CUDA(cudaMemcpyAsync(d2_host, dd2, n * k * sizeof(float), cudaMemcpyDeviceToHost, st));
  }
  JZ_CUDA(cudaFreeAsync(didx, st));
  JZ_CUDA(cudaFreeAsync(dd2, st));
  JZ_CUDA(cudaStreamSynchronize(st));
  return rc;
  JZ_API_END
}

int jz_knn_stats(const jz_knn_index *ix, int64_t out[9]) {
  if (!ix || !out) return fail(JZ_EINVAL, "NULL argument");
  out[0] = ix->evals;
  out[1] = ix->inserts;
  out[2] = ix->planes.empty() ? 0 : ix->planes[0].nnodes;
  out[3] = (int64_t)ix->planes.size();
  for (int i = 0; i < 5; ++i) out[4 + i] = ix->walk[i];
  return JZ_OK;
}

int jz_knn_stage_times(const jz_knn_index *ix, float out_ms[6], int64_t *evals) {
  if (!ix || !out_ms) return fail(JZ_EINVAL, "NULL argument");
  for (int i = 0; i < 6; ++i) out_ms[i] = ix->times[i];
  if (evals) *evals = ix->evals;
  return JZ_OK;
}

// ---- introspection for stage tests: copy internal arrays to host (returns bytes needed)
// what: 0 sorted keys u64[n], 1 sorted pts float4[n], 2 perm i32[n],
//       3 plane beg i32[nnodes+1], 4 plane boxes NodeBox[nnodes], 5 number of planes (int64 in dst)
int64_t jz_knn_debug_copy(const jz_knn_index *ix, int what, int plane, void *dst, int64_t cap) {
  if (!ix) return -1;
  size_t bytes = 0;
  const void *src = nullptr;
  switch (what) {
    case 0: bytes = ix->n * 8; src = ix->keys; break;
    case 1: bytes = ix->n * 16; src = ix->pts; break;
    case 2: bytes = ix->n * 4; src = ix->perm; break;
    case 3:
      if (plane < 0 || plane >= (int)ix->planes.size()) return -1;
      bytes = (ix->planes[plane].nnodes + 1) * 4;
      src = ix->planes[plane].beg;
      break;
    case 4:
      if (plane < 0 || plane >= (int)ix->planes.size()) return -1;
      bytes = ix->planes[plane].nnodes * sizeof(jz::NodeBox);
      src = ix->planes[plane].box;
      break;
    case 5:
      if (dst && cap >= 8) *(int64_t *)dst = (int64_t)ix->planes.size();
      return 8;
    default: return -1;
  }
  if (dst && cap >= (int64_t)bytes && bytes) {
    if (cudaMemcpy(dst, src, bytes, cudaMemcpyDeviceToHost) != cudaSuccess) return -1;
  }
  return (int64_t)bytes;
}

}  // extern "C"
