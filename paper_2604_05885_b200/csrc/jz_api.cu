#include <chrono>
// jz_api.cu -- C ABI (include/jz_knn.h) and host orchestration of the hot path.
//
//   jz_knn_build  : A1 frame/validate -> A2/A3 encode + radix sort + gather -> A4-A8 planes
//   jz_knn_query  : A9/A10 walk to the leaf plane -> A11/A12 LeafToLeaf with fused output
// (Alg. 1). Device memory comes from the stream-ordered pool
// (cudaMallocAsync), so repeated build/query calls reuse memory without device syncs.
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <ctime>
#include <string>
#include <vector>

#include "jz_common.cuh"
#include "jz_internal.h"



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
  if (r.nmax0 <= 0) r.nmax0 = 80;  // larger leaves amortise the walk (paper default 48)
  if (r.coarsen <= 0) r.coarsen = 16;   // fewer, larger plane-1 nodes (paper 8)
  if (r.ntarget <= 0) r.ntarget = 30;  // with c = 16: planes 1-4 at 10^8 (paper ~1000; tools/variants/g_nt.sh)
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

// ---- point types: a point is a query iff its input position < n_query,
// a source iff its gidx (.w) >= 0. After the joint sort + tree build the points are separated
// into type-specific z-ordered arrays with per-type leaf splits.
__global__ void k_type_flags(const float4 *__restrict__ pts, const int32_t *__restrict__ perm, int64_t n, int64_t nq,
                             int32_t *__restrict__ fs, int32_t *__restrict__ fq) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    fs[i] = __float_as_int(pts[i].w) >= 0;
    fq[i] = perm[i] < nq;
  }
}
__global__ void k_type_scatter(const float4 *__restrict__ pts, const int32_t *__restrict__ perm, int64_t n, int64_t nq,
                               const int64_t *__restrict__ srank, const int64_t *__restrict__ qrank,
                               float4 *__restrict__ spts, float4 *__restrict__ qpts, int32_t *__restrict__ qin) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    float4 p = pts[i];
    const int in = perm[i];
    const int g = __float_as_int(p.w);
    if (spts && g >= 0) spts[srank[i]] = p;
    if (qpts && in < nq) {
      if (g < 0) p.w = __int_as_float(in);  // query-only point: report its input row
      qpts[qrank[i]] = p;
      qin[qrank[i]] = in;
    }
  }
}
__global__ void k_type_beg(const int32_t *__restrict__ beg, int64_t m, const int64_t *__restrict__ srank,
                           const int64_t *__restrict__ qrank, int32_t *__restrict__ sbeg, int32_t *__restrict__ qbeg) {
  for (int64_t l = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; l < m; l += (int64_t)gridDim.x * blockDim.x) {
    if (sbeg) sbeg[l] = (int32_t)srank[beg[l]];
    if (qbeg) qbeg[l] = (int32_t)qrank[beg[l]];
  }
}
__global__ void k_pack_xq(const float *__restrict__ qry, int64_t nq, const float *__restrict__ src, int64_t ns,
                          float4 *__restrict__ out) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nq + ns; i += (int64_t)gridDim.x * blockDim.x) {
    if (i < nq) out[i] = make_float4(qry[3 * i], qry[3 * i + 1], qry[3 * i + 2], __int_as_float(-1));
    else {
      const int64_t j = i - nq;
      out[i] = make_float4(src[3 * j], src[3 * j + 1], src[3 * j + 2], __int_as_float((int)j));
    }
  }
}

void split_types(jz_knn_index *ix, bool typed) {
  const int64_t n = ix->n, nleaf = ix->planes[0].nnodes;
  cudaStream_t st = ix->st;
  ix->spts = ix->qpts = ix->pts;
  ix->sbeg = ix->qbeg = ix->planes[0].beg;
  ix->qin = ix->perm;
  ix->n_src = n;
  if (!typed) return;
  int32_t *fs = nullptr, *fq = nullptr;
  int64_t *sr = nullptr, *qr = nullptr;
  JZ_CUDA(cudaMallocAsync(&fs, n * sizeof(int32_t), st));
  JZ_CUDA(cudaMallocAsync(&fq, n * sizeof(int32_t), st));
  JZ_CUDA(cudaMallocAsync(&sr, (n + 1) * sizeof(int64_t), st));
  JZ_CUDA(cudaMallocAsync(&qr, (n + 1) * sizeof(int64_t), st));
  k_type_flags<<<jz::grid_for(n, 256), 256, 0, st>>>(ix->pts, ix->perm, n, ix->n_query, fs, fq);
  JZ_LAUNCH_CHECK();
  jz::exclusive_scan_i32_to_i64(fs, sr, n, st);
  jz::exclusive_scan_i32_to_i64(fq, qr, n, st);
  ix->n_src = jz::read_i64(sr + n, st);
  const bool sep_s = ix->n_src < n, sep_q = ix->n_query < n;
  if (sep_s) {
    JZ_CUDA(cudaMallocAsync(&ix->spts, (ix->n_src > 0 ? ix->n_src : 1) * sizeof(float4), st));
    JZ_CUDA(cudaMallocAsync(&ix->sbeg, (nleaf + 1) * sizeof(int32_t), st));
    ix->own_s = true;
  }
  if (sep_q || sep_s) {  // query-only points get their input row in .w
    JZ_CUDA(cudaMallocAsync(&ix->qpts, (ix->n_query > 0 ? ix->n_query : 1) * sizeof(float4), st));
    JZ_CUDA(cudaMallocAsync(&ix->qbeg, (nleaf + 1) * sizeof(int32_t), st));
    JZ_CUDA(cudaMallocAsync(&ix->qin, (ix->n_query > 0 ? ix->n_query : 1) * sizeof(int32_t), st));
    ix->own_q = true;
  }
  if (sep_s || sep_q) {
    k_type_scatter<<<jz::grid_for(n, 256), 256, 0, st>>>(ix->pts, ix->perm, n, ix->n_query, sr, qr,
                                                         sep_s ? ix->spts : nullptr, ix->own_q ? ix->qpts : nullptr,
                                                         ix->own_q ? ix->qin : nullptr);
    JZ_LAUNCH_CHECK();
    k_type_beg<<<jz::grid_for(nleaf + 1, 256), 256, 0, st>>>(ix->planes[0].beg, nleaf + 1, sr, qr,
                                                             sep_s ? ix->sbeg : nullptr, ix->own_q ? ix->qbeg : nullptr);
    JZ_LAUNCH_CHECK();
  }
  JZ_CUDA(cudaFreeAsync(fs, st));
  JZ_CUDA(cudaFreeAsync(fq, st));
  JZ_CUDA(cudaFreeAsync(sr, st));
  JZ_CUDA(cudaFreeAsync(qr, st));
}

// ---- friends-of-friends (§5)
__global__ void k_fof_init(int32_t *__restrict__ par, int32_t *__restrict__ minlab, int64_t n) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    par[i] = (int32_t)i;
    minlab[i] = INT32_MAX;
  }
}
// contraction ("setting every pointer to its root"): runs after every link is done
__global__ void k_fof_flatten(int32_t *__restrict__ par, int64_t n) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    int32_t x = par[i];
    while (par[x] != x) x = par[x];
    par[i] = x;
  }
}
__global__ void k_fof_minlab(const float4 *__restrict__ pts, const int32_t *__restrict__ par, int64_t n,
                             int32_t *__restrict__ minlab) {
  for (int64_t i0 = (int64_t)blockIdx.x * blockDim.x; i0 < n; i0 += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = i0 + threadIdx.x;
    const bool ok = i < n;
    const int32_t r = ok ? par[i] : -1;
    const int g = ok ? __float_as_int(pts[i].w) : INT32_MAX;
    const unsigned peers = __match_any_sync(0xffffffffu, r);
    const int gm = __reduce_min_sync(peers, g);  // one atomic per (warp, group)
    if (ok && (threadIdx.x & 31) == __ffs(peers) - 1) atomicMin(&minlab[r], gm);
  }
}
// label of input row gidx = smallest input index of its group (R21)
__global__ void k_fof_labels(const float4 *__restrict__ pts, const int32_t *__restrict__ par,
                             const int32_t *__restrict__ minlab, int64_t n, int32_t *__restrict__ labels) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    labels[__float_as_int(pts[i].w)] = minlab[par[i]];
}
__device__ __forceinline__ double fof_disp(float x, float xr, int periodic, float L) {
  double d = (double)x - (double)xr;
  if (periodic) d -= (double)L * rint(d / (double)L);  // minimal image w.r.t. the group's root point
  return d;
}
// Per-group sums with one set of atomics per (warp, group): consecutive z positions mostly share
// a root, so the lanes of a group put their values in shared memory and the group's first lane
// adds them up (a group of 10^5 points would otherwise serialise 10^5 FP64 atomics on one address).
constexpr int kFofThreads = 256;
__global__ void __launch_bounds__(kFofThreads) k_fof_sum1(const float4 *__restrict__ pts,
                                                          const int32_t *__restrict__ par, int64_t n, jz::Dom D,
                                                          int32_t *__restrict__ cnt, double *__restrict__ sum) {
  __shared__ double s_v[kFofThreads][3];
  const int lane = threadIdx.x & 31, wb = threadIdx.x & ~31;
  for (int64_t i0 = (int64_t)blockIdx.x * blockDim.x; i0 < n; i0 += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = i0 + threadIdx.x;
    const bool ok = i < n;
    int32_t r = -1;
    double dx = 0.0, dy = 0.0, dz = 0.0;
    if (ok) {
      r = par[i];
      const float4 p = pts[i], q = pts[r];
      dx = fof_disp(p.x, q.x, D.periodic, D.L[0]);
      dy = fof_disp(p.y, q.y, D.periodic, D.L[1]);
      dz = fof_disp(p.z, q.z, D.periodic, D.L[2]);
    }
    s_v[threadIdx.x][0] = dx;
    s_v[threadIdx.x][1] = dy;
    s_v[threadIdx.x][2] = dz;
    const unsigned peers = __match_any_sync(0xffffffffu, r);
    __syncwarp();
    if (ok && lane == __ffs(peers) - 1) {
      double a = 0.0, b = 0.0, c = 0.0;
      for (unsigned m = peers; m; m &= m - 1) {
        const int t = wb + __ffs(m) - 1;
        a += s_v[t][0];
        b += s_v[t][1];
        c += s_v[t][2];
      }
      atomicAdd(&cnt[r], __popc(peers));
      atomicAdd(&sum[3 * (int64_t)r + 0], a);
      atomicAdd(&sum[3 * (int64_t)r + 1], b);
      atomicAdd(&sum[3 * (int64_t)r + 2], c);
    }
    __syncwarp();
  }
}
__global__ void __launch_bounds__(kFofThreads) k_fof_sum2(const float4 *__restrict__ pts,
                                                          const int32_t *__restrict__ par, int64_t n, jz::Dom D,
                                                          const int32_t *__restrict__ cnt,
                                                          const double *__restrict__ sum, double *__restrict__ ss) {
  __shared__ double s_v[kFofThreads];
  const int lane = threadIdx.x & 31, wb = threadIdx.x & ~31;
  for (int64_t i0 = (int64_t)blockIdx.x * blockDim.x; i0 < n; i0 += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = i0 + threadIdx.x;
    const bool ok = i < n;
    int32_t r = -1;
    double v = 0.0;
    if (ok) {
      r = par[i];
      const float4 p = pts[i], q = pts[r];
      const double c = (double)cnt[r];
      const double dx = fof_disp(p.x, q.x, D.periodic, D.L[0]) - sum[3 * (int64_t)r] / c;
      const double dy = fof_disp(p.y, q.y, D.periodic, D.L[1]) - sum[3 * (int64_t)r + 1] / c;
      const double dz = fof_disp(p.z, q.z, D.periodic, D.L[2]) - sum[3 * (int64_t)r + 2] / c;
      v = dx * dx + dy * dy + dz * dz;
    }
    s_v[threadIdx.x] = v;
    const unsigned peers = __match_any_sync(0xffffffffu, r);
    __syncwarp();
    if (ok && lane == __ffs(peers) - 1) {
      double a = 0.0;
      for (unsigned m = peers; m; m &= m - 1) a += s_v[wb + __ffs(m) - 1];
      atomicAdd(&ss[r], a);
    }
    __syncwarp();
  }
}
__global__ void k_fof_flags(const int32_t *__restrict__ par, const int32_t *__restrict__ cnt, int64_t n, int min_count,
                            int32_t *__restrict__ flag) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    flag[i] = par[i] == (int32_t)i && cnt[i] >= min_count;
}
__global__ void k_fof_cat(const float4 *__restrict__ pts, const int32_t *__restrict__ flag,
                          const int64_t *__restrict__ pos, const int32_t *__restrict__ minlab,
                          const int32_t *__restrict__ cnt, const double *__restrict__ sum,
                          const double *__restrict__ ss, int64_t n, jz::Dom D, int32_t *__restrict__ olab,
                          int32_t *__restrict__ ocnt, double *__restrict__ ocom, double *__restrict__ orad) {
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < n; r += (int64_t)gridDim.x * blockDim.x) {
    if (!flag[r]) continue;
    const int64_t o = pos[r];
    const double c = (double)cnt[r];
    const float4 q = pts[r];
    const float qq[3] = {q.x, q.y, q.z};
    for (int d = 0; d < 3; ++d) {
      double v = (double)qq[d] + sum[3 * r + d] / c;
      if (D.periodic) v -= (double)D.L[d] * floor(v / (double)D.L[d]);  // wrapped into [0, L)
      ocom[3 * o + d] = v;
    }
    olab[o] = minlab[r];
    ocnt[o] = cnt[r];
    orad[o] = sqrt(ss[r] / c);
  }
}

}  // namespace

jz_knn_index *jz::build_impl(const float *pos, int64_t n, int stride, int gidx_mode, int64_t n_query, const float *box,
                             const jz_knn_params *p, cudaStream_t st) {
  if (!pos) throw jz::Error(JZ_EINVAL, "pos is NULL");
  if (n < 1 || n > (int64_t)INT32_MAX - 1) throw jz::Error(JZ_EINVAL, "n must be in [1, 2^31 - 2]");
  if (n_query < 0 || n_query > n) throw jz::Error(JZ_EINVAL, "n_query must be in [0, n]");
  check_box(box);
  jz_knn_params prm = normalize(p);
  if (prm.nmax0 > jz::kMaxLeaf) throw jz::Error(JZ_EINVAL, "nmax0 must be <= 128");
  if (prm.coarsen < 2) throw jz::Error(JZ_EINVAL, "coarsen must be >= 2");
  if (prm.reg_fmax < 0) throw jz::Error(JZ_EINVAL, "reg_fmax must be >= 0");
  if ((prm.flags & JZ_FLAG_FRAME) && !(prm.frame_extent > 0.f)) throw jz::Error(JZ_EINVAL, "frame_extent must be > 0");
  init_pool();
  auto *ix = new jz_knn_index();
  ix->st = st;
  ix->n = n;
  ix->n_query = n_query;
  ix->D = make_dom(box);
  ix->prm = prm;
  ix->input_ids = gidx_mode == 0;
  ix->timing = timing_enabled();
  try {
    if (ix->timing)
      for (auto &e : ix->ev) JZ_CUDA(cudaEventCreate(&e));
    static const bool bprof = getenv("JZ_BUILD_PROF") != nullptr;
    timespec tq;
    auto wall = [&]() {
      clock_gettime(CLOCK_MONOTONIC, &tq);
      return tq.tv_sec * 1e3 + tq.tv_nsec * 1e-6;
    };
    double tb = wall();
    auto bmark = [&](const char *w) {  // diagnostics: host wall time of each build step
      if (!bprof) return;
      cudaStreamSynchronize(st);
      const double t = wall();
      fprintf(stderr, "build n=%lld %-8s %8.2f ms\n", (long long)n, w, t - tb);
      tb = t;
    };
    jz::NvtxRange nv_build("jz build");
    rec(ix, 0);
    jz::Frame frame;
    {
      jz::NvtxRange nv("jz A1 frame");
      jz::compute_frame(pos, n, stride, ix->D, prm, &frame, st);
    }
    bmark("frame");
    rec(ix, 1);
    JZ_CUDA(cudaMallocAsync(&ix->pts, n * sizeof(float4), st));
    JZ_CUDA(cudaMallocAsync(&ix->keys, n * sizeof(uint64_t), st));
    JZ_CUDA(cudaMallocAsync(&ix->perm, n * sizeof(int32_t), st));
    bmark("alloc");
    {
      jz::NvtxRange nv("jz A2-A3 sort");
      jz::sort_points(pos, n, stride, gidx_mode, 0, frame, ix->keys, ix->perm, ix->pts, st);
    }
    bmark("sort");
    rec(ix, 2);
    {
      jz::NvtxRange nv("jz A4-A8 planes");
      jz::build_planes(ix->keys, ix->pts, n, prm, ix->planes, st);
    }
    bmark("planes");
    split_types(ix, gidx_mode != 0);
    bmark("types");
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

namespace jz {
void set_last_error(const std::string &m) { g_err = m; }
}  // namespace jz

#ifdef JZ_SEED_EXP
namespace jz { void exp_set_seed(const float *p); }
extern "C" __attribute__((visibility("default"))) void jz_exp_seed(const float *p) { jz::exp_set_seed(p); }
#endif
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
  *out = jz::build_impl(pos, n, 3, 0, n, box, p, (cudaStream_t)s);
  return JZ_OK;
  JZ_API_END
}

int jz_knn_build_xyzg(const float *pts4, int64_t n, int64_t n_query, const float *box, const jz_knn_params *p,
                      jz_stream_t s, jz_knn_index **out) {
  JZ_API_BEGIN
  if (!out) return fail(JZ_EINVAL, "out is NULL");
  *out = jz::build_impl(pts4, n, 4, 1, n_query, box, p, (cudaStream_t)s);
  return JZ_OK;
  JZ_API_END
}

int jz_knn_build_xq(const float *src, int64_t n_src, const float *qry, int64_t n_qry, const float *box,
                    const jz_knn_params *p, jz_stream_t s, jz_knn_index **out) {
  JZ_API_BEGIN
  if (!out || !src || (!qry && n_qry > 0)) return fail(JZ_EINVAL, "NULL argument");
  if (n_src < 1 || n_qry < 0 || n_src + n_qry > (int64_t)INT32_MAX - 1)
    return fail(JZ_EINVAL, "need n_src >= 1, n_qry >= 0, n_src + n_qry <= 2^31 - 2");
  cudaStream_t st = (cudaStream_t)s;
  init_pool();
  float4 *tmp = nullptr;
  JZ_CUDA(cudaMallocAsync(&tmp, (n_src + n_qry) * sizeof(float4), st));
  k_pack_xq<<<jz::grid_for(n_src + n_qry, 256), 256, 0, st>>>(qry, n_qry, src, n_src, tmp);
  JZ_LAUNCH_CHECK();
  try {
    *out = jz::build_impl(reinterpret_cast<const float *>(tmp), n_src + n_qry, 4, 1, n_qry, box, p, st);
  } catch (...) {
    cudaFreeAsync(tmp, st);
    throw;
  }
  JZ_CUDA(cudaFreeAsync(tmp, st));
  return JZ_OK;
  JZ_API_END
}

int jz_knn_rows(const jz_knn_index *ix, int64_t *m) {
  if (!ix || !m) return fail(JZ_EINVAL, "NULL argument");
  *m = ix->n_query;
  return JZ_OK;
}

static int query_impl(jz_knn_index *ix, int k, int order, int32_t *out_idx, float *out_d2, int32_t *out_row_gidx,
                      jz_stream_t s, int chunks, const std::function<void(int64_t, int64_t)> &on_rows) {
  if (!ix) return fail(JZ_EINVAL, "NULL index");
  if (ix->n_query > 0 && (!out_idx || !out_d2)) return fail(JZ_EINVAL, "NULL argument");
  if (k < 1) return fail(JZ_EINVAL, "k must be >= 1");
  if (k > ix->n_src) return fail(JZ_EINVAL, "k must not exceed the number of source points");
  if (order != JZ_ORDER_INPUT && order != JZ_ORDER_Z) return fail(JZ_EINVAL, "bad order");
  if (order == JZ_ORDER_Z && !out_row_gidx && ix->n_query > 0) return fail(JZ_EINVAL, "JZ_ORDER_Z needs out_row_gidx");
  cudaStream_t st = (cudaStream_t)s;
  ix->st = st;
  if (ix->n_query == 0) return JZ_OK;
  jz::NvtxRange nv_query("jz query");
  rec(ix, 4);
  jz::IList il;
  float *rmax2 = nullptr;
  int32_t *superbeg = nullptr;
  // walk down to plane 1: its nodes are the receiving parents of LeafToLeaf (jz_leaf.cu)
  {
    jz::NvtxRange nv("jz A9-A10 NodeToNode");
    jz::walk_to(ix->planes, ix->D, k, ix->prm.ngr, ix->prm.flags, 1, il, &rmax2, &superbeg, st, -1.f,
                ix->n_query < ix->n ? ix->qbeg : nullptr);
  }
  rec(ix, 5);
  if (!ix->d_evals) JZ_CUDA(cudaMallocAsync(&ix->d_evals, 16 * sizeof(unsigned long long), st));
  JZ_CUDA(cudaMemsetAsync(ix->d_evals, 0, 16 * sizeof(unsigned long long), st));
  const bool one_plane = ix->planes.size() == 1;
  jz::LeafArgs la;
  la.spts = ix->spts;
  la.sbeg = ix->sbeg;
  la.qpts = ix->qpts;
  la.qbeg = ix->qbeg;
  la.qin = ix->qin;
  la.leaf_box = ix->planes[0].box;
  la.nleaf = ix->planes[0].nnodes;
  la.par_leaf = one_plane ? superbeg : ix->planes[1].beg;
  la.par_box = one_plane ? nullptr : ix->planes[1].box;
  la.npar = il.nrecv;
  la.il = &il;
  la.rmax2 = rmax2;
  la.k = k;
  la.order = order;
  la.flags = ix->prm.flags;
  la.out_idx = out_idx;
  la.out_d2 = out_d2;
  la.out_row_gidx = out_row_gidx;
  la.evals = ix->d_evals;
  la.chunks = chunks;
  la.nq = ix->n_query;
  la.on_rows = on_rows;
  {
    jz::NvtxRange nv("jz A11-A12 LeafToLeaf");
    jz::leaf_to_leaf(la, ix->D, st);
  }
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
  if (getenv("JZ_DIAG_STATS") && ev[6]) {  // diagnostic builds (-DJZ_STATS=1): per-item own-pass / walk split
    const double it = (double)ev[6];
    fprintf(stderr, "JZ_STATS per item: appends %.1f (own %.1f) rounds %.1f (own %.1f) compactions %.2f (own %.2f) "
            "steps %.1f (own %.1f) passing %.1f (own %.1f) staged %.1f\n", ev[2] / it, ev[7] / it, ev[3] / it, ev[8] / it,
            ev[4] / it, ev[9] / it, ev[12] / it, ev[10] / it, ev[13] / it, ev[11] / it, ev[5] / it);
  }

  if (ix->timing) {
    cudaEventElapsedTime(&ix->times[3], ix->ev[4], ix->ev[5]);
    cudaEventElapsedTime(&ix->times[4], ix->ev[5], ix->ev[6]);
    ix->times[5] = ix->times[0] + ix->times[1] + ix->times[2] + ix->times[3] + ix->times[4];
  }
  return JZ_OK;
}

int jz_knn_query(jz_knn_index *ix, int k, int order, int32_t *out_idx, float *out_d2, int32_t *out_row_gidx,
                 jz_stream_t s) {
  JZ_API_BEGIN
  return query_impl(ix, k, order, out_idx, out_d2, out_row_gidx, s, 1, nullptr);
  JZ_API_END
}

void jz_knn_free(jz_knn_index *ix) {
  if (!ix) return;
  cudaStream_t st = ix->st;
  if (ix->own_s) {
    cudaFreeAsync(ix->spts, st);
    cudaFreeAsync(ix->sbeg, st);
  }
  if (ix->own_q) {
    cudaFreeAsync(ix->qpts, st);
    cudaFreeAsync(ix->qbeg, st);
    cudaFreeAsync(ix->qin, st);
  }
  jz::free_planes(ix->planes, st);
  if (ix->pts) cudaFreeAsync(ix->pts, st);
  if (ix->keys) cudaFreeAsync(ix->keys, st);
  if (ix->perm) cudaFreeAsync(ix->perm, st);
  if (ix->d_evals) cudaFreeAsync(ix->d_evals, st);
  if (ix->fof_label) cudaFreeAsync(ix->fof_label, st);
  if (ix->fof_root) cudaFreeAsync(ix->fof_root, st);
  if (ix->fof_count) cudaFreeAsync(ix->fof_count, st);
  if (ix->fof_com) cudaFreeAsync(ix->fof_com, st);
  if (ix->fof_rad) cudaFreeAsync(ix->fof_rad, st);
  cudaStreamSynchronize(st);
  for (auto &e : ix->ev)
    if (e) cudaEventDestroy(e);
  delete ix;
}

__global__ void k_iota_u32(uint32_t *__restrict__ a, int64_t n) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    a[i] = (uint32_t)i;
}
// group order: input id (.w) of the z position at each group-order slot
__global__ void k_group_order_out(const float4 *__restrict__ pts, const uint32_t *__restrict__ zpos, int64_t n,
                                  int32_t *__restrict__ order) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    order[i] = __float_as_int(pts[zpos[i]].w);
}
__global__ void k_group_heads(const uint32_t *__restrict__ root, int64_t n, int32_t *__restrict__ head) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    head[i] = (i == 0 || root[i] != root[i - 1]) ? 1 : 0;
}
__global__ void k_group_beg(const int32_t *__restrict__ head, const int64_t *__restrict__ off, int64_t n,
                            int32_t *__restrict__ beg) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    if (head[i]) beg[off[i]] = (int32_t)i;
}

namespace {
// owners released on every exit path (stream-ordered frees; the index syncs its stream)
struct DevBuf {
  void *p = nullptr;
  cudaStream_t st = nullptr;
  ~DevBuf() {
    if (p) cudaFreeAsync(p, st);
  }
};
struct IndexOwner {
  jz_knn_index *ix = nullptr;
  ~IndexOwner() { jz_knn_free(ix); }
};
}  // namespace

int jz_knn_search_host(const float *pos_host, int64_t n, const float *box, const jz_knn_params *p, int k,
                       int32_t *idx_host, float *d2_host, jz_stream_t s) {
  JZ_API_BEGIN
  if (!pos_host || !idx_host || !d2_host) return fail(JZ_EINVAL, "NULL argument");
  if (n < 1) return fail(JZ_EINVAL, "n must be >= 1");
  if (k < 1 || k > n) return fail(JZ_EINVAL, "k must be in [1, n]");
  cudaStream_t st = (cudaStream_t)s;
  init_pool();
  DevBuf dpos{nullptr, st}, didx{nullptr, st}, dd2{nullptr, st};
  IndexOwner own;
  // the large buffers first, in the same order every call: the stream-ordered pool then hands the
  // same blocks back (allocated after the build's temporaries they were split for them, and the
  // pool grew by gigabytes on some calls: 283-1340 ms per call instead of 278, tools/e2e_var.py)
  JZ_CUDA(cudaMallocAsync(&dpos.p, n * 3 * sizeof(float), st));
  JZ_CUDA(cudaMallocAsync(&didx.p, n * k * sizeof(int32_t), st));
  JZ_CUDA(cudaMallocAsync(&dd2.p, n * k * sizeof(float), st));
  JZ_CUDA(cudaMemcpyAsync(dpos.p, pos_host, n * 3 * sizeof(float), cudaMemcpyHostToDevice, st));
  int rc = jz_knn_build(static_cast<const float *>(dpos.p), n, box, p, s, &own.ix);
  if (rc != JZ_OK) return rc;
  rc = jz_knn_query(own.ix, k, JZ_ORDER_INPUT, static_cast<int32_t *>(didx.p), static_cast<float *>(dd2.p), nullptr, s);
  if (rc != JZ_OK) return rc;
  JZ_CUDA(cudaMemcpyAsync(idx_host, didx.p, n * k * sizeof(int32_t), cudaMemcpyDeviceToHost, st));
  JZ_CUDA(cudaMemcpyAsync(d2_host, dd2.p, n * k * sizeof(float), cudaMemcpyDeviceToHost, st));
  JZ_CUDA(cudaStreamSynchronize(st));
  return JZ_OK;
  JZ_API_END
}

int jz_knn_search_host_z(const float *pos_host, int64_t n, const float *box, const jz_knn_params *p, int k,
                         int32_t *idx_host, float *d2_host, int32_t *row_gidx_host, jz_stream_t s) {
  JZ_API_BEGIN
  if (!pos_host || !idx_host || !d2_host || !row_gidx_host) return fail(JZ_EINVAL, "NULL argument");
  if (n < 1) return fail(JZ_EINVAL, "n must be >= 1");
  if (k < 1 || k > n) return fail(JZ_EINVAL, "k must be in [1, n]");
  cudaStream_t st = (cudaStream_t)s;
  init_pool();
  static const bool hprof = getenv("JZ_HOST_PROF") != nullptr;
  const auto t0 = std::chrono::steady_clock::now();
  auto lap = [&](const char *what) {
    if (!hprof) return;
    cudaStreamSynchronize(st);
    fprintf(stderr, "  host_z %-10s %8.1f ms\n", what,
            std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count());
  };
  DevBuf dpos{nullptr, st}, didx{nullptr, st}, dd2{nullptr, st}, drg{nullptr, st};
  IndexOwner own;
  // the large buffers first (see jz_knn_search_host)
  JZ_CUDA(cudaMallocAsync(&dpos.p, n * 3 * sizeof(float), st));
  JZ_CUDA(cudaMallocAsync(&didx.p, n * k * sizeof(int32_t), st));
  JZ_CUDA(cudaMallocAsync(&dd2.p, n * k * sizeof(float), st));
  JZ_CUDA(cudaMallocAsync(&drg.p, n * sizeof(int32_t), st));
  lap("alloc");
  JZ_CUDA(cudaMemcpyAsync(dpos.p, pos_host, n * 3 * sizeof(float), cudaMemcpyHostToDevice, st));
  lap("h2d");
  int rc = jz_knn_build(static_cast<const float *>(dpos.p), n, box, p, s, &own.ix);
  if (rc != JZ_OK) return rc;
  lap("build");
  // rows of each finished chunk of work items (a contiguous z-order range) go to the host on a
  // second stream while the next chunk runs: the PCIe transfer overlaps LeafToLeaf
  struct Copier {
    cudaStream_t cs = nullptr;
    std::vector<cudaEvent_t> ev;
    ~Copier() {
      if (cs) cudaStreamSynchronize(cs);
      for (auto e : ev) cudaEventDestroy(e);
      if (cs) cudaStreamDestroy(cs);
    }
  } cp;
  JZ_CUDA(cudaStreamCreateWithFlags(&cp.cs, cudaStreamNonBlocking));
  auto *hi = idx_host;
  auto *hd = d2_host;
  auto *hr = row_gidx_host;
  const auto *gi = static_cast<const int32_t *>(didx.p);
  const auto *gd = static_cast<const float *>(dd2.p);
  const auto *gr = static_cast<const int32_t *>(drg.p);
  auto on_rows = [&](int64_t q0, int64_t q1) {
    cudaEvent_t e;
    JZ_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    cp.ev.push_back(e);
    JZ_CUDA(cudaEventRecord(e, st));
    JZ_CUDA(cudaStreamWaitEvent(cp.cs, e, 0));
    JZ_CUDA(cudaMemcpyAsync(hi + q0 * k, gi + q0 * k, (q1 - q0) * k * sizeof(int32_t), cudaMemcpyDeviceToHost, cp.cs));
    JZ_CUDA(cudaMemcpyAsync(hd + q0 * k, gd + q0 * k, (q1 - q0) * k * sizeof(float), cudaMemcpyDeviceToHost, cp.cs));
    JZ_CUDA(cudaMemcpyAsync(hr + q0, gr + q0, (q1 - q0) * sizeof(int32_t), cudaMemcpyDeviceToHost, cp.cs));
  };
  const int chunks = k <= jz::kMaxK ? 16 : 1;
  rc = query_impl(own.ix, k, JZ_ORDER_Z, static_cast<int32_t *>(didx.p), static_cast<float *>(dd2.p),
                  static_cast<int32_t *>(drg.p), s, chunks, on_rows);
  if (rc != JZ_OK) return rc;
  if (cp.ev.empty()) on_rows(0, n);  // not chunked (k > k_max): one copy at the end
  lap("query");
  JZ_CUDA(cudaStreamSynchronize(cp.cs));
  JZ_CUDA(cudaStreamSynchronize(st));
  lap("d2h done");
  return JZ_OK;
  JZ_API_END
}

int jz_fof(jz_knn_index *ix, float r_link, int32_t min_count, int32_t *labels, int64_t *ngroups, jz_stream_t s) {
  JZ_API_BEGIN
  if (!ix || !labels) return fail(JZ_EINVAL, "NULL argument");
  if (!(r_link >= 0.f) || !std::isfinite(r_link)) return fail(JZ_EINVAL, "r_link must be finite and >= 0");
  if (min_count < 1) return fail(JZ_EINVAL, "min_count must be >= 1");
  if (ix->n_query != ix->n || ix->n_src != ix->n || !ix->input_ids)
    return fail(JZ_EINVAL, "friends-of-friends needs an index built by jz_knn_build (every point a source and a query)");
  cudaStream_t st = (cudaStream_t)s;
  ix->st = st;
  const int64_t n = ix->n;
  const float b2 = r_link * r_link;  // RN32(r_link^2): the threshold on the canonical d2 (R21)
  rec(ix, 4);
  jz::IList il;
  float *rmax2 = nullptr;
  int32_t *superbeg = nullptr;
  int32_t *par = nullptr, *minlab = nullptr, *cnt = nullptr, *flag = nullptr;
  double *sum = nullptr, *ss = nullptr;
  int64_t *pos = nullptr;
  JZ_CUDA(cudaMallocAsync(&par, n * sizeof(int32_t), st));
  JZ_CUDA(cudaMallocAsync(&minlab, n * sizeof(int32_t), st));
  k_fof_init<<<jz::grid_for(n, 256), 256, 0, st>>>(par, minlab, n);
  JZ_LAUNCH_CHECK();
  jz::NvtxRange nv_fof("jz friends-of-friends");
  // node-level walk: ParentToNode, three-case NodeToNode with node links; linked
  // leaves' points start in their group (par), the remaining pairs go to the leaf stage
  jz::fof_walk(ix->planes, ix->D, ix->prm.ngr, b2, il, &superbeg, par, n, st);
  rec(ix, 5);
  if (!ix->d_evals) JZ_CUDA(cudaMallocAsync(&ix->d_evals, 16 * sizeof(unsigned long long), st));
  JZ_CUDA(cudaMemsetAsync(ix->d_evals, 0, 16 * sizeof(unsigned long long), st));
  const bool one_plane = ix->planes.size() == 1;
  jz::LeafArgs la{};
  la.spts = ix->pts;
  la.sbeg = ix->planes[0].beg;
  la.qpts = ix->pts;
  la.qbeg = ix->planes[0].beg;
  la.qin = ix->perm;
  la.leaf_box = ix->planes[0].box;
  la.nleaf = ix->planes[0].nnodes;
  la.par_leaf = one_plane ? superbeg : ix->planes[1].beg;
  la.par_box = one_plane ? nullptr : ix->planes[1].box;
  la.npar = il.nrecv;
  la.il = &il;
  la.flags = ix->prm.flags;
  la.evals = ix->d_evals;
  jz::fof_leaf(la, ix->D, b2, par, st);
  k_fof_flatten<<<jz::grid_for(n, 256), 256, 0, st>>>(par, n);
  JZ_LAUNCH_CHECK();
  k_fof_minlab<<<jz::grid_for(n, 256), 256, 0, st>>>(ix->pts, par, n, minlab);
  JZ_LAUNCH_CHECK();
  k_fof_labels<<<jz::grid_for(n, 256), 256, 0, st>>>(ix->pts, par, minlab, n, labels);
  JZ_LAUNCH_CHECK();
  // catalogue: groups with >= min_count points, in root z-order (the paper's group order)
  JZ_CUDA(cudaMallocAsync(&cnt, n * sizeof(int32_t), st));
  JZ_CUDA(cudaMallocAsync(&sum, 3 * n * sizeof(double), st));
  JZ_CUDA(cudaMallocAsync(&ss, n * sizeof(double), st));
  JZ_CUDA(cudaMallocAsync(&flag, n * sizeof(int32_t), st));
  JZ_CUDA(cudaMallocAsync(&pos, (n + 1) * sizeof(int64_t), st));
  JZ_CUDA(cudaMemsetAsync(cnt, 0, n * sizeof(int32_t), st));
  JZ_CUDA(cudaMemsetAsync(sum, 0, 3 * n * sizeof(double), st));
  JZ_CUDA(cudaMemsetAsync(ss, 0, n * sizeof(double), st));
  k_fof_sum1<<<jz::grid_for(n, kFofThreads), kFofThreads, 0, st>>>(ix->pts, par, n, ix->D, cnt, sum);
  JZ_LAUNCH_CHECK();
  k_fof_sum2<<<jz::grid_for(n, kFofThreads), kFofThreads, 0, st>>>(ix->pts, par, n, ix->D, cnt, sum, ss);
  JZ_LAUNCH_CHECK();
  k_fof_flags<<<jz::grid_for(n, 256), 256, 0, st>>>(par, cnt, n, min_count, flag);
  JZ_LAUNCH_CHECK();
  jz::exclusive_scan_i32_to_i64(flag, pos, n, st);
  const int64_t ng = jz::read_i64(pos + n, st);
  if (ix->fof_label) JZ_CUDA(cudaFreeAsync(ix->fof_label, st));
  if (ix->fof_count) JZ_CUDA(cudaFreeAsync(ix->fof_count, st));
  if (ix->fof_com) JZ_CUDA(cudaFreeAsync(ix->fof_com, st));
  if (ix->fof_rad) JZ_CUDA(cudaFreeAsync(ix->fof_rad, st));
  const int64_t ga = ng > 0 ? ng : 1;
  JZ_CUDA(cudaMallocAsync(&ix->fof_label, ga * sizeof(int32_t), st));
  JZ_CUDA(cudaMallocAsync(&ix->fof_count, ga * sizeof(int32_t), st));
  JZ_CUDA(cudaMallocAsync(&ix->fof_com, 3 * ga * sizeof(double), st));
  JZ_CUDA(cudaMallocAsync(&ix->fof_rad, ga * sizeof(double), st));
  k_fof_cat<<<jz::grid_for(n, 256), 256, 0, st>>>(ix->pts, flag, pos, minlab, cnt, sum, ss, n, ix->D, ix->fof_label,
                                                  ix->fof_count, ix->fof_com, ix->fof_rad);
  JZ_LAUNCH_CHECK();
  ix->fof_ngroups = ng;
  rec(ix, 6);
  il.release(st);
  if (rmax2) JZ_CUDA(cudaFreeAsync(rmax2, st));
  if (superbeg) JZ_CUDA(cudaFreeAsync(superbeg, st));
  for (void *p : {(void *)minlab, (void *)cnt, (void *)sum, (void *)ss, (void *)flag, (void *)pos})
    JZ_CUDA(cudaFreeAsync(p, st));
  if (ix->fof_root) JZ_CUDA(cudaFreeAsync(ix->fof_root, st));
  ix->fof_root = par;  // roots (flattened) kept for jz_fof_group_order
  unsigned long long ev = 0;
  JZ_CUDA(cudaMemcpyAsync(&ev, ix->d_evals, sizeof(ev), cudaMemcpyDeviceToHost, st));
  JZ_CUDA(cudaStreamSynchronize(st));
  ix->evals = (long long)ev;
  if (ix->timing) {
    cudaEventElapsedTime(&ix->times[3], ix->ev[4], ix->ev[5]);
    cudaEventElapsedTime(&ix->times[4], ix->ev[5], ix->ev[6]);
    ix->times[5] = ix->times[0] + ix->times[1] + ix->times[2] + ix->times[3] + ix->times[4];
  }
  if (ngroups) *ngroups = ng;
  return JZ_OK;
  JZ_API_END
}

int jz_fof_catalogue(const jz_knn_index *ix, int64_t cap, int32_t *label, int32_t *count, double *com, double *rad,
                     jz_stream_t s) {
  JZ_API_BEGIN
  if (!ix) return fail(JZ_EINVAL, "NULL index");
  const int64_t ng = ix->fof_ngroups;
  if (cap < ng) return fail(JZ_ECAPACITY, "catalogue capacity below the number of groups");
  if (ng > 0 && (!label || !count || !com || !rad)) return fail(JZ_EINVAL, "NULL argument");
  cudaStream_t st = (cudaStream_t)s;
  if (ng > 0) {
    JZ_CUDA(cudaMemcpyAsync(label, ix->fof_label, ng * sizeof(int32_t), cudaMemcpyDeviceToDevice, st));
    JZ_CUDA(cudaMemcpyAsync(count, ix->fof_count, ng * sizeof(int32_t), cudaMemcpyDeviceToDevice, st));
    JZ_CUDA(cudaMemcpyAsync(com, ix->fof_com, 3 * ng * sizeof(double), cudaMemcpyDeviceToDevice, st));
    JZ_CUDA(cudaMemcpyAsync(rad, ix->fof_rad, ng * sizeof(double), cudaMemcpyDeviceToDevice, st));
  }
  return JZ_OK;
  JZ_API_END
}

int jz_fof_group_order(const jz_knn_index *ix, int32_t *order, int32_t *group_beg, int64_t *ngroups_all,
                       jz_stream_t s) {
  JZ_API_BEGIN
  if (!ix || !order) return fail(JZ_EINVAL, "NULL argument");
  if (!ix->fof_root) return fail(JZ_EINVAL, "no friends-of-friends result in this index (call jz_fof first)");
  cudaStream_t st = (cudaStream_t)s;
  const int64_t n = ix->n;
  // stable sort of the z positions by their root z position: roots stay in z order and
  // every group is a contiguous block, internally in z order
  DevBuf iota{nullptr, st}, skey{nullptr, st}, sval{nullptr, st}, flag{nullptr, st}, off{nullptr, st};
  JZ_CUDA(cudaMallocAsync(&iota.p, n * sizeof(uint32_t), st));
  JZ_CUDA(cudaMallocAsync(&skey.p, n * sizeof(uint32_t), st));
  JZ_CUDA(cudaMallocAsync(&sval.p, n * sizeof(uint32_t), st));
  k_iota_u32<<<jz::grid_for(n, 256), 256, 0, st>>>(static_cast<uint32_t *>(iota.p), n);
  JZ_LAUNCH_CHECK();
  jz::sort_pairs_u32(reinterpret_cast<const uint32_t *>(ix->fof_root), static_cast<const uint32_t *>(iota.p), n,
                     static_cast<uint32_t *>(skey.p), static_cast<uint32_t *>(sval.p), st);
  k_group_order_out<<<jz::grid_for(n, 256), 256, 0, st>>>(ix->pts, static_cast<const uint32_t *>(sval.p), n, order);
  JZ_LAUNCH_CHECK();
  if (group_beg || ngroups_all) {  // group starts: positions where the root changes
    JZ_CUDA(cudaMallocAsync(&flag.p, n * sizeof(int32_t), st));
    JZ_CUDA(cudaMallocAsync(&off.p, (n + 1) * sizeof(int64_t), st));
    k_group_heads<<<jz::grid_for(n, 256), 256, 0, st>>>(static_cast<const uint32_t *>(skey.p), n,
                                                        static_cast<int32_t *>(flag.p));
    JZ_LAUNCH_CHECK();
    jz::exclusive_scan_i32_to_i64(static_cast<int32_t *>(flag.p), static_cast<int64_t *>(off.p), n, st);
    const int64_t ng = jz::read_i64(static_cast<int64_t *>(off.p) + n, st);
    if (group_beg) {
      k_group_beg<<<jz::grid_for(n, 256), 256, 0, st>>>(static_cast<const int32_t *>(flag.p),
                                                        static_cast<const int64_t *>(off.p), n, group_beg);
      JZ_LAUNCH_CHECK();
      const int32_t nn = (int32_t)n;
      JZ_CUDA(cudaMemcpyAsync(group_beg + ng, &nn, sizeof(int32_t), cudaMemcpyHostToDevice, st));
    }
    if (ngroups_all) *ngroups_all = ng;
  }
  JZ_CUDA(cudaStreamSynchronize(st));
  return JZ_OK;
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
