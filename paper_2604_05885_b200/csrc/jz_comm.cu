// jz_comm.cu -- communicators of the multi-GPU path (SURVEY.md §8(b) comm bootstrap, §8(e)
// exchanges; PAPER.md L388-393 distributed kNN, L112 sample-splitter partition).
//
// jz_comm is the library's collective layer: one rank per GPU. Two implementations:
//   * NCCL (jz_comm_unique_id / jz_comm_init): libnccl.so.2 is opened at run time (dlopen: the
//     library loads without NCCL; in a torch process the already-loaded NCCL is reused). The
//     unique id is created on rank 0 and broadcast by the caller (torch.distributed), as in
//     ncclCommInitRank's usual bootstrap.
//   * in-process logical ranks (jz_comm_local_world / jz_comm_init_local): R threads of one
//     process on one device exchange device buffers through a shared table with barriers.
//     The multi-GPU orchestration (jz_dist.cu) runs unchanged on it: the tests use it to run
//     R = 1..8 ranks on one B200.
// Collectives: all-gather of fixed-size device blocks, all-to-all-v of device buffers (grouped
// point-to-point sends / receives), all-reduce of small host vectors (min / max / sum).
#include <dlfcn.h>

#include <chrono>
#include <condition_variable>
#include <cstdlib>
#include <cstring>
#include <ctime>
#include <mutex>
#include <vector>

#include "jz_comm.h"

namespace jz {

// ---------------------------------------------------------------- NCCL (run-time loaded)
namespace {
struct NcclId {
  char internal[128];
};
typedef int (*p_get_unique_id)(NcclId *);
typedef int (*p_comm_init_rank)(void **, int, NcclId, int);
typedef int (*p_comm_destroy)(void *);
typedef int (*p_all_gather)(const void *, void *, size_t, int, void *, cudaStream_t);
typedef int (*p_all_reduce)(const void *, void *, size_t, int, int, void *, cudaStream_t);
typedef int (*p_send)(const void *, size_t, int, int, void *, cudaStream_t);
typedef int (*p_recv)(void *, size_t, int, int, void *, cudaStream_t);
typedef int (*p_group)();
typedef const char *(*p_err)(int);
enum { kNcclUint8 = 1, kNcclInt64 = 4, kNcclFloat64 = 8 };
enum { kNcclSum = 0, kNcclMax = 2, kNcclMin = 3 };

struct NcclApi {
  bool ok = false;
  std::string why;
  p_get_unique_id get_unique_id = nullptr;
  p_comm_init_rank comm_init_rank = nullptr;
  p_comm_destroy comm_destroy = nullptr;
  p_all_gather all_gather = nullptr;
  p_all_reduce all_reduce = nullptr;
  p_send send = nullptr;
  p_recv recv = nullptr;
  p_group group_start = nullptr, group_end = nullptr;
  p_err err = nullptr;
};

NcclApi &nccl() {
  static NcclApi a;
  static std::once_flag once;
  std::call_once(once, [] {
    void *h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      a.why = std::string("cannot open libnccl.so.2: ") + dlerror();
      return;
    }
#define JZ_SYM(f, n)                                        \
  a.f = reinterpret_cast<decltype(a.f)>(dlsym(h, n));       \
  if (!a.f) {                                               \
    a.why = std::string("libnccl lacks ") + n;              \
    return;                                                 \
  }
    JZ_SYM(get_unique_id, "ncclGetUniqueId");
    JZ_SYM(comm_init_rank, "ncclCommInitRank");
    JZ_SYM(comm_destroy, "ncclCommDestroy");
    JZ_SYM(all_gather, "ncclAllGather");
    JZ_SYM(all_reduce, "ncclAllReduce");
    JZ_SYM(send, "ncclSend");
    JZ_SYM(recv, "ncclRecv");
    JZ_SYM(group_start, "ncclGroupStart");
    JZ_SYM(group_end, "ncclGroupEnd");
    JZ_SYM(err, "ncclGetErrorString");
#undef JZ_SYM
    a.ok = true;
  });
  return a;
}

void nccl_check(int r, const char *what) {
  if (r != 0) throw Error(JZ_ENCCL, std::string(what) + ": " + (nccl().err ? nccl().err(r) : "NCCL error"));
}

struct NcclComm : Comm {
  void *c = nullptr;
  double *scratch = nullptr;  // small host-vector all-reduces
  int scap = 0;
  ~NcclComm() override {
    if (scratch) cudaFree(scratch);
    if (c) nccl().comm_destroy(c);
  }
  void all_gather(const void *send, void *recv, size_t bytes, cudaStream_t st) override {
    nccl_check(nccl().all_gather(send, recv, bytes, kNcclUint8, c, st), "ncclAllGather");
  }
  void all_to_all_v(const void *send, const int64_t *scount, const int64_t *soff, void *recv, const int64_t *rcount,
                    const int64_t *roff, size_t elem, cudaStream_t st) override {
    nccl_check(nccl().group_start(), "ncclGroupStart");
    for (int r = 0; r < size; ++r) {
      if (scount[r] > 0)
        nccl_check(nccl().send(static_cast<const char *>(send) + soff[r] * elem, scount[r] * elem, kNcclUint8, r, c, st),
                   "ncclSend");
      if (rcount[r] > 0)
        nccl_check(nccl().recv(static_cast<char *>(recv) + roff[r] * elem, rcount[r] * elem, kNcclUint8, r, c, st),
                   "ncclRecv");
    }
    nccl_check(nccl().group_end(), "ncclGroupEnd");
  }
  void all_reduce_host(double *v, int n, jz::RedOp op, cudaStream_t st) override {
    if (n > scap) {
      if (scratch) JZ_CUDA(cudaFree(scratch));
      JZ_CUDA(cudaMalloc(&scratch, n * sizeof(double)));
      scap = n;
    }
    JZ_CUDA(cudaMemcpyAsync(scratch, v, n * sizeof(double), cudaMemcpyHostToDevice, st));
    const int o = op == RedOp::kMin ? kNcclMin : (op == RedOp::kMax ? kNcclMax : kNcclSum);
    nccl_check(nccl().all_reduce(scratch, scratch, n, kNcclFloat64, o, c, st), "ncclAllReduce");
    JZ_CUDA(cudaMemcpyAsync(v, scratch, n * sizeof(double), cudaMemcpyDeviceToHost, st));
    JZ_CUDA(cudaStreamSynchronize(st));
  }
  void all_reduce_max_i32(int32_t *dev, int64_t n, cudaStream_t st) override {
    // int32 max as the bytes of non-negative flags: use float64-free path via int64? NCCL has int32 (2)
    nccl_check(nccl().all_reduce(dev, dev, (size_t)n, 2 /* ncclInt32 */, kNcclMax, c, st), "ncclAllReduce");
  }
};
}  // namespace

// ---------------------------------------------------------------- in-process logical ranks
struct LocalWorld {
  int R;
  std::mutex mu;
  std::condition_variable cv;
  int arrived = 0;
  long gen = 0;
  bool aborted = false;  // a rank failed: every barrier throws instead of waiting for it
  // serial mode (JZ_LOCAL_SERIAL=1 at world creation): a rank runs device work only while it
  // holds the token, so the ranks' compute segments do not overlap on the shared device and
  // each rank's busy time is its uncontended per-rank time (tools/dist_phases.py)
  bool serial = false;
  std::mutex token;
  std::vector<const void *> ptr;
  std::vector<std::vector<int64_t>> meta;
  std::vector<std::vector<double>> vals;
  explicit LocalWorld(int r) : R(r), ptr(r), meta(r), vals(r) {
    const char *e = getenv("JZ_LOCAL_SERIAL");
    serial = e && e[0] == '1';
  }
  static double now() {
    timespec t;
    clock_gettime(CLOCK_MONOTONIC, &t);
    return t.tv_sec * 1e3 + t.tv_nsec * 1e-6;
  }
  void barrier(double *busy = nullptr, double *t_in = nullptr) {
    if (serial && busy) {
      *busy += now() - *t_in;
      token.unlock();
    }
    struct Relock {  // re-take the token on every exit path
      LocalWorld *w;
      double *busy, *t_in;
      ~Relock() {
        if (w->serial && busy) {
          w->token.lock();
          *t_in = now();
        }
      }
    } relock{this, busy, t_in};
    std::unique_lock<std::mutex> lk(mu);
    if (aborted) throw Error(JZ_ECUDA, "a peer logical rank failed");
    const long g = gen;
    if (++arrived == R) {
      arrived = 0;
      ++gen;
      cv.notify_all();
    } else if (!cv.wait_for(lk, std::chrono::seconds(900), [&] { return gen != g || aborted; }) || aborted) {
      aborted = true;
      cv.notify_all();
      throw Error(JZ_ECUDA, "a peer logical rank failed or timed out");
    }
  }
  void abort() {
    std::lock_guard<std::mutex> lk(mu);
    aborted = true;
    cv.notify_all();
  }
};

namespace {
struct LocalComm : Comm {
  LocalWorld *w = nullptr;
  double t_in = 0;
  void abort() override { w->abort(); }
  void enter() override {
    if (w->serial) {
      w->token.lock();
      t_in = LocalWorld::now();
    }
  }
  void leave(cudaStream_t st) override {
    if (w->serial) {
      cudaStreamSynchronize(st);
      busy_ms += LocalWorld::now() - t_in;
      w->token.unlock();
    }
  }
  void bar() { w->barrier(&busy_ms, &t_in); }
  void all_gather(const void *send, void *recv, size_t bytes, cudaStream_t st) override {
    JZ_CUDA(cudaStreamSynchronize(st));  // the block is complete before peers read it
    w->ptr[rank] = send;
    bar();
    for (int r = 0; r < size; ++r)
      if (bytes)
        JZ_CUDA(cudaMemcpyAsync(static_cast<char *>(recv) + r * bytes, w->ptr[r], bytes, cudaMemcpyDeviceToDevice, st));
    JZ_CUDA(cudaStreamSynchronize(st));
    bar();  // peers may now reuse their send blocks
  }
  void all_to_all_v(const void *send, const int64_t *scount, const int64_t *soff, void *recv, const int64_t *rcount,
                    const int64_t *roff, size_t elem, cudaStream_t st) override {
    JZ_CUDA(cudaStreamSynchronize(st));
    w->ptr[rank] = send;
    w->meta[rank].assign(soff, soff + size);
    bar();
    for (int r = 0; r < size; ++r)
      if (rcount[r] > 0)
        JZ_CUDA(cudaMemcpyAsync(static_cast<char *>(recv) + roff[r] * elem,
                                static_cast<const char *>(w->ptr[r]) + w->meta[r][rank] * elem, rcount[r] * elem,
                                cudaMemcpyDeviceToDevice, st));
    JZ_CUDA(cudaStreamSynchronize(st));
    bar();
    (void)scount;
  }
  void all_reduce_host(double *v, int n, jz::RedOp op, cudaStream_t st) override {
    JZ_CUDA(cudaStreamSynchronize(st));  // no device work of this rank outlives its token
    w->vals[rank].assign(v, v + n);
    bar();
    for (int i = 0; i < n; ++i) {
      double a = w->vals[0][i];
      for (int r = 1; r < size; ++r) {
        const double b = w->vals[r][i];
        a = op == RedOp::kMin ? (b < a ? b : a) : (op == RedOp::kMax ? (b > a ? b : a) : a + b);
      }
      v[i] = a;
    }
    bar();
  }
  void all_reduce_max_i32(int32_t *dev, int64_t n, cudaStream_t st) override;
};

__global__ void k_max_i32(int32_t *__restrict__ acc, const int32_t *__restrict__ x, int64_t n) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    acc[i] = max(acc[i], x[i]);
}

void LocalComm::all_reduce_max_i32(int32_t *dev, int64_t n, cudaStream_t st) {
  int32_t *acc = nullptr;
  JZ_CUDA(cudaMallocAsync(&acc, (n > 0 ? n : 1) * sizeof(int32_t), st));
  JZ_CUDA(cudaStreamSynchronize(st));
  w->ptr[rank] = dev;
  bar();
  JZ_CUDA(cudaMemcpyAsync(acc, w->ptr[0], n * sizeof(int32_t), cudaMemcpyDeviceToDevice, st));
  for (int r = 1; r < size; ++r) {
    k_max_i32<<<grid_for(n, 256), 256, 0, st>>>(acc, static_cast<const int32_t *>(w->ptr[r]), n);
    JZ_LAUNCH_CHECK();
  }
  JZ_CUDA(cudaStreamSynchronize(st));
  bar();  // every rank has read every input
  JZ_CUDA(cudaMemcpyAsync(dev, acc, n * sizeof(int32_t), cudaMemcpyDeviceToDevice, st));
  JZ_CUDA(cudaFreeAsync(acc, st));
  JZ_CUDA(cudaStreamSynchronize(st));
}
}  // namespace

}  // namespace jz

void jz_comm::all_gather_i64_host(const int64_t *v, int n, int64_t *out, cudaStream_t st) {
  int64_t *d = nullptr;
  JZ_CUDA(cudaMallocAsync(&d, (size_t)n * (size + 1) * sizeof(int64_t), st));
  JZ_CUDA(cudaMemcpyAsync(d, v, n * sizeof(int64_t), cudaMemcpyHostToDevice, st));
  all_gather(d, d + n, n * sizeof(int64_t), st);
  JZ_CUDA(cudaMemcpyAsync(out, d + n, (size_t)n * size * sizeof(int64_t), cudaMemcpyDeviceToHost, st));
  JZ_CUDA(cudaFreeAsync(d, st));
  JZ_CUDA(cudaStreamSynchronize(st));
}

struct jz_comm_world {
  jz::LocalWorld w;
  explicit jz_comm_world(int r) : w(r) {}
};

extern "C" {

int jz_comm_unique_id(uint8_t id[128]) {
  if (!id) return JZ_EINVAL;
  auto &a = jz::nccl();
  if (!a.ok) {
    jz::set_last_error(a.why);
    return JZ_ENCCL;
  }
  jz::NcclId u;
  const int r = a.get_unique_id(&u);
  if (r != 0) {
    jz::set_last_error(std::string("ncclGetUniqueId: ") + a.err(r));
    return JZ_ENCCL;
  }
  memcpy(id, u.internal, 128);
  return JZ_OK;
}

int jz_comm_init(const uint8_t id[128], int nranks, int rank, jz_comm **out) {
  if (!id || !out || nranks < 1 || nranks > 32 || rank < 0 || rank >= nranks) {
    jz::set_last_error("jz_comm_init: bad argument (1 <= nranks <= 32, 0 <= rank < nranks)");
    return JZ_EINVAL;
  }
  auto &a = jz::nccl();
  if (!a.ok) {
    jz::set_last_error(a.why);
    return JZ_ENCCL;
  }
  jz::NcclId u;
  memcpy(u.internal, id, 128);
  auto *c = new jz::NcclComm();
  c->rank = rank;
  c->size = nranks;
  const int r = a.comm_init_rank(&c->c, nranks, u, rank);
  if (r != 0) {
    jz::set_last_error(std::string("ncclCommInitRank: ") + a.err(r));
    c->c = nullptr;
    delete c;
    return JZ_ENCCL;
  }
  *out = c;
  return JZ_OK;
}

int jz_comm_local_world(int nranks, jz_comm_world **out) {
  if (!out || nranks < 1 || nranks > 32) {
    jz::set_last_error("jz_comm_local_world: 1 <= nranks <= 32");
    return JZ_EINVAL;
  }
  *out = new jz_comm_world(nranks);
  return JZ_OK;
}

int jz_comm_init_local(jz_comm_world *w, int rank, jz_comm **out) {
  if (!w || !out || rank < 0 || rank >= w->w.R) {
    jz::set_last_error("jz_comm_init_local: bad argument");
    return JZ_EINVAL;
  }
  auto *c = new jz::LocalComm();
  c->w = &w->w;
  c->rank = rank;
  c->size = w->w.R;
  *out = c;
  return JZ_OK;
}

int jz_comm_rank_size(const jz_comm *c, int32_t *rank, int32_t *size) {
  if (!c || !rank || !size) return JZ_EINVAL;
  *rank = c->rank;
  *size = c->size;
  return JZ_OK;
}

void jz_comm_free(jz_comm *c) { delete c; }

void jz_comm_world_free(jz_comm_world *w) { delete w; }

}  // extern "C"
