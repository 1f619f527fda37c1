// jz_comm.h -- the collective layer of the multi-GPU path (jz_comm.cu): the C ABI's opaque
// jz_comm is this abstract class; NCCL and in-process logical ranks implement it.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "jz_internal.h"

namespace jz {
enum class RedOp { kMin, kMax, kSum };
struct LocalWorld;
}  // namespace jz

struct jz_comm {
  int rank = 0, size = 1;
  virtual ~jz_comm() {}
  // every rank contributes `bytes` from send (device); recv (device) gets size * bytes, rank order
  virtual void all_gather(const void *send, void *recv, size_t bytes, cudaStream_t st) = 0;
  // device buffers; counts / offsets (host, elements) per peer; rcount[r] == peer r's scount[me]
  virtual void all_to_all_v(const void *send, const int64_t *scount, const int64_t *soff, void *recv,
                            const int64_t *rcount, const int64_t *roff, size_t elem, cudaStream_t st) = 0;
  // small host vectors (frames, counts, timings)
  virtual void all_reduce_host(double *v, int n, jz::RedOp op, cudaStream_t st) = 0;
  // element-wise max of a device int32 vector (hit flags)
  virtual void all_reduce_max_i32(int32_t *dev, int64_t n, cudaStream_t st) = 0;
  // this rank failed inside a collective sequence: release the peers (logical ranks); NCCL
  // peers are left to the caller (the error code is returned on every rank that sees it)
  virtual void abort() {}
  // a collective API call begins / ends on this rank (serial logical ranks take the device token)
  virtual void enter() {}
  virtual void leave(cudaStream_t st) { (void)st; }
  double busy_ms = 0;  // serial logical ranks: accumulated device-busy wall time of this rank
  // out (host) = size * n values, rank order
  void all_gather_i64_host(const int64_t *v, int n, int64_t *out, cudaStream_t st);
};

namespace jz {
using Comm = ::jz_comm;
}
