// jz_scan.cu -- device exclusive scan (CumulativeSumPrep0, Alg. 2 line 3 / L350-352)
// used for interaction-list offsets and stream compaction. Reduce-then-scan in three
// launches: per-tile sums, a single-block scan of the tile sums, per-tile rescan + add.
#include "jz_common.cuh"

namespace jz {

constexpr int kScanThreads = 256;
constexpr int kScanIPT = 8;
constexpr int kScanTile = kScanThreads * kScanIPT;

template <typename T>
__device__ __forceinline__ T warp_incl_scan(T v) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    T u = __shfl_up_sync(0xffffffffu, v, o);
    if (lane >= o) v += u;
  }
  return v;
}

// block-wide exclusive scan of one value per thread; returns exclusive prefix, *total = block sum
template <typename T>
__device__ __forceinline__ T block_excl_scan(T v, T *total) {
  __shared__ T s_w[33];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  T inc = warp_incl_scan(v);
  if (lane == 31) s_w[w] = inc;
  __syncthreads();
  if (w == 0) {
    T x = lane < nw ? s_w[lane] : T(0);
    T xi = warp_incl_scan(x);
    if (lane < nw) s_w[lane] = xi - x;
    if (lane == nw - 1) s_w[32] = xi;
  }
  __syncthreads();
  T r = inc - v + s_w[w];
  *total = s_w[32];
  __syncthreads();
  return r;
}

__global__ void k_scan_tilesum(const int32_t *__restrict__ in, int64_t n, int64_t *__restrict__ tsum) {
  int64_t base = (int64_t)blockIdx.x * kScanTile;
  int64_t s = 0;
#pragma unroll
  for (int i = 0; i < kScanIPT; ++i) {
    int64_t idx = base + (int64_t)i * kScanThreads + threadIdx.x;
    if (idx < n) s += in[idx];
  }
  int64_t tot;
  block_excl_scan<int64_t>(s, &tot);
  if (threadIdx.x == 0) tsum[blockIdx.x] = tot;
}

__global__ void k_scan_tiles(int64_t *__restrict__ tsum, int64_t ntiles) {
  // single block: exclusive scan of tile sums in place, tsum[ntiles] = grand total
  int64_t carry = 0;
  for (int64_t b = 0; b < ntiles; b += blockDim.x) {
    int64_t i = b + threadIdx.x;
    int64_t v = i < ntiles ? tsum[i] : 0;
    int64_t tot;
    int64_t ex = block_excl_scan<int64_t>(v, &tot);
    if (i < ntiles) tsum[i] = carry + ex;
    carry += tot;
  }
  if (threadIdx.x == 0) tsum[ntiles] = carry;
}

__global__ void k_scan_apply(const int32_t *__restrict__ in, int64_t n, const int64_t *__restrict__ tsum,
                             int64_t *__restrict__ out) {
  // blocked arrangement: thread t owns items [t*IPT, t*IPT+IPT) of the tile (reads via smem transpose)
  __shared__ int32_t s_v[kScanTile];
  int64_t base = (int64_t)blockIdx.x * kScanTile;
#pragma unroll
  for (int i = 0; i < kScanIPT; ++i) {
    int64_t idx = base + (int64_t)i * kScanThreads + threadIdx.x;
    s_v[i * kScanThreads + threadIdx.x] = idx < n ? in[idx] : 0;
  }
  __syncthreads();
  int64_t loc[kScanIPT];
  int64_t s = 0;
#pragma unroll
  for (int i = 0; i < kScanIPT; ++i) {
    loc[i] = s;
    s += s_v[threadIdx.x * kScanIPT + i];
  }
  int64_t tot;
  int64_t ex = block_excl_scan<int64_t>(s, &tot) + tsum[blockIdx.x];
  __syncthreads();
  // write back through smem as int64 would double smem; write directly (stride IPT*8 B per thread)
#pragma unroll
  for (int i = 0; i < kScanIPT; ++i) {
    int64_t idx = base + (int64_t)threadIdx.x * kScanIPT + i;
    if (idx < n) out[idx] = ex + loc[i];
  }
  if (blockIdx.x == gridDim.x - 1 && threadIdx.x == 0) out[n] = tsum[gridDim.x];
}

void exclusive_scan_i32_to_i64(const int32_t *in, int64_t *out, int64_t n, cudaStream_t st) {
  int64_t ntiles = ceil_div(n, kScanTile);
  if (ntiles < 1) ntiles = 1;
  int64_t *tsum = nullptr;
  JZ_CUDA(cudaMallocAsync(&tsum, (ntiles + 1) * sizeof(int64_t), st));
  k_scan_tilesum<<<(unsigned)ntiles, kScanThreads, 0, st>>>(in, n, tsum);
  JZ_LAUNCH_CHECK();
  k_scan_tiles<<<1, 1024, 0, st>>>(tsum, ntiles);
  JZ_LAUNCH_CHECK();
  k_scan_apply<<<(unsigned)ntiles, kScanThreads, 0, st>>>(in, n, tsum, out);
  JZ_LAUNCH_CHECK();
  JZ_CUDA(cudaFreeAsync(tsum, st));
}

int64_t read_i64(const int64_t *dev, cudaStream_t st) {
  int64_t v = 0;
  JZ_CUDA(cudaMemcpyAsync(&v, dev, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
  JZ_CUDA(cudaStreamSynchronize(st));
  return v;
}

}  // namespace jz
