// jz_common.cuh -- shared device/host helpers of the CUDA path (never used by oracle/).
//
// Distance of record (R1; PAPER.md L432 float32): per axis
//   t = RN(q - s); periodic: t >= h -> RN(t - L), t < -h -> RN(t + L)  (h = L/2)
//   d2 = fma(tz, tz, fma(ty, ty, tx * tx))
// written with explicit __f*_rn intrinsics so nvcc can neither contract nor reorder.
//
// Node bounds (d_low / d_up) are evaluated on FP32 AABBs with the
// SAME rounded operations, so they bound the canonical d2 of every point pair exactly
// (R8): RN is monotone, so for q in [A.lo, A.hi], s in [B.lo, B.hi]
// RN(q - s) lies in [RN(A.lo - B.hi), RN(A.hi - B.lo)]; the wrapped magnitude is a
// tent function of t, so its min/max over that interval sit at the endpoints (or 0 / h);
// fma and mul are monotone in |t|. No safety margins are needed.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>
#include <stdexcept>
#include <string>

namespace jz {

constexpr int kKeyBits = 21;          // bits per axis (R4)
constexpr int kLevelSentinel = 64;    // level of boundary gaps (> 63, R5)
constexpr int kMaxK = 32;             // k_max
constexpr int kMaxLeaf = 128;         // largest supported N_max^(0)

struct Error : std::runtime_error {
  int code;
  Error(int c, const std::string &m) : std::runtime_error(m), code(c) {}
};

#define JZ_CUDA(call)                                                                                      \
  do {                                                                                                     \
    cudaError_t e_ = (call);                                                                               \
    if (e_ != cudaSuccess)                                                                                 \
      throw ::jz::Error(e_ == cudaErrorMemoryAllocation ? 7 : 5,                                            \
                        std::string(#call) + ": " + cudaGetErrorString(e_) + " at " + __FILE__ + ":" +      \
                            std::to_string(__LINE__));                                                     \
  } while (0)

// NVTX range for the host-side phases (visible in Nsight Systems / ncu --nvtx; no cost without
// an attached tool)
struct NvtxRange {
  explicit NvtxRange(const char *name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange &) = delete;
  NvtxRange &operator=(const NvtxRange &) = delete;
};

// every kernel launch is followed by JZ_LAUNCH_CHECK(); it also counts launches (jz_launch_count)
void count_launch();
#define JZ_LAUNCH_CHECK()       \
  do {                          \
    ::jz::count_launch();       \
    JZ_CUDA(cudaGetLastError()); \
  } while (0)

// Periodic domain (or open when periodic == 0).
struct Dom {
  int periodic;
  float L[3];
  float h[3];
};

struct NodeBox {  // 32 B per node: lo.xyz + point count, hi.xyz + unused
  float4 lo;
  float4 hi;
};

__device__ __forceinline__ float wrapt(float t, float L, float h) {
  return t >= h ? __fsub_rn(t, L) : (t < -h ? __fadd_rn(t, L) : t);
}

__device__ __forceinline__ float canon_d2_open(float qx, float qy, float qz, float sx, float sy, float sz) {
  float tx = __fsub_rn(qx, sx), ty = __fsub_rn(qy, sy), tz = __fsub_rn(qz, sz);
  return __fmaf_rn(tz, tz, __fmaf_rn(ty, ty, __fmul_rn(tx, tx)));
}

__device__ __forceinline__ float canon_d2_per(float qx, float qy, float qz, float sx, float sy, float sz,
                                              const Dom &D) {
  float tx = wrapt(__fsub_rn(qx, sx), D.L[0], D.h[0]);
  float ty = wrapt(__fsub_rn(qy, sy), D.L[1], D.h[1]);
  float tz = wrapt(__fsub_rn(qz, sz), D.L[2], D.h[2]);
  return __fmaf_rn(tz, tz, __fmaf_rn(ty, ty, __fmul_rn(tx, tx)));
}

// min over q in [alo,ahi], s in [blo,bhi] of |wrap(RN(q - s))|
__device__ __forceinline__ float axis_low(float alo, float ahi, float blo, float bhi, int periodic, float L,
                                          float h) {
  float tmin = __fsub_rn(alo, bhi), tmax = __fsub_rn(ahi, blo);
  if (tmin <= 0.f && tmax >= 0.f) return 0.f;
  if (!periodic) return tmin > 0.f ? tmin : -tmax;
  return fminf(fabsf(wrapt(tmin, L, h)), fabsf(wrapt(tmax, L, h)));
}

// max over the same set
__device__ __forceinline__ float axis_up(float alo, float ahi, float blo, float bhi, int periodic, float L,
                                         float h) {
  float tmin = __fsub_rn(alo, bhi), tmax = __fsub_rn(ahi, blo);
  if (!periodic) return fmaxf(fabsf(tmin), fabsf(tmax));
  if ((tmin <= h && tmax >= h) || (tmin <= -h && tmax >= -h)) return h;
  return fmaxf(fabsf(wrapt(tmin, L, h)), fabsf(wrapt(tmax, L, h)));
}

__device__ __forceinline__ float box_dlow2(const NodeBox &a, const NodeBox &b, const Dom &D) {
  float gx = axis_low(a.lo.x, a.hi.x, b.lo.x, b.hi.x, D.periodic, D.L[0], D.h[0]);
  float gy = axis_low(a.lo.y, a.hi.y, b.lo.y, b.hi.y, D.periodic, D.L[1], D.h[1]);
  float gz = axis_low(a.lo.z, a.hi.z, b.lo.z, b.hi.z, D.periodic, D.L[2], D.h[2]);
  return __fmaf_rn(gz, gz, __fmaf_rn(gy, gy, __fmul_rn(gx, gx)));
}

__device__ __forceinline__ float box_dup2(const NodeBox &a, const NodeBox &b, const Dom &D) {
  float ux = axis_up(a.lo.x, a.hi.x, b.lo.x, b.hi.x, D.periodic, D.L[0], D.h[0]);
  float uy = axis_up(a.lo.y, a.hi.y, b.lo.y, b.hi.y, D.periodic, D.L[1], D.h[1]);
  float uz = axis_up(a.lo.z, a.hi.z, b.lo.z, b.hi.z, D.periodic, D.L[2], D.h[2]);
  return __fmaf_rn(uz, uz, __fmaf_rn(uy, uy, __fmul_rn(ux, ux)));
}

// point-to-box lower bound: min over s in [lo, hi] of the canonical d2(q, s) (exact, as above)
__device__ __forceinline__ float pt_box_dlow2(float qx, float qy, float qz, const NodeBox &b, const Dom &D) {
  float gx = axis_low(qx, qx, b.lo.x, b.hi.x, D.periodic, D.L[0], D.h[0]);
  float gy = axis_low(qy, qy, b.lo.y, b.hi.y, D.periodic, D.L[1], D.h[1]);
  float gz = axis_low(qz, qz, b.lo.z, b.hi.z, D.periodic, D.L[2], D.h[2]);
  return __fmaf_rn(gz, gz, __fmaf_rn(gy, gy, __fmul_rn(gx, gx)));
}

__device__ __forceinline__ int box_count(const NodeBox &b) { return __float_as_int(b.lo.w); }

__host__ __device__ inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

inline unsigned grid_for(int64_t n, int threads, int64_t cap = 148 * 64) {
  int64_t g = ceil_div(n, threads);
  if (g < 1) g = 1;
  if (g > cap) g = cap;
  return (unsigned)g;
}

// ---------------------------------------------------------------- launchers (host)
struct Frame {  // Morton quantisation q_d = trunc(clamp(RN(RN(x - o_d) * s_d), 0, 2^21-1))
  float o[3];
  float s[3];
};

// scan.cu
void exclusive_scan_i32_to_i64(const int32_t *in, int64_t *out, int64_t n, cudaStream_t st);  // out has n+1
int64_t read_i64(const int64_t *dev, cudaStream_t st);

}  // namespace jz
