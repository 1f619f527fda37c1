// jz_leaf.cu -- LeafToLeaf (Alg. 1 line 6 L321, L386, L398).
//
// B200 design:
//  * Work item = 32 consecutive (z-order) query points of one receiving plane-1 node J, one
//    query per lane, one warp per item; warps are independent (no CTA barriers).
//    The item walks J's plane-1 interaction list (sorted by r_low): the leaf-level
//    NodeToNode pass is not materialised. Leaf pairs are pruned on the fly: the bounding box
//    of the warp's queries is tested against each source node S and then, one lane per child
//    leaf, against S's child leaves (a ballot gives the survivors), and every lane tests its
//    own query against each survivor (the early exit of P:L398, per lane).
//  * Pruning bounds use centre / half-extent boxes whose extents carry an absolute rounding
//    margin, and the bound is scaled by (1 - 2^-19): branch-free, and never above the
//    canonical d2 of any pair in the boxes (R8b).
//  * Surviving leaves are staged by the warp into its own shared-memory slot as separate
//    x / y / z / gidx arrays (coalesced 16-byte loads, leaf starts aligned to 4, tails padded
//    with NaN coordinates so their d2 is NaN and never passes a comparison).
//  * Distances: two sources per packed f32x2 instruction, query coordinate as the broadcast
//    operand: FADD2 x3, FMUL2, FFMA2 x2 per source pair = the canonical scalar formula with
//    per-element round-to-nearest (bit-identical). Periodic leaf pairs whose pairs all wrap
//    the same way get one extra exact FADD2 per axis; straddling pairs use the per-pair select.
//  * Top-k: each lane keeps the K smallest d2 VALUES in a sorted register
//    list updated by a min/max bubble (2 FMNMX per slot, no predicates) and appends every
//    candidate with d2 <= its current k-th value to a lane-private log in shared memory
//    (key = d2_bits << 32 | gidx + 1, so unsigned order == (d2, index) order, R2).
//    The log is compacted to the entries <= the current k-th value when it fills; at the end
//    the k smallest keys of the log are the row (bitonic sort in registers). The list starts
//    full of R_max^2(J), which bounds every contained query's k-th distance.
//  * Rows are written straight to their final place (input or z order): no reorder pass.
#include <cstdio>
#include <vector>

#include "jz_common.cuh"
#include "jz_internal.h"

namespace jz {

#ifndef JZ_LWARPS
#define JZ_LWARPS 1  // one work item per CTA: CTAs retire independently (2 warps: 132.5 ms, 1: 127.0 ms)
#endif
constexpr int kLWarps = JZ_LWARPS;  // warps (independent work items) per LeafToLeaf CTA
constexpr int kLThreads = kLWarps * 32;
#ifndef JZ_LCAP
#define JZ_LCAP 128
#endif
#ifndef JZ_MINB
#define JZ_MINB 18  // 18 one-warp CTAs per SM: 96 registers (5 warps per SM partition; smem allows 18 at K = 16)
#endif
constexpr int kLCap = JZ_LCAP;  // staged source points per warp (2 KB SoA); >= the largest leaf (kMaxLeaf)
static_assert(JZ_LCAP >= kMaxLeaf, "a leaf must fit the staging buffer");

#ifndef JZ_LOGX
#define JZ_LOGX 16  // K = 16: 32-entry log (10 KB per one-warp CTA with staging)
#endif
#ifndef JZ_STATS
#define JZ_STATS 0  // per-lane walk counters (appends, merge rounds, compactions): diagnostic builds (tools/mkvar.py)
#endif

#ifndef JZ_WIN_SMEM
#define JZ_WIN_SMEM 0  // 1: z-window read from the staged own block when it fits one batch (measured slower: 104.6 vs 102.9 ms)
#endif

#ifndef JZ_VEC_ROWS
#define JZ_VEC_ROWS 2  // 2: rows staged in shared memory, 8 whole rows per warp store; 1: 128-bit stores per lane; 0: scalar (119.5 -> 107.3 -> 106.8 ms)
#endif

#ifndef JZ_FOF_FULL
#define JZ_FOF_FULL 0  // 1: link whole (item, leaf) pairs within R_link without evaluating them (measured slower at 10^8 C4: 104 vs 89 ms)
#endif

#ifndef JZ_MERGE_T
#define JZ_MERGE_T 0  // > 0: merge at a batch end only when some lane has >= JZ_MERGE_T new log entries
#endif

#ifndef JZ_LANE_TEST
#define JZ_LANE_TEST 1  // per-lane point-box test of each leaf that passes the warp-box test
#endif

#ifndef JZ_LOGX32
#define JZ_LOGX32 16  // K = 32: 48-entry log (14 KB per warp with staging) -> 7 CTAs per SM
#endif
#ifndef JZ_MINB32
#define JZ_MINB32 14  // K = 32: 144 registers, no spills (the K = 16 budget of 96 spilled: C3 48 -> 33 ms)
#endif
template <int K>
struct LogCap {
  static constexpr int C = K + (K > 16 ? JZ_LOGX32 : JZ_LOGX);  // log entries per lane
};
#ifndef JZ_MINB8
#define JZ_MINB8 JZ_MINB
#endif
template <int K>
struct MinBlocks {
  static constexpr int v = K > 16 ? JZ_MINB32 : (K <= 8 ? JZ_MINB8 : JZ_MINB);  // CTAs per SM the register budget targets
};

typedef unsigned long long u64;

__device__ __forceinline__ u64 pk(float lo, float hi) {
  u64 r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
  return r;
}
__device__ __forceinline__ void upk(u64 v, float &lo, float &hi) {
  asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(v));
}
__device__ __forceinline__ u64 sub2(u64 a, u64 b) {
  u64 d;
  asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
__device__ __forceinline__ u64 add2(u64 a, u64 b) {
  u64 d;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
__device__ __forceinline__ u64 mul2(u64 a, u64 b) {
  u64 d;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
__device__ __forceinline__ u64 fma2(u64 a, u64 b, u64 c) {
  u64 d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  return d;
}

// ---------------------------------------------------------------- pruning bounds
// Box as centre c and half extent e, e including an absolute margin m >= 2^-18 * (largest
// coordinate magnitude of the box, or L when periodic). For any q in box A and s in box B the
// canonical per-axis difference t = wrap(RN(q - s)) satisfies |t| >= gap = max(0, |c_A - c_B|
// (minimal image) - e_A - e_B): the margin absorbs the rounding of c, e, RN(q - s) and of the
// gap itself. The sum of squares is then scaled by (1 - 2^-19) to absorb the relative error
// of the rounded squares, so dlow2 <= canonical d2(q, s) for every pair (R8b).
struct CE {
  float4 c;  // centre (w unused)
  float4 e;  // half extent + margin (w unused)
};

constexpr float kLowScale = 1.0f - 1.0f / 524288.0f;  // 1 - 2^-19

template <bool PER>
__device__ __forceinline__ float gap1(float dc, float E, float L) {
  float a = fabsf(dc);
  if (PER) a = fminf(a, __fsub_rn(L, a));
  return fmaxf(__fsub_rn(a, E), 0.f);
}

template <bool PER>
__device__ __forceinline__ float dlow2_ce(float dcx, float dcy, float dcz, float Ex, float Ey, float Ez, const Dom &D) {
  const float gx = gap1<PER>(dcx, Ex, D.L[0]);
  const float gy = gap1<PER>(dcy, Ey, D.L[1]);
  const float gz = gap1<PER>(dcz, Ez, D.L[2]);
  return __fmul_rn(__fmaf_rn(gz, gz, __fmaf_rn(gy, gy, __fmul_rn(gx, gx))), kLowScale);
}

// per-axis periodic shift class of a box pair from the signed centre difference dc and the
// summed extents E (margins included): every pair's RN(q - s) lies in [dc - E, dc + E].
// 0 = no pair wraps, 1 = every pair wraps by -L, 2 = every pair wraps by +L, 3 = straddles.
__device__ __forceinline__ int ce_class(float dc, float E, float h) {
  const float tlo = __fsub_rn(dc, E), thi = __fadd_rn(dc, E);
  if (tlo >= h) return 1;
  if (thi < -h) return 2;
  if (tlo >= -h && thi < h) return 0;
  return 3;
}

__device__ __forceinline__ bool any_straddle(int c) {
  return ((c & 3) == 3) || (((c >> 2) & 3) == 3) || (((c >> 4) & 3) == 3);
}
__device__ __forceinline__ float class_shift(int c, float L) { return c == 1 ? -L : (c == 2 ? L : 0.f); }

__device__ __forceinline__ float ce_margin(float lx, float ly, float lz, float hx, float hy, float hz, float Lmax) {
  float m = fmaxf(fmaxf(fmaxf(fabsf(lx), fabsf(hx)), fmaxf(fabsf(ly), fabsf(hy))), fmaxf(fabsf(lz), fabsf(hz)));
  return __fmul_ru(fmaxf(m, Lmax), 1.0f / 262144.0f);  // 2^-18
}

__device__ __forceinline__ CE make_ce(float lx, float ly, float lz, float hx, float hy, float hz, float Lmax) {
  const float m = ce_margin(lx, ly, lz, hx, hy, hz, Lmax);
  CE r;
  r.c = make_float4(__fmul_rn(__fadd_rn(lx, hx), 0.5f), __fmul_rn(__fadd_rn(ly, hy), 0.5f),
                    __fmul_rn(__fadd_rn(lz, hz), 0.5f), 0.f);
  r.e = make_float4(__fadd_ru(__fmul_ru(__fsub_ru(hx, lx), 0.5f), m), __fadd_ru(__fmul_ru(__fsub_ru(hy, ly), 0.5f), m),
                    __fadd_ru(__fmul_ru(__fsub_ru(hz, lz), 0.5f), m), 0.f);
  return r;
}

__global__ void k_box_ce(const NodeBox *__restrict__ box, int64_t n, float Lmax, CE *__restrict__ out) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const NodeBox b = box[i];
    out[i] = make_ce(b.lo.x, b.lo.y, b.lo.z, b.hi.x, b.hi.y, b.hi.z, Lmax);
  }
}

// insert value d into the sorted list F, dropping the largest (identity when d >= F[K-1]):
// F'[j] = max(F[j-1], min(F[j], d)), F'[0] = min(F[0], d) -- every slot independent (depth 2, no
// serial chain); the lower half runs only when some lane's d lands there (late insertions land
// in the upper half). Warp-converged callers only.
template <int K>
__device__ __forceinline__ void bubble(float (&F)[K], float d) {
  constexpr int J0 = K / 2;
#pragma unroll
  for (int j = K - 1; j >= J0 && j > 0; --j) F[j] = fmaxf(F[j - 1], fminf(F[j], d));
  if (__any_sync(0xffffffffu, d < F[J0 > 0 ? J0 - 1 : 0])) {
#pragma unroll
    for (int j = J0 - 1; j > 0; --j) F[j] = fmaxf(F[j - 1], fminf(F[j], d));
    F[0] = fminf(F[0], d);
  }
}

// insert two values a <= b at once: F'[j] = max(F[j-2], min(F[j-1], b), min(F[j], a)) (the
// (j+1)-th smallest of F, a, b), 3 instructions per slot for two insertions; same gating.
template <int K>
__device__ __forceinline__ void bubble2(float (&F)[K], float a, float b) {
  constexpr int J0 = K / 2;
#pragma unroll
  for (int j = K - 1; j >= J0 && j > 1; --j) F[j] = fmaxf(fmaxf(F[j - 2], fminf(F[j - 1], b)), fminf(F[j], a));
  if (__any_sync(0xffffffffu, a < F[J0 > 0 ? J0 - 1 : 0])) {
#pragma unroll
    for (int j = J0 - 1; j > 1; --j) F[j] = fmaxf(fmaxf(F[j - 2], fminf(F[j - 1], b)), fminf(F[j], a));
    if (K > 1) F[1] = fmaxf(fminf(F[0], b), fminf(F[1], a));
    F[0] = fminf(F[0], a);
  }
}

#ifdef JZ_DIAG_WALK
__device__ unsigned long long g_diag[8];  // [0] entries reached [1] entries passing the node test [2] 32-leaf chunks
                                           // [3] leaves passing the warp test [4] leaves staged [5] items
#define JZ_DIAG(i, v) (((threadIdx.x & 31) == 0) ? (void)atomicAdd(&g_diag[i], (unsigned long long)(v)) : (void)0)
#else
#define JZ_DIAG(i, v) ((void)0)
#endif

template <int K>
struct WarpBuf {
  float x[kLCap + 8], y[kLCap + 8], z[kLCap + 8];  // + 8: padding to a multiple of 8
  int g[kLCap + 8];
  u64 lk[LogCap<K>::C][32];  // log: keys d2_bits << 32 | gidx + 1 (lane-minor: conflict-free)
};

template <int K, bool LB>
struct Lane {
  float F[K];  // K smallest d2 values seen (ascending); F[K-1] = current k-th value
  u64 lb;      // keys <= lb were found by earlier passes (0 on the first pass)
  float kth;   // F[K-1] (inactive lanes: -1, never passes a comparison)
  int nl;      // log entries
  int nf;      // log entries already merged into F
  unsigned ins;
  unsigned app;   // log appends (lane)
  unsigned rnd;   // merge rounds (warp-uniform)
  unsigned cmp;   // compactions (warp-uniform)
  unsigned stg;   // staged leaves (warp-uniform)
  unsigned stp;   // 8-source eval steps (warp-uniform, JZ_STATS)
  unsigned pst;   // steps whose vote passed (warp-uniform, JZ_STATS)
  bool act;
};

#ifndef JZ_MERGE_NET
#define JZ_MERGE_NET 0  // > 0: merges with >= JZ_MERGE_NET new entries in some lane use the 8-value network
#endif
template <int K>
__device__ __forceinline__ void net_merge8(float (&F)[K], float (&N)[8]);

// merge the lane's new log entries into F (all lanes in lockstep: max(new) rounds)
template <int K, bool LB>
__device__ __forceinline__ void merge(WarpBuf<K> &B, Lane<K, LB> &L) {
  const int lane = threadIdx.x & 31;
  const int nr = (int)__reduce_max_sync(0xffffffffu, (unsigned)(L.nl - L.nf));
  if (JZ_STATS) L.rnd += nr;
  int i = 0;
#if JZ_MERGE_NET > 0
  // many new entries in some lane: 8 at a time through the sort / bitonic-merge network
#pragma unroll 1
  for (; nr - i >= JZ_MERGE_NET; i += 8) {
    float N[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int r = L.nf + i + u;
      N[u] = __uint_as_float(r < L.nl ? (unsigned)(B.lk[r][lane] >> 32) : 0x7f800000u);
    }
    net_merge8<K>(L.F, N);
  }
#endif
#pragma unroll 1
  for (; i < nr; i += 2) {  // two entries per round
    const int r = L.nf + i;
    const float d1 = __uint_as_float(r < L.nl ? (unsigned)(B.lk[r][lane] >> 32) : 0x7f800000u);
    const float d2 = __uint_as_float(r + 1 < L.nl ? (unsigned)(B.lk[r + 1][lane] >> 32) : 0x7f800000u);
    const float lo = fminf(d1, d2), hi = fmaxf(d1, d2);
    const bool in = lo < L.F[K - 1];
    if (__any_sync(0xffffffffu, in)) bubble2<K>(L.F, lo, hi);
    if (JZ_STATS) L.ins += in + (hi < L.F[K - 1]);
  }
  L.nf = L.nl;
  L.kth = L.act ? L.F[K - 1] : -1.f;
}

// keep only the log entries with d2 <= k-th value; with massive exact ties at the k-th value
// drop the largest keys until K remain (they cannot be among the K smallest keys)
template <int K>
__device__ __noinline__ int drop_largest(WarpBuf<K> &B, int nl, int keep) {
  const int lane = threadIdx.x & 31;
  while (nl > keep) {
    int im = 0;
    u64 mk = 0;
    for (int r = 0; r < nl; ++r) {
      const u64 e = B.lk[r][lane];
      if (e > mk) {
        mk = e;
        im = r;
      }
    }
    B.lk[im][lane] = B.lk[nl - 1][lane];
    --nl;
  }
  return nl;
}

template <int K, bool LB>
__device__ __forceinline__ void compact(WarpBuf<K> &B, Lane<K, LB> &L) {
  constexpr int C = LogCap<K>::C;
  const int lane = threadIdx.x & 31;
  if (JZ_STATS) ++L.cmp;
  merge<K, LB>(B, L);
  const unsigned kb = __float_as_uint(L.kth);
  const int r1 = (int)__reduce_max_sync(0xffffffffu, (unsigned)L.nl);
  int j = 0;
#pragma unroll 1
  for (int r = 0; r < r1; r += 4) {  // 4 independent loads per step
    u64 e[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) e[u] = r + u < L.nl ? B.lk[r + u][lane] : ~0ull;
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      if ((unsigned)(e[u] >> 32) <= kb) {  // ~0 (no entry) never passes: kb <= 0x7f800000 or inactive
        B.lk[j][lane] = e[u];
        ++j;
      }
    }
  }
  L.nl = L.nf = j;
  if (__any_sync(0xffffffffu, j > C - 8)) L.nl = L.nf = drop_largest<K>(B, L.nl, K);
}

template <int K, bool LB>
__device__ __forceinline__ void append(WarpBuf<K> &B, Lane<K, LB> &L, float d2, int g) {
  if (d2 <= L.kth) {
    const u64 key = ((u64)__float_as_uint(d2) << 32) | (unsigned)(g + 1);
    if (!LB || key > L.lb) {
      B.lk[L.nl][threadIdx.x & 31] = key;
      ++L.nl;
      if (JZ_STATS) ++L.app;
    }
  }
}

template <int K, bool LB>
__device__ __forceinline__ void append_chk(WarpBuf<K> &B, Lane<K, LB> &L, float d2, int g) {
  append<K, LB>(B, L, d2, g);
  if (__any_sync(0xffffffffu, L.nl > LogCap<K>::C - 8)) compact<K, LB>(B, L);  // keep nl <= C - 8 between steps
}

// ---------------------------------------------------------------- distance evaluation
// d2 of 4 staged sources [j, j+4) against the lane's query (packed: 2 sources per instruction)
__device__ __forceinline__ void d2x4(const float *bx, const float *by, const float *bz, int j, u64 QX, u64 QY, u64 QZ,
                                     bool shift, u64 SX, u64 SY, u64 SZ, float &a0, float &a1, float &a2, float &a3) {
  const float4 X = *reinterpret_cast<const float4 *>(&bx[j]);
  const float4 Y = *reinterpret_cast<const float4 *>(&by[j]);
  const float4 Z = *reinterpret_cast<const float4 *>(&bz[j]);
  u64 tx0 = sub2(QX, pk(X.x, X.y)), tx1 = sub2(QX, pk(X.z, X.w));
  u64 ty0 = sub2(QY, pk(Y.x, Y.y)), ty1 = sub2(QY, pk(Y.z, Y.w));
  u64 tz0 = sub2(QZ, pk(Z.x, Z.y)), tz1 = sub2(QZ, pk(Z.z, Z.w));
  if (shift) {  // warp-uniform
    tx0 = add2(tx0, SX);
    tx1 = add2(tx1, SX);
    ty0 = add2(ty0, SY);
    ty1 = add2(ty1, SY);
    tz0 = add2(tz0, SZ);
    tz1 = add2(tz1, SZ);
  }
  const u64 d0 = fma2(tz0, tz0, fma2(ty0, ty0, mul2(tx0, tx0)));
  const u64 d1 = fma2(tz1, tz1, fma2(ty1, ty1, mul2(tx1, tx1)));
  upk(d0, a0, a1);
  upk(d1, a2, a3);
}

template <int MW>
__device__ __forceinline__ void mask4(int j, int wl, float &a0, float &a1, float &a2, float &a3) {
  if constexpr (MW > 0) {
    const unsigned u = (unsigned)(j - wl);
    const float nan = __int_as_float(0x7fc00000);
    if (u < (unsigned)MW) a0 = nan;
    if (u + 1u < (unsigned)MW) a1 = nan;
    if (u + 2u < (unsigned)MW) a2 = nan;
    if (u + 3u < (unsigned)MW) a3 = nan;
  }
}

// staged sources [0, n) (n multiple of 8, NaN padded) against the lane's query; 8 sources per
// step (two independent packed chains) and one vote. shift: every pair wraps by (shx, shy, shz)
// (exact, warp-uniform); mw > 0: skip the lane's own window of mw staged sources starting at
// staged index wl (already in the list, see window_init). One copy of this loop per call site:
// the flags are runtime (warp-uniform) to keep the hot code small (instruction cache).
template <int K, bool LB>
__device__ __forceinline__ void eval_block(WarpBuf<K> &B, int n, float qx, float qy, float qz, bool shift, float shx,
                                           float shy, float shz, Lane<K, LB> &L, int mw, int wl) {
  constexpr int C = LogCap<K>::C;
  const u64 QX = pk(qx, qx), QY = pk(qy, qy), QZ = pk(qz, qz);
  const u64 SX = pk(shx, shx), SY = pk(shy, shy), SZ = pk(shz, shz);
#pragma unroll 1
  for (int j = 0; j < n; j += 8) {
    float a0, a1, a2, a3, b0, b1, b2, b3;
    d2x4(B.x, B.y, B.z, j, QX, QY, QZ, shift, SX, SY, SZ, a0, a1, a2, a3);
    d2x4(B.x, B.y, B.z, j + 4, QX, QY, QZ, shift, SX, SY, SZ, b0, b1, b2, b3);
    if (mw > 0) {
      const unsigned u = (unsigned)(j - wl);
      const float nan = __int_as_float(0x7fc00000);
      a0 = u < (unsigned)mw ? nan : a0;
      a1 = u + 1u < (unsigned)mw ? nan : a1;
      a2 = u + 2u < (unsigned)mw ? nan : a2;
      a3 = u + 3u < (unsigned)mw ? nan : a3;
      b0 = u + 4u < (unsigned)mw ? nan : b0;
      b1 = u + 5u < (unsigned)mw ? nan : b1;
      b2 = u + 6u < (unsigned)mw ? nan : b2;
      b3 = u + 7u < (unsigned)mw ? nan : b3;
    }
    const float m = fminf(fminf(fminf(a0, a1), fminf(a2, a3)), fminf(fminf(b0, b1), fminf(b2, b3)));  // NaN ignored
    if (JZ_STATS) ++L.stp;
    if (__any_sync(0xffffffffu, m <= L.kth)) {
      if (JZ_STATS) ++L.pst;
      const int4 G = *reinterpret_cast<const int4 *>(&B.g[j]);
      const int4 H = *reinterpret_cast<const int4 *>(&B.g[j + 4]);
      append<K, LB>(B, L, a0, G.x);
      append<K, LB>(B, L, a1, G.y);
      append<K, LB>(B, L, a2, G.z);
      append<K, LB>(B, L, a3, G.w);
      append<K, LB>(B, L, b0, H.x);
      append<K, LB>(B, L, b1, H.y);
      append<K, LB>(B, L, b2, H.z);
      append<K, LB>(B, L, b3, H.w);
      if (__any_sync(0xffffffffu, L.nl > C - 8)) compact<K, LB>(B, L);
    }
  }
  // refresh the k-th value for the next pruning decisions (merge rounds = max new entries)
#if JZ_MERGE_T > 0
  if (__any_sync(0xffffffffu, L.nl - L.nf >= JZ_MERGE_T))
#endif
  merge<K, LB>(B, L);
}

// pad a staged batch [0, n) (n multiple of 4) with NaN sources to a multiple of 8
template <int K>
__device__ __forceinline__ int pad8(WarpBuf<K> &B, int n) {
  const int lane = threadIdx.x & 31;
  if (n & 4) {
    if (lane < 4) {
      const float nan = __int_as_float(0x7fc00000);
      B.x[n + lane] = nan;
      B.y[n + lane] = nan;
      B.z[n + lane] = nan;
      B.g[n + lane] = 0;
    }
    n += 4;
  }
  return n;
}

// asynchronous 4-byte global -> shared copies (LDGSTS): every source of a batch is in flight at
// once and no registers hold staged data; cp.async.wait_all + __syncwarp before the batch is read
__device__ __forceinline__ void cpa4(void *sdst, const void *gsrc) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(sdst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(sa), "l"(gsrc) : "memory");
}
__device__ __forceinline__ void cpa_wait() { asm volatile("cp.async.wait_all;" ::: "memory"); }

// stage m sources (float4 {x, y, z, bits(gidx)} at src) into slots [n, n + mp) as SoA; the
// slots [n + m, n + mp) (mp = m rounded up to 4) get NaN coordinates
template <int K>
__device__ __forceinline__ void stage_async(WarpBuf<K> &B, int n, const float4 *__restrict__ src, int m, int mp) {
  const int lane = threadIdx.x & 31;
  for (int t = lane; t < mp; t += 32) {
    if (t < m) {
      const float *p = reinterpret_cast<const float *>(src + t);
      cpa4(&B.x[n + t], p);
      cpa4(&B.y[n + t], p + 1);
      cpa4(&B.z[n + t], p + 2);
      cpa4(&B.g[n + t], p + 3);
    } else {
      const float nan = __int_as_float(0x7fc00000);
      B.x[n + t] = nan;
      B.y[n + t] = nan;
      B.z[n + t] = nan;
      B.g[n + t] = 0;
    }
  }
}

template <int K, bool LB, int MW = 0>
__device__ __forceinline__ void eval_generic(WarpBuf<K> &B, int n, float qx, float qy, float qz, const Dom &D,
                                             Lane<K, LB> &L, int wl = 0) {
  for (int j = 0; j < n; ++j) {
    float d2 = canon_d2_per(qx, qy, qz, B.x[j], B.y[j], B.z[j], D);  // NaN padding -> NaN
    if constexpr (MW > 0) {
      if ((unsigned)(j - wl) < (unsigned)MW) d2 = __int_as_float(0x7fc00000);
    }
    append_chk<K, LB>(B, L, d2, B.g[j]);
  }
  merge<K, LB>(B, L);
}

struct LeafPK {
  const float4 *spts;        // source points, z order (type-separated)
  const int32_t *sbeg;       // [nleaf+1] first source of each leaf
  const float4 *qpts;        // query points, z order
  const int32_t *qbeg;       // [nleaf+1] first query of each leaf
  const int32_t *qin;        // [nq] input row of each query
  const CE *leaf_ce;         // [nleaf]
  const int32_t *par_leaf;   // [npar+1] first leaf of each receiving parent
  const CE *par_ce;          // [npar] or nullptr
  const int64_t *ispl;       // parent-level interaction list
  const int32_t *isrc;
  const float *rlow;
  const float *rmax2;        // [npar] or nullptr (= +inf)
  const int32_t *item_par;   // [nitems] receiving parent of each 32-query work item
  const int32_t *item_q0;    // [nitems] first query (sorted position) of the item
  int64_t nitems;            // end of the launched item range
  int64_t item_off;          // first item of the launched range (chunked launches)
  float Lmax;  // periodic: largest box length (margin scale); open: 0
  int k;       // neighbours found by this pass (<= K)
  int col0;    // first output column of this pass (k > k_max chunking)
  int ldo;     // output row stride (total k)
  int order;
  int early;
  int sorted;
  int32_t *out_idx;
  float *out_d2;
  int32_t *out_row_gidx;
  int self;    // queries == sources (self-query): enables the z-window initialisation
  unsigned long long *stats;  // counters (jz_knn_stats) or nullptr
  unsigned long long *counter;  // JZ_PERSIST work-item counter of this launch (zeroed) or nullptr
};

// Pending batch of staged source leaves (one periodic shift class), carried across source nodes
// so that batches are full: n staged slots, c0 their class.
struct Batch {
  int n;
  int c0;
};

// evaluate the pending batch against the lane's query and refresh the k-th value
template <int K, bool LB, bool PER>
__device__ __forceinline__ void flush(WarpBuf<K> &B, Batch &W, float qx, float qy, float qz, const Dom &D,
                                      Lane<K, LB> &L) {
  if (W.n == 0) return;
  const int n = pad8<K>(B, W.n);
  cpa_wait();
  __syncwarp();
  const int c0 = W.c0;
  if (!PER || !any_straddle(c0)) {  // no axis straddles: no wrap, or a uniform exact shift
    eval_block<K, LB>(B, n, qx, qy, qz, PER && c0 != 0, class_shift(c0 & 3, D.L[0]), class_shift((c0 >> 2) & 3, D.L[1]),
                      class_shift((c0 >> 4) & 3, D.L[2]), L, 0, 0);
  } else {
    eval_generic<K, LB>(B, n, qx, qy, qz, D, L);
  }
  __syncwarp();
  W.n = 0;
}

// Visit the child leaves [la, lb) of one source node, skipping [xa, xb): one lane tests one
// leaf against the warp's query box (bound vs the warp's current max k-th value), then every
// lane tests its own query against each surviving leaf (skip unless some lane needs it);
// survivors are appended to the pending batch (asynchronous copies), which is evaluated when
// it is full, when the shift class changes, or at the end of the walk.
template <int K, bool LB, bool PER>
__device__ __forceinline__ void visit_leaves(const LeafPK &a, const Dom &D, WarpBuf<K> &B, Batch &W, const CE &wb,
                                             float wmax, int la, int lb, int xa, int xb, float qx, float qy, float qz,
                                             bool act, Lane<K, LB> &L, unsigned long long &nev) {
  const int lane = threadIdx.x & 31;
  for (int l0 = la; l0 < lb; l0 += 32) {
    const int l = l0 + lane;
    bool pass = false;
    int cls = 0, s0 = 0, s1 = 0;
    float cx = 0.f, cy = 0.f, cz = 0.f, ex = 0.f, ey = 0.f, ez = 0.f;
    if (l < lb && (l < xa || l >= xb)) {
      const CE lc = a.leaf_ce[l];
      cx = lc.c.x;
      cy = lc.c.y;
      cz = lc.c.z;
      ex = lc.e.x;
      ey = lc.e.y;
      ez = lc.e.z;
      const float dcx = __fsub_rn(wb.c.x, cx), dcy = __fsub_rn(wb.c.y, cy), dcz = __fsub_rn(wb.c.z, cz);
      const float Ex = __fadd_ru(wb.e.x, ex), Ey = __fadd_ru(wb.e.y, ey), Ez = __fadd_ru(wb.e.z, ez);
      pass = dlow2_ce<PER>(dcx, dcy, dcz, Ex, Ey, Ez, D) <= wmax;
      if (PER && pass)
        cls = ce_class(dcx, Ex, D.h[0]) | (ce_class(dcy, Ey, D.h[1]) << 2) | (ce_class(dcz, Ez, D.h[2]) << 4);
      if (pass) {
        s0 = a.sbeg[l];
        s1 = a.sbeg[l + 1];
      }
    }
    unsigned bal = __ballot_sync(0xffffffffu, pass);
    JZ_DIAG(2, 1);
    JZ_DIAG(3, __popc(bal));
    while (bal) {
      const int src = __ffs(bal) - 1;
      bal &= bal - 1;
      // per-lane test: does any lane's query reach this leaf within its own k-th value?
      if (JZ_LANE_TEST) {
        const float lcx = __shfl_sync(0xffffffffu, cx, src), lcy = __shfl_sync(0xffffffffu, cy, src),
                    lcz = __shfl_sync(0xffffffffu, cz, src);
        const float lex = __shfl_sync(0xffffffffu, ex, src), ley = __shfl_sync(0xffffffffu, ey, src),
                    lez = __shfl_sync(0xffffffffu, ez, src);
        const float dl = dlow2_ce<PER>(__fsub_rn(qx, lcx), __fsub_rn(qy, lcy), __fsub_rn(qz, lcz), lex, ley, lez, D);
        if (!__any_sync(0xffffffffu, dl <= L.kth)) continue;
        JZ_DIAG(6, (unsigned long long)__popc(__ballot_sync(0xffffffffu, act && dl <= L.kth)) *
                       (unsigned)(__shfl_sync(0xffffffffu, s1, src) - __shfl_sync(0xffffffffu, s0, src)));
        JZ_DIAG(7, (unsigned long long)__popc(__ballot_sync(0xffffffffu, act)) *
                       (unsigned)(__shfl_sync(0xffffffffu, s1, src) - __shfl_sync(0xffffffffu, s0, src)));
      }
      const int c = __shfl_sync(0xffffffffu, cls, src);
      const int lp = __shfl_sync(0xffffffffu, s0, src), m = __shfl_sync(0xffffffffu, s1, src) - lp;
      const int mp = (m + 3) & ~3;
      if (W.n > 0 && (c != W.c0 || W.n + mp > kLCap)) flush<K, LB, PER>(B, W, qx, qy, qz, D, L);
      if (W.n == 0) W.c0 = c;
      stage_async<K>(B, W.n, a.spts + lp, m, mp);
      W.n += mp;
      nev += act ? (unsigned)m : 0u;
      JZ_DIAG(4, 1);
      ++L.stg;
    }
  }
}

__device__ __forceinline__ float warp_max_kth(float kth) {
  return __uint_as_float(__reduce_max_sync(0xffffffffu, __float_as_uint(fmaxf(kth, 0.f))));
}

template <int K>
__device__ __forceinline__ void bitonic_sort(u64 (&T)[K]) {
#pragma unroll
  for (int size = 2; size <= K; size <<= 1) {
#pragma unroll
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
#pragma unroll
      for (int i = 0; i < K; ++i) {
        const int j = i ^ stride;
        if (j > i) {
          const bool asc = (i & size) == 0;
          const u64 x = T[i], y = T[j];
          const bool sw = asc ? (x > y) : (x < y);
          T[i] = sw ? y : x;
          T[j] = sw ? x : y;
        }
      }
    }
  }
}

template <int K>
__device__ __forceinline__ void bitonic_sort_f(float (&T)[K]) {
#pragma unroll
  for (int size = 2; size <= K; size <<= 1) {
#pragma unroll
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
#pragma unroll
      for (int i = 0; i < K; ++i) {
        const int j = i ^ stride;
        if (j > i) {
          const float lo = fminf(T[i], T[j]), hi = fmaxf(T[i], T[j]);
          const bool asc = (i & size) == 0;
          T[i] = asc ? lo : hi;
          T[j] = asc ? hi : lo;
        }
      }
    }
  }
}

// window width: K sources (a 2K window with the K smallest kept cut insertions 26 -> 15 per
// query but cost more than it saved)
template <int K>
struct WinN {
  static constexpr int N = K;
};

// z-window initialisation (self-query): the N = WinN<K>::N sources at sorted positions
// [wpos, wpos + N) around the lane's own query are evaluated first; their keys start the log
// and their sorted values the list, so the k-th value is already close before the own
// leaves are scanned (z-order neighbours are mostly spatial neighbours, P:L69 / Fig. 2).
template <int K, bool LB, bool PER>
__device__ __forceinline__ void window_init(const LeafPK &a, const Dom &D, WarpBuf<K> &B, int wpos, float qx,
                                            float qy, float qz, bool act, Lane<K, LB> &L) {
  constexpr int N = WinN<K>::N;
  static_assert(N <= LogCap<K>::C, "the window must fit the log");
  const int lane = threadIdx.x & 31;
  float W[K];
#pragma unroll
  for (int o = 0; o < N; ++o) {
    float d = INFINITY;
    if (act) {
      const float4 p = a.spts[wpos + o];
      d = PER ? canon_d2_per(qx, qy, qz, p.x, p.y, p.z, D) : canon_d2_open(qx, qy, qz, p.x, p.y, p.z);
      B.lk[o][lane] = ((u64)__float_as_uint(d) << 32) | (unsigned)(__float_as_int(p.w) + 1);
    }
    W[o] = d;
  }
  bitonic_sort_f<K>(W);
#pragma unroll
  for (int j = 0; j < K; ++j) L.F[j] = W[j];
  L.nl = L.nf = act ? N : 0;
  L.app += act ? N : 0;
  L.kth = act ? L.F[K - 1] : -1.f;
}

// the same window read from the staged own block (own sources [b0, b0 + m) already in smem):
// no global loads; wl = wpos - b0
template <int K, bool LB, bool PER>
__device__ __forceinline__ void window_init_smem(const Dom &D, WarpBuf<K> &B, int wl, float qx, float qy, float qz,
                                                 bool act, Lane<K, LB> &L) {
  constexpr int N = WinN<K>::N;
  const int lane = threadIdx.x & 31;
  float W[K];
#pragma unroll
  for (int o = 0; o < N; ++o) {
    float d = INFINITY;
    if (act) {
      const int j = wl + o;
      const float sx = B.x[j], sy = B.y[j], sz = B.z[j];
      d = PER ? canon_d2_per(qx, qy, qz, sx, sy, sz, D) : canon_d2_open(qx, qy, qz, sx, sy, sz);
      B.lk[o][lane] = ((u64)__float_as_uint(d) << 32) | (unsigned)(B.g[j] + 1);
    }
    W[o] = d;
  }
  bitonic_sort_f<K>(W);
#pragma unroll
  for (int j = 0; j < K; ++j) L.F[j] = W[j];
  L.nl = L.nf = act ? N : 0;
  L.app += act ? N : 0;
  L.kth = act ? L.F[K - 1] : -1.f;
}

// pre-pass over the warp's own sources [s0, s1) (the sources of the leaves holding its
// queries; contiguous in z order): staged without per-leaf alignment, lanes skip their
// window (already in the list); cls_all = OR of the own leaves' shift classes.
template <int K, bool LB, bool PER>
__device__ __forceinline__ void own_pass(const LeafPK &a, const Dom &D, WarpBuf<K> &B, int s0, int s1, int cls_all,
                                         int wpos, float qx, float qy, float qz, bool act, Lane<K, LB> &L,
                                         unsigned long long &nev, bool staged0 = false) {
  for (int b0 = s0; b0 < s1; b0 += kLCap) {
    const int m = min(kLCap, s1 - b0), mp = (m + 3) & ~3;
    if (!(staged0 && b0 == s0)) stage_async<K>(B, 0, a.spts + b0, m, mp);
    nev += act ? (unsigned)m : 0u;
    const int np = pad8<K>(B, mp);
    cpa_wait();
    __syncwarp();
    const int wl = wpos - b0;
    if (!PER || cls_all == 0) {
      eval_block<K, LB>(B, np, qx, qy, qz, false, 0.f, 0.f, 0.f, L, WinN<K>::N, wl);
    } else {
      eval_generic<K, LB, WinN<K>::N>(B, mp, qx, qy, qz, D, L, wl);
    }
    __syncwarp();
  }
}

// ---------------------------------------------------------------- exact own pass (JZ_OWN_EXACT)
// The own block (the sources of the leaves holding the warp's queries, "the leaf's own
// points") is where most candidates fall below a loose k-th value: with the log it cost ~80% of
// the appends and ~45% of the merge rounds of an item. Here it is done in two fixed-cost sweeps:
//  A. every lane merges the d2 of 8 sources at a time into its sorted list F by a network (sort
//     the 8 values, min against F's reversed tail, bitonic merge): no log, no divergence; after
//     the sweep F holds the K smallest values of the own block exactly;
//  B. the block is evaluated again and every candidate with d2 <= F[K-1] is logged: the K
//     smallest keys (+ exact ties) with no merges (F is already final for the block).
// The walk then starts from the exact own-block k-th value and a log of ~K entries.
#ifndef JZ_OWN_EXACT
#define JZ_OWN_EXACT 1
#endif
#ifndef JZ_OWN_EXT
#define JZ_OWN_EXT 0  // leaves of J added on each side of the own block (exact pass over more sources)
#endif

// F (ascending, K values) := the K smallest of F and N (8 values, no NaN)
template <int K>
__device__ __forceinline__ void net_merge8(float (&F)[K], float (&N)[8]) {
  bitonic_sort_f<8>(N);
  if (!__any_sync(0xffffffffu, N[0] < F[K - 1])) return;
  constexpr int T = K < 8 ? K : 8;
#pragma unroll
  for (int i = 0; i < T; ++i) F[K - 1 - i] = fminf(F[K - 1 - i], N[i]);  // ascending F, descending N: bitonic
#pragma unroll
  for (int s = K / 2; s > 0; s >>= 1) {
#pragma unroll
    for (int i = 0; i < K; ++i) {
      if ((i & s) == 0) {
        const float lo = fminf(F[i], F[i + s]), hi = fmaxf(F[i], F[i + s]);
        F[i] = lo;
        F[i + s] = hi;
      }
    }
  }
}

// d2 of the 8 staged sources [j, j + 8): packed (no wrap inside the block) or per pair (gen)
template <int K, bool PER>
__device__ __forceinline__ void d2x8(const WarpBuf<K> &B, int j, float qx, float qy, float qz, u64 QX, u64 QY, u64 QZ,
                                     bool gen, const Dom &D, float (&N)[8]) {
  if (PER && gen) {
#pragma unroll
    for (int u = 0; u < 8; ++u) N[u] = canon_d2_per(qx, qy, qz, B.x[j + u], B.y[j + u], B.z[j + u], D);
  } else {
    d2x4(B.x, B.y, B.z, j, QX, QY, QZ, false, 0ull, 0ull, 0ull, N[0], N[1], N[2], N[3]);
    d2x4(B.x, B.y, B.z, j + 4, QX, QY, QZ, false, 0ull, 0ull, 0ull, N[4], N[5], N[6], N[7]);
  }
}

template <int K, bool LB, bool PER>
__device__ __forceinline__ void own_exact(const LeafPK &a, const Dom &D, WarpBuf<K> &B, int s0, int s1, int cls_all,
                                          float qx, float qy, float qz, bool act, Lane<K, LB> &L,
                                          unsigned long long &nev) {
  constexpr int C = LogCap<K>::C;
  const bool gen = PER && cls_all != 0;
  const u64 QX = pk(qx, qx), QY = pk(qy, qy), QZ = pk(qz, qz);
  const int nb = (s1 - s0 + kLCap - 1) / kLCap;  // batches
  // A: exact K smallest values of the block (batches in order; the last one stays staged)
  for (int b = 0; b < nb; ++b) {
    const int b0 = s0 + b * kLCap, m = min(kLCap, s1 - b0), mp = (m + 3) & ~3;
    stage_async<K>(B, 0, a.spts + b0, m, mp);
    nev += act ? (unsigned)m : 0u;
    const int np = pad8<K>(B, mp);
    cpa_wait();
    __syncwarp();
#pragma unroll 1
    for (int j = 0; j < np; j += 8) {
      float N[8];
      d2x8<K, PER>(B, j, qx, qy, qz, QX, QY, QZ, gen, D, N);
#pragma unroll
      for (int u = 0; u < 8; ++u) N[u] = fminf(N[u], INFINITY);  // NaN padding -> +inf
      net_merge8<K>(L.F, N);
    }
    __syncwarp();
  }
  L.kth = act ? L.F[K - 1] : -1.f;
  // B: log the candidates <= the block's k-th value (last batch first: it is still staged)
  for (int b = nb - 1; b >= 0; --b) {
    const int b0 = s0 + b * kLCap, m = min(kLCap, s1 - b0), mp = (m + 3) & ~3;
    if (b != nb - 1) {
      stage_async<K>(B, 0, a.spts + b0, m, mp);
      pad8<K>(B, mp);
      cpa_wait();
      __syncwarp();
    }
    const int np = (mp + 7) & ~7;
#pragma unroll 1
    for (int j = 0; j < np; j += 8) {
      float N[8];
      d2x8<K, PER>(B, j, qx, qy, qz, QX, QY, QZ, gen, D, N);
      const float mn = fminf(fminf(fminf(N[0], N[1]), fminf(N[2], N[3])), fminf(fminf(N[4], N[5]), fminf(N[6], N[7])));
      if (__any_sync(0xffffffffu, mn <= L.kth)) {
        const int4 G = *reinterpret_cast<const int4 *>(&B.g[j]);
        const int4 H = *reinterpret_cast<const int4 *>(&B.g[j + 4]);
        append<K, LB>(B, L, N[0], G.x);
        append<K, LB>(B, L, N[1], G.y);
        append<K, LB>(B, L, N[2], G.z);
        append<K, LB>(B, L, N[3], G.w);
        append<K, LB>(B, L, N[4], H.x);
        append<K, LB>(B, L, N[5], H.y);
        append<K, LB>(B, L, N[6], H.z);
        append<K, LB>(B, L, N[7], H.w);
        // massive exact ties only: the K smallest keys of the log are the block's K smallest keys
        if (__any_sync(0xffffffffu, L.nl > C - 8)) L.nl = drop_largest<K>(B, L.nl, K);
      }
    }
    __syncwarp();
  }
  L.nf = L.nl;
}

#ifdef JZ_SEED_EXP
// experiment only (tools/mkvar.py -DJZ_SEED_EXP): per-row k-th d2 seed (ideal-threshold bound)
__device__ const float *g_seed = nullptr;
void exp_set_seed(const float *p) { cudaMemcpyToSymbol(g_seed, &p, sizeof(p)); }
#endif

// one 32-query work item (see the file header)
template <int K, bool LB, bool PER>
__device__ __forceinline__ void leaf_item(const LeafPK &a, const Dom &D, WarpBuf<K> &B, int64_t item,
                                          unsigned long long &acc_ev) {
  const int lane = threadIdx.x & 31;
  const int J = a.item_par[item];
  const int LJa = a.par_leaf[J], LJb = a.par_leaf[J + 1];
  const int qhi = a.qbeg[LJb];
  const int q0 = a.item_q0[item];
  const int qi = q0 + lane;
  const bool act = qi < qhi;
  float qx = 0.f, qy = 0.f, qz = 0.f, qw = 0.f;
  if (act) {
    const float4 q = a.qpts[qi];
    qx = q.x;
    qy = q.y;
    qz = q.z;
    qw = q.w;
  }
  const int64_t row = !act ? 0 : (a.order == JZ_ORDER_INPUT ? (int64_t)a.qin[qi] : (int64_t)qi);
  if (!__any_sync(0xffffffffu, act)) return;
  float blo[3] = {act ? qx : INFINITY, act ? qy : INFINITY, act ? qz : INFINITY};
  float bhi[3] = {act ? qx : -INFINITY, act ? qy : -INFINITY, act ? qz : -INFINITY};
#pragma unroll
  for (int d = 0; d < 3; ++d) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      blo[d] = fminf(blo[d], __shfl_xor_sync(0xffffffffu, blo[d], o));
      bhi[d] = fmaxf(bhi[d], __shfl_xor_sync(0xffffffffu, bhi[d], o));
    }
  }
  const CE wb = make_ce(blo[0], blo[1], blo[2], bhi[0], bhi[1], bhi[2], a.Lmax);

  const float R0 = a.rmax2 ? a.rmax2[J] : INFINITY;
  Lane<K, LB> L;
  {
#pragma unroll
    for (int j = 0; j < K; ++j) L.F[j] = (j < K - a.k) ? 0.f : R0;  // K - k placeholders <= any d2
    L.kth = act ? R0 : -1.f;
    L.lb = 0;
    if (LB && act) {  // continue after the last (d2, index) of the previous pass
      const int64_t o = row * a.ldo + a.col0 - 1;
      L.lb = ((u64)__float_as_uint(a.out_d2[o]) << 32) | (unsigned)(a.out_idx[o] + 1);
    }
    L.ins = 0;
    L.app = L.rnd = L.cmp = L.stg = L.stp = L.pst = 0;
    L.nl = 0;
    L.nf = 0;
    L.act = act;
  }
  unsigned long long nev = 0;
  // pre-pass: the leaves holding the warp's own queries (tightens the k-th bound early)
  int xa = 0x7fffffff, xb = -1;
  {
    const int qend = min(q0 + 32, qhi);
    for (int l0 = LJa; l0 < LJb; l0 += 32) {
      const int l = l0 + lane;
      const bool ov = l < LJb && a.qbeg[l] < qend && a.qbeg[l + 1] > q0;
      const unsigned b = __ballot_sync(0xffffffffu, ov);
      if (b) {
        xa = min(xa, l0 + __ffs(b) - 1);
        xb = max(xb, l0 + 32 - __clz(b));
      }
    }
    if (JZ_OWN_EXT > 0 && JZ_OWN_EXACT && !LB) {  // widen the own block by neighbouring leaves of J
      xa = max(LJa, xa - JZ_OWN_EXT);
      xb = min(LJb, xb + JZ_OWN_EXT);
    }
    const int s0o = a.sbeg[xa], s1o = a.sbeg[xb];
    int wpos = -0x40000000;  // far from every staged index: no window
    constexpr int NW = WinN<K>::N;
    bool staged0 = false;
    if (!JZ_OWN_EXACT && !LB && a.self && a.k == K && s1o - s0o >= NW) {
      if (act) wpos = min(max(qi - NW / 2, s0o), s1o - NW);
      if (JZ_WIN_SMEM && s1o - s0o <= kLCap) {  // the own block fits one batch: window from smem
        const int m = s1o - s0o;
        stage_async<K>(B, 0, a.spts + s0o, m, (m + 3) & ~3);
        cpa_wait();
        __syncwarp();
        window_init_smem<K, LB, PER>(D, B, wpos - s0o, qx, qy, qz, act, L);
        staged0 = true;
      } else {
        window_init<K, LB, PER>(a, D, B, wpos, qx, qy, qz, act, L);
      }
    }
    int cls_all = 0;
    if (PER) {
      for (int l = xa + lane; l < xb; l += 32) {
        const CE lc = a.leaf_ce[l];
        const float dcx = __fsub_rn(wb.c.x, lc.c.x), dcy = __fsub_rn(wb.c.y, lc.c.y), dcz = __fsub_rn(wb.c.z, lc.c.z);
        cls_all |= ce_class(dcx, __fadd_ru(wb.e.x, lc.e.x), D.h[0]) | ce_class(dcy, __fadd_ru(wb.e.y, lc.e.y), D.h[1]) |
                   ce_class(dcz, __fadd_ru(wb.e.z, lc.e.z), D.h[2]);
      }
      cls_all = __reduce_or_sync(0xffffffffu, cls_all);
    }
#ifdef JZ_SEED_EXP
    if (g_seed) {
      const float t = act ? g_seed[row] : R0;
#pragma unroll
      for (int j = 0; j < K; ++j) L.F[j] = fminf(L.F[j], t);
      L.kth = act ? L.F[K - 1] : -1.f;
    }
#endif
    L.stg += xb - xa;
    if (JZ_OWN_EXACT && !LB)
      own_exact<K, LB, PER>(a, D, B, s0o, s1o, cls_all, qx, qy, qz, act, L, nev);
    else
      own_pass<K, LB, PER>(a, D, B, s0o, s1o, cls_all, wpos, qx, qy, qz, act, L, nev, staged0);
    if (JZ_MERGE_T > 0) merge<K, LB>(B, L);
  }
  const unsigned o_app = L.app, o_rnd = L.rnd, o_cmp = L.cmp, o_stp = L.stp, o_pst = L.pst;
  const int64_t eb = a.ispl[J], ee = a.ispl[J + 1];
  Batch W;
  W.n = 0;
  W.c0 = 0;
  // entries in chunks of 32, one lane per entry (list order = r_low order): the node tests run in
  // parallel instead of one dependent load chain per entry; survivors are visited in list order
  for (int64_t c0 = eb; c0 < ee; c0 += 32) {
    const float wc = a.early ? warp_max_kth(L.kth) : INFINITY;
    const int64_t e = c0 + lane;
    bool ok = false, past = false;
    int S = 0;
    if (e < ee) {
      const float rl = a.rlow[e];
      S = a.isrc[e];
      past = rl > wc;
      ok = !past;
      if (ok && a.par_ce) {
        const CE pc = a.par_ce[S];
        ok = dlow2_ce<PER>(__fsub_rn(wb.c.x, pc.c.x), __fsub_rn(wb.c.y, pc.c.y), __fsub_rn(wb.c.z, pc.c.z),
                           __fadd_ru(wb.e.x, pc.e.x), __fadd_ru(wb.e.y, pc.e.y), __fadd_ru(wb.e.z, pc.e.z), D) <= wc;
      }
    }
    JZ_DIAG(0, __popc(__ballot_sync(0xffffffffu, e < ee && !past)));
    unsigned bal = __ballot_sync(0xffffffffu, ok);
    JZ_DIAG(1, __popc(bal));
    const bool stop = a.sorted && __any_sync(0xffffffffu, past);  // later chunks have larger r_low
    while (bal) {
      const int src = __ffs(bal) - 1;
      bal &= bal - 1;
      const int Se = __shfl_sync(0xffffffffu, S, src);
      const float wmax = a.early ? warp_max_kth(L.kth) : INFINITY;
      visit_leaves<K, LB, PER>(a, D, B, W, wb, wmax, a.par_leaf[Se], a.par_leaf[Se + 1], Se == J ? xa : 0,
                               Se == J ? xb : 0, qx, qy, qz, act, L, nev);
    }
    if (stop) break;
  }
  flush<K, LB, PER>(B, W, qx, qy, qz, D, L);
  JZ_DIAG(5, 1);
  // the row: the k smallest keys of the log (all entries <= the final k-th value)
  compact<K, LB>(B, L);
  if (L.nl > a.k) L.nl = drop_largest<K>(B, L.nl, a.k);
  if (a.stats && !JZ_STATS) {  // evaluations only, summed per warp over its items (one atomic per warp)
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) nev += __shfl_xor_sync(0xffffffffu, nev, o);
    acc_ev += nev;
  }
  if (a.stats && JZ_STATS) {
    unsigned long long tot = nev, ins = L.ins, app = L.app;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      tot += __shfl_xor_sync(0xffffffffu, tot, o);
      ins += __shfl_xor_sync(0xffffffffu, ins, o);
      app += __shfl_xor_sync(0xffffffffu, app, o);
    }
    if (lane == 0) {
      atomicAdd(&a.stats[0], tot);
      atomicAdd(&a.stats[1], ins);
      atomicAdd(&a.stats[2], app);
      atomicAdd(&a.stats[3], (unsigned long long)L.rnd);
      atomicAdd(&a.stats[4], (unsigned long long)L.cmp);
      atomicAdd(&a.stats[5], (unsigned long long)L.stg);
      atomicAdd(&a.stats[6], 1ull);
    }
    if (JZ_STATS) {
      unsigned long long oa = o_app;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) oa += __shfl_xor_sync(0xffffffffu, oa, o);
      if (lane == 0) {
        atomicAdd(&a.stats[7], oa);
        atomicAdd(&a.stats[8], (unsigned long long)o_rnd);
        atomicAdd(&a.stats[9], (unsigned long long)o_cmp);
        atomicAdd(&a.stats[10], (unsigned long long)o_stp);
        atomicAdd(&a.stats[11], (unsigned long long)o_pst);
        atomicAdd(&a.stats[12], (unsigned long long)L.stp);
        atomicAdd(&a.stats[13], (unsigned long long)L.pst);
      }
    }
  }
  {
    u64 T[K];
#pragma unroll
    for (int j = 0; j < K; ++j) T[j] = (act && j < L.nl) ? B.lk[j][lane] : ~0ull;
    bitonic_sort<K>(T);
    if (JZ_VEC_ROWS == 2 && a.k == K && ((a.ldo | a.col0) & 3) == 0) {
      // rows through shared memory (the log area is free now): one warp store covers 8 whole
      // rows (4 lanes x 16 B each) instead of 32 partial rows. Row stride K + 4 words keeps the
      // 16-byte alignment (4-way bank conflicts on the writes)
      constexpr int RS = K + 4;
      static_assert(2 * 32 * RS * 4 <= LogCap<K>::C * 32 * 8, "row staging must fit the log area");
      unsigned *sidx = reinterpret_cast<unsigned *>(&B.lk[0][0]);  // [32][RS] idx, then [32][RS] d2
      unsigned *sd2 = sidx + 32 * RS;
      __syncwarp();
#pragma unroll
      for (int j = 0; j < K; ++j) {
        sidx[lane * RS + j] = (unsigned)(T[j] & 0xffffffffu) - 1u;
        sd2[lane * RS + j] = (unsigned)(T[j] >> 32);
      }
      __syncwarp();
      constexpr int LPR = K / 4;  // lanes per row (16 B each)
#pragma unroll
      for (int r0 = 0; r0 < 32; r0 += 32 / LPR) {
        const int r = r0 + lane / LPR, c = lane % LPR;
        const int64_t rr = __shfl_sync(0xffffffffu, row, r);
        const int ra = __shfl_sync(0xffffffffu, (int)act, r);
        if (ra) {
          reinterpret_cast<uint4 *>(a.out_idx + rr * a.ldo + a.col0)[c] = reinterpret_cast<const uint4 *>(sidx + r * RS)[c];
          reinterpret_cast<uint4 *>(a.out_d2 + rr * a.ldo + a.col0)[c] = reinterpret_cast<const uint4 *>(sd2 + r * RS)[c];
        }
      }
    } else if (act) {
      int32_t *oi = a.out_idx + row * a.ldo + a.col0;
      float *od = a.out_d2 + row * a.ldo + a.col0;
      if (JZ_VEC_ROWS && a.k == K && ((a.ldo | a.col0) & 3) == 0) {
        // full 16-byte aligned rows: 128-bit stores (K / 4 per array instead of K scalar stores)
#pragma unroll
        for (int j = 0; j < K; j += 4) {
          reinterpret_cast<int4 *>(oi)[j / 4] = make_int4(
              (int32_t)((unsigned)(T[j] & 0xffffffffu) - 1u), (int32_t)((unsigned)(T[j + 1] & 0xffffffffu) - 1u),
              (int32_t)((unsigned)(T[j + 2] & 0xffffffffu) - 1u), (int32_t)((unsigned)(T[j + 3] & 0xffffffffu) - 1u));
          reinterpret_cast<float4 *>(od)[j / 4] =
              make_float4(__uint_as_float((unsigned)(T[j] >> 32)), __uint_as_float((unsigned)(T[j + 1] >> 32)),
                          __uint_as_float((unsigned)(T[j + 2] >> 32)), __uint_as_float((unsigned)(T[j + 3] >> 32)));
        }
      } else {
#pragma unroll
        for (int j = 0; j < K; ++j) {
          if (j < a.k) {
            oi[j] = (int32_t)((unsigned)(T[j] & 0xffffffffu) - 1u);
            od[j] = __uint_as_float((unsigned)(T[j] >> 32));
          }
        }
      }
    }
    if (act && a.out_row_gidx) a.out_row_gidx[row] = __float_as_int(qw);
  }
}

// JZ_PERSIST: one resident CTA set; each warp takes the next work item from a counter until the
// launched range is exhausted (no CTA launch per item, same dynamic retirement as one item per CTA)
#ifndef JZ_PERSIST
#define JZ_PERSIST 1
#endif
template <int K, bool LB, bool PER>
__global__ void __launch_bounds__(kLThreads, MinBlocks<K>::v) k_leaf(LeafPK a, Dom D) {
  __shared__ __align__(16) WarpBuf<K> s_buf[kLWarps];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  unsigned long long acc_ev = 0, acc_it = 0;  // evaluations / items of this warp (stats, non-JZ_STATS builds)
  if (JZ_PERSIST && a.counter) {
    while (true) {
      unsigned long long t = 0;
      if (lane == 0) t = atomicAdd(a.counter, 1ull);
      const int64_t item = a.item_off + (int64_t)__shfl_sync(0xffffffffu, t, 0);
      if (item >= a.nitems) break;
      leaf_item<K, LB, PER>(a, D, s_buf[warp], item, acc_ev);
      ++acc_it;
      __syncwarp();
    }
  } else {
    const int64_t item = a.item_off + (int64_t)blockIdx.x * kLWarps + warp;
    if (item >= a.nitems) return;
    leaf_item<K, LB, PER>(a, D, s_buf[warp], item, acc_ev);
    acc_it = 1;
  }
  if (!JZ_STATS && a.stats && lane == 0 && acc_it) {
    atomicAdd(&a.stats[0], acc_ev);
    atomicAdd(&a.stats[6], acc_it);
  }
}

// ---------------------------------------------------------------- friends-of-friends (F4)
// PAPER.md §5 (L466-474, L488-490): every pair of points with canonical d2 <= b2 is linked in a
// union-find over sorted positions; a link hangs the larger root under the smaller one with an
// atomic compare-and-swap and retries on failure, so a root is its component's smallest
// position. The walk is the kNN one with a fixed radius: the same 32-query work items, own
// pre-pass, plane-1 interaction lists (d_low^2 <= b2), per-leaf warp-box and per-lane tests, packed
// FP32 distances. Each unordered pair is linked from its lower-positioned point only.
struct FofBuf {
  float x[kLCap + 8], y[kLCap + 8], z[kLCap + 8];
  int g[kLCap + 8];  // sorted position of the staged source
};

// root of x with path halving (x only ever points to one of its ancestors, so the plain
// stores are benign under concurrent unions); L2 loads: other SMs link concurrently
__device__ __forceinline__ int fof_find(int32_t *par, int x) {
  while (true) {
    const int p = __ldcg(&par[x]);
    if (p == x) return x;
    const int pp = __ldcg(&par[p]);
    if (pp == p) return p;
    __stcg(&par[x], pp);
    x = pp;
  }
}

__device__ __forceinline__ void fof_union(int32_t *par, int a, int b) {
  while (true) {
    a = fof_find(par, a);
    b = fof_find(par, b);
    if (a == b) return;
    if (a > b) {
      const int t = a;
      a = b;
      b = t;
    }
    const int old = atomicCAS(&par[b], b, a);  // hang the larger root under the smaller one
    if (old == b) return;
    b = old;  // b stopped being a root: retry from its new parent
  }
}

struct FofPK {
  const float4 *spts;
  const int32_t *sbeg;
  const CE *leaf_ce;
  const NodeBox *leaf_box;  // exact boxes: d_up test of a whole (item, leaf) pair
  const int32_t *par_leaf;
  const CE *par_ce;
  const int64_t *ispl;
  const int32_t *isrc;
  const float *rlow;
  const int32_t *item_par;
  const int32_t *item_q0;
  int64_t nitems;
  float b2;
  float Lmax;
  int sorted;
  int32_t *par;
  unsigned long long *stats;  // [0] distance evaluations
  unsigned long long *counter;  // JZ_PERSIST work-item counter (zeroed) or nullptr
};

// staged sources [0, n) (n multiple of 8) against the lane's query qi
template <bool PER>
__device__ __forceinline__ void fof_eval(FofBuf &B, int n, int qi, float qx, float qy, float qz, bool shift, float shx,
                                         float shy, float shz, bool generic, const Dom &D, float b2, int32_t *par,
                                         bool act) {
  const u64 QX = pk(qx, qx), QY = pk(qy, qy), QZ = pk(qz, qz);
  const u64 SX = pk(shx, shx), SY = pk(shy, shy), SZ = pk(shz, shz);
#pragma unroll 1
  for (int j = 0; j < n; j += 8) {
    float a0, a1, a2, a3, b0, b1, b2v, b3;
    if (!PER || !generic) {
      d2x4(B.x, B.y, B.z, j, QX, QY, QZ, shift, SX, SY, SZ, a0, a1, a2, a3);
      d2x4(B.x, B.y, B.z, j + 4, QX, QY, QZ, shift, SX, SY, SZ, b0, b1, b2v, b3);
    } else {  // straddling pair: per-pair minimal image (canonical select)
      a0 = canon_d2_per(qx, qy, qz, B.x[j], B.y[j], B.z[j], D);
      a1 = canon_d2_per(qx, qy, qz, B.x[j + 1], B.y[j + 1], B.z[j + 1], D);
      a2 = canon_d2_per(qx, qy, qz, B.x[j + 2], B.y[j + 2], B.z[j + 2], D);
      a3 = canon_d2_per(qx, qy, qz, B.x[j + 3], B.y[j + 3], B.z[j + 3], D);
      b0 = canon_d2_per(qx, qy, qz, B.x[j + 4], B.y[j + 4], B.z[j + 4], D);
      b1 = canon_d2_per(qx, qy, qz, B.x[j + 5], B.y[j + 5], B.z[j + 5], D);
      b2v = canon_d2_per(qx, qy, qz, B.x[j + 6], B.y[j + 6], B.z[j + 6], D);
      b3 = canon_d2_per(qx, qy, qz, B.x[j + 7], B.y[j + 7], B.z[j + 7], D);
    }
    const float m = fminf(fminf(fminf(a0, a1), fminf(a2, a3)), fminf(fminf(b0, b1), fminf(b2v, b3)));  // NaN ignored
    if (__any_sync(0xffffffffu, act && m <= b2)) {
      unsigned mk = act ? ((a0 <= b2) | ((a1 <= b2) << 1) | ((a2 <= b2) << 2) | ((a3 <= b2) << 3) | ((b0 <= b2) << 4) |
                           ((b1 <= b2) << 5) | ((b2v <= b2) << 6) | ((b3 <= b2) << 7))
                        : 0u;
      while (mk) {  // one inlined union site
        const int i = __ffs(mk) - 1;
        mk &= mk - 1;
        const int g = B.g[j + i];
        if (g > qi) fof_union(par, qi, g);
      }
    }
  }
}

__device__ __forceinline__ int fof_pad8(FofBuf &B, int n) {
  const int lane = threadIdx.x & 31;
  if (n & 4) {
    if (lane < 4) {
      const float nan = __int_as_float(0x7fc00000);
      B.x[n + lane] = nan;
      B.y[n + lane] = nan;
      B.z[n + lane] = nan;
      B.g[n + lane] = -1;
    }
    n += 4;
  }
  return n;
}

template <bool PER>
__device__ __forceinline__ void fof_item(const FofPK &a, const Dom &D, FofBuf &B, int64_t item) {
  const int lane = threadIdx.x & 31;
  const int J = a.item_par[item];
  const int LJa = a.par_leaf[J], LJb = a.par_leaf[J + 1];
  const int qhi = a.sbeg[LJb];
  const int q0 = a.item_q0[item];
  const int qi = q0 + lane;
  const bool act = qi < qhi;
  float qx = 0.f, qy = 0.f, qz = 0.f;
  if (act) {
    const float4 q = a.spts[qi];
    qx = q.x;
    qy = q.y;
    qz = q.z;
  }
  float blo[3] = {act ? qx : INFINITY, act ? qy : INFINITY, act ? qz : INFINITY};
  float bhi[3] = {act ? qx : -INFINITY, act ? qy : -INFINITY, act ? qz : -INFINITY};
#pragma unroll
  for (int d = 0; d < 3; ++d) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      blo[d] = fminf(blo[d], __shfl_xor_sync(0xffffffffu, blo[d], o));
      bhi[d] = fmaxf(bhi[d], __shfl_xor_sync(0xffffffffu, bhi[d], o));
    }
  }
  const CE wb = make_ce(blo[0], blo[1], blo[2], bhi[0], bhi[1], bhi[2], a.Lmax);
  NodeBox wnb;  // the item's query box (exact bounds for the d_up test)
  wnb.lo = make_float4(blo[0], blo[1], blo[2], 0.f);
  wnb.hi = make_float4(bhi[0], bhi[1], bhi[2], 0.f);
  // a whole (item, leaf) pair can only be within R_link if the item box is (d_up >= diag / 2)
  const bool small = JZ_FOF_FULL && __fmul_rd(box_dup2(wnb, wnb, D), 0.25f) <= a.b2;
  const float b2 = a.b2;
  unsigned long long nev = 0;
  // own leaves [xa, xb): their sources are contiguous; every pair inside is a candidate
  int xa = 0x7fffffff, xb = -1;
  {
    const int qend = min(q0 + 32, qhi);
    for (int l0 = LJa; l0 < LJb; l0 += 32) {
      const int l = l0 + lane;
      const bool ov = l < LJb && a.sbeg[l] < qend && a.sbeg[l + 1] > q0;
      const unsigned b = __ballot_sync(0xffffffffu, ov);
      if (b) {
        xa = min(xa, l0 + __ffs(b) - 1);
        xb = max(xb, l0 + 32 - __clz(b));
      }
    }
    int cls_all = 0;
    if (PER) {
      for (int l = xa + lane; l < xb; l += 32) {
        const CE lc = a.leaf_ce[l];
        cls_all |= ce_class(__fsub_rn(wb.c.x, lc.c.x), __fadd_ru(wb.e.x, lc.e.x), D.h[0]) |
                   ce_class(__fsub_rn(wb.c.y, lc.c.y), __fadd_ru(wb.e.y, lc.e.y), D.h[1]) |
                   ce_class(__fsub_rn(wb.c.z, lc.c.z), __fadd_ru(wb.e.z, lc.e.z), D.h[2]);
      }
      cls_all = __reduce_or_sync(0xffffffffu, cls_all);
    }
    const int s0 = a.sbeg[xa], s1 = a.sbeg[xb];
    for (int b0 = max(s0, q0 + 1); b0 < s1; b0 += kLCap) {  // only sources after the warp's first query
      const int m = min(kLCap, s1 - b0), mp = (m + 3) & ~3;
      for (int t = lane; t < mp; t += 32) {
        float4 p = make_float4(__int_as_float(0x7fc00000), __int_as_float(0x7fc00000), __int_as_float(0x7fc00000), 0.f);
        if (t < m) p = a.spts[b0 + t];
        B.x[t] = p.x;
        B.y[t] = p.y;
        B.z[t] = p.z;
        B.g[t] = t < m ? b0 + t : -1;
      }
      nev += act ? (unsigned)m : 0u;
      const int np = fof_pad8(B, mp);
      __syncwarp();
      fof_eval<PER>(B, np, qi, qx, qy, qz, false, 0.f, 0.f, 0.f, PER && cls_all != 0, D, b2, a.par, act);
      __syncwarp();
    }
  }
  const int64_t eb = a.ispl[J], ee = a.ispl[J + 1];
  for (int64_t e = eb; e < ee; ++e) {
    if (a.rlow[e] > b2) {
      if (a.sorted) break;
      continue;
    }
    const int S = a.isrc[e];
    if (a.par_ce) {
      const CE pc = a.par_ce[S];
      if (dlow2_ce<PER>(__fsub_rn(wb.c.x, pc.c.x), __fsub_rn(wb.c.y, pc.c.y), __fsub_rn(wb.c.z, pc.c.z),
                        __fadd_ru(wb.e.x, pc.e.x), __fadd_ru(wb.e.y, pc.e.y), __fadd_ru(wb.e.z, pc.e.z), D) > b2)
        continue;
    }
    const int la = a.par_leaf[S], lb = a.par_leaf[S + 1];
    const int ya = S == J ? xa : 0, yb = S == J ? xb : 0;
    for (int l0 = la; l0 < lb; l0 += 32) {
      const int l = l0 + lane;
      bool pass = false, full = false;
      int cls = 0, s0 = 0, s1 = 0;
      float cx = 0.f, cy = 0.f, cz = 0.f, ex = 0.f, ey = 0.f, ez = 0.f;
      if (l < lb && (l < ya || l >= yb)) {
        const CE lc = a.leaf_ce[l];
        cx = lc.c.x;
        cy = lc.c.y;
        cz = lc.c.z;
        ex = lc.e.x;
        ey = lc.e.y;
        ez = lc.e.z;
        const float dcx = __fsub_rn(wb.c.x, cx), dcy = __fsub_rn(wb.c.y, cy), dcz = __fsub_rn(wb.c.z, cz);
        const float Ex = __fadd_ru(wb.e.x, ex), Ey = __fadd_ru(wb.e.y, ey), Ez = __fadd_ru(wb.e.z, ez);
        s0 = a.sbeg[l];
        s1 = a.sbeg[l + 1];
        pass = s1 > q0 + 1 && dlow2_ce<PER>(dcx, dcy, dcz, Ex, Ey, Ez, D) <= b2;  // a source after some query
        if (PER && pass)
          cls = ce_class(dcx, Ex, D.h[0]) | (ce_class(dcy, Ey, D.h[1]) << 2) | (ce_class(dcz, Ez, D.h[2]) << 4);
        // every (query, source) pair of the item and the leaf within R_link (P:L486 case 2 at the
        // leaf level): link all of them through the leaf's first point instead of evaluating pairs
        full = small && pass && box_dup2(wnb, a.leaf_box[l], D) <= b2;
      }
      const unsigned fb = __ballot_sync(0xffffffffu, full);
      for (unsigned f = fb; f; f &= f - 1) {
        const int src = __ffs(f) - 1;
        const int lp = __shfl_sync(0xffffffffu, s0, src), le = __shfl_sync(0xffffffffu, s1, src);
        if (act) fof_union(a.par, qi, lp);
        for (int t = lp + 1 + lane; t < le; t += 32) fof_union(a.par, t, lp);
      }
      unsigned bal = __ballot_sync(0xffffffffu, pass && !full);
      while (bal) {
        const int c0 = __shfl_sync(0xffffffffu, cls, __ffs(bal) - 1);
        int n = 0;
        while (bal) {
          const int src = __ffs(bal) - 1;
          if (__shfl_sync(0xffffffffu, cls, src) != c0) break;
          {
            const float lcx = __shfl_sync(0xffffffffu, cx, src), lcy = __shfl_sync(0xffffffffu, cy, src),
                        lcz = __shfl_sync(0xffffffffu, cz, src);
            const float lex = __shfl_sync(0xffffffffu, ex, src), ley = __shfl_sync(0xffffffffu, ey, src),
                        lez = __shfl_sync(0xffffffffu, ez, src);
            const float dl =
                dlow2_ce<PER>(__fsub_rn(qx, lcx), __fsub_rn(qy, lcy), __fsub_rn(qz, lcz), lex, ley, lez, D);
            if (!__any_sync(0xffffffffu, act && dl <= b2)) {
              bal &= bal - 1;
              continue;
            }
          }
          const int lp = __shfl_sync(0xffffffffu, s0, src), m = __shfl_sync(0xffffffffu, s1, src) - lp;
          if (n + ((m + 3) & ~3) > kLCap) break;
          bal &= bal - 1;
          for (int t = lane; t < ((m + 3) & ~3); t += 32) {
            float4 p = make_float4(__int_as_float(0x7fc00000), __int_as_float(0x7fc00000), __int_as_float(0x7fc00000),
                                   0.f);
            if (t < m) p = a.spts[lp + t];
            B.x[n + t] = p.x;
            B.y[n + t] = p.y;
            B.z[n + t] = p.z;
            B.g[n + t] = t < m ? lp + t : -1;
          }
          nev += act ? (unsigned)m : 0u;
          n += (m + 3) & ~3;
        }
        if (n == 0) continue;
        n = fof_pad8(B, n);
        __syncwarp();
        fof_eval<PER>(B, n, qi, qx, qy, qz, PER && c0 != 0, class_shift(c0 & 3, D.L[0]),
                      class_shift((c0 >> 2) & 3, D.L[1]), class_shift((c0 >> 4) & 3, D.L[2]), PER && any_straddle(c0),
                      D, b2, a.par, act);
        __syncwarp();
      }
    }
  }
  if (a.stats) {
    unsigned long long tot = nev;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) tot += __shfl_xor_sync(0xffffffffu, tot, o);
    if (lane == 0) atomicAdd(&a.stats[0], tot);
  }
}

// persistent like k_leaf (JZ_PERSIST): resident CTAs take 32-query items from a counter
template <bool PER>
__global__ void __launch_bounds__(kLThreads, 12) k_fof_leaf(FofPK a, Dom D) {
  __shared__ __align__(16) FofBuf s_buf[kLWarps];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (JZ_PERSIST && a.counter) {
    while (true) {
      unsigned long long t = 0;
      if (lane == 0) t = atomicAdd(a.counter, 1ull);
      const int64_t item = (int64_t)__shfl_sync(0xffffffffu, t, 0);
      if (item >= a.nitems) return;
      fof_item<PER>(a, D, s_buf[warp], item);
      __syncwarp();
    }
  }
  const int64_t item = (int64_t)blockIdx.x * kLWarps + warp;
  if (item >= a.nitems) return;
  fof_item<PER>(a, D, s_buf[warp], item);
}

// work items: 32-query groups of each receiving parent, in z order
__global__ void k_item_count(const int32_t *__restrict__ par_leaf, const int32_t *__restrict__ leaf_beg, int64_t npar,
                             int chunk, int32_t *__restrict__ cnt) {
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < npar; j += (int64_t)gridDim.x * blockDim.x) {
    const int n = leaf_beg[par_leaf[j + 1]] - leaf_beg[par_leaf[j]];
    cnt[j] = (n + chunk - 1) / chunk;
  }
}

__global__ void k_item_fill(const int32_t *__restrict__ par_leaf, const int32_t *__restrict__ leaf_beg, int64_t npar,
                            int chunk, const int64_t *__restrict__ off, int32_t *__restrict__ item_par,
                            int32_t *__restrict__ item_q0) {
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < npar; j += (int64_t)gridDim.x * blockDim.x) {
    const int q0 = leaf_beg[par_leaf[j]], q1 = leaf_beg[par_leaf[j + 1]];
    int64_t o = off[j];
    for (int q = q0; q < q1; q += chunk, ++o) {
      item_par[o] = (int32_t)j;
      item_q0[o] = q;
    }
  }
}

// persistent launches: as many CTAs as can be resident (occupancy x SMs), capped by the items
template <int K, bool LB, bool PER>
static void launch_kl(const LeafPK &la, const Dom &D, unsigned blocks, cudaStream_t st) {
  if (la.counter) {
    static int resident = 0;  // per instantiation
    if (resident == 0) {
      int nb = 0, dev = 0, sms = 0;
      JZ_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k_leaf<K, LB, PER>, kLThreads, 0));
      JZ_CUDA(cudaGetDevice(&dev));
      JZ_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
      resident = nb * sms > 0 ? nb * sms : 1;
    }
    if (blocks > (unsigned)resident) blocks = (unsigned)resident;
  }
  k_leaf<K, LB, PER><<<blocks, kLThreads, 0, st>>>(la, D);
}

template <int K>
static void launch_l(const LeafPK &la, const Dom &D, unsigned blocks, cudaStream_t st) {
  if (la.col0 > 0) {  // later pass of a k > k_max query
    if (D.periodic) launch_kl<K, true, true>(la, D, blocks, st);
    else launch_kl<K, true, false>(la, D, blocks, st);
  } else {
    if (D.periodic) launch_kl<K, false, true>(la, D, blocks, st);
    else launch_kl<K, false, false>(la, D, blocks, st);
  }
}

void leaf_to_leaf(const LeafArgs &a, const Dom &D, cudaStream_t st) {
  if (a.npar == 0) return;
  int32_t *cnt = nullptr;
  int64_t *off = nullptr;
  JZ_CUDA(cudaMallocAsync(&cnt, a.npar * sizeof(int32_t), st));
  JZ_CUDA(cudaMallocAsync(&off, (a.npar + 1) * sizeof(int64_t), st));
  const int chunk = 32;
  k_item_count<<<grid_for(a.npar, 256), 256, 0, st>>>(a.par_leaf, a.qbeg, a.npar, chunk, cnt);
  JZ_LAUNCH_CHECK();
  exclusive_scan_i32_to_i64(cnt, off, a.npar, st);
  const int64_t nitems = read_i64(off + a.npar, st);
  int32_t *item_par = nullptr, *item_q0 = nullptr;
  JZ_CUDA(cudaMallocAsync(&item_par, (nitems + 1) * sizeof(int32_t), st));
  JZ_CUDA(cudaMallocAsync(&item_q0, (nitems + 1) * sizeof(int32_t), st));
  k_item_fill<<<grid_for(a.npar, 256), 256, 0, st>>>(a.par_leaf, a.qbeg, a.npar, chunk, off, item_par, item_q0);
  JZ_LAUNCH_CHECK();
  const float Lmax = D.periodic ? fmaxf(fmaxf(D.L[0], D.L[1]), D.L[2]) : 0.f;
  CE *leaf_ce = nullptr, *par_ce = nullptr;
  JZ_CUDA(cudaMallocAsync(&leaf_ce, (a.nleaf > 0 ? a.nleaf : 1) * sizeof(CE), st));
  k_box_ce<<<grid_for(a.nleaf, 256), 256, 0, st>>>(a.leaf_box, a.nleaf, Lmax, leaf_ce);
  JZ_LAUNCH_CHECK();
  if (a.par_box) {
    JZ_CUDA(cudaMallocAsync(&par_ce, a.npar * sizeof(CE), st));
    k_box_ce<<<grid_for(a.npar, 256), 256, 0, st>>>(a.par_box, a.npar, Lmax, par_ce);
    JZ_LAUNCH_CHECK();
  }

  LeafPK la;
  la.spts = a.spts;
  la.sbeg = a.sbeg;
  la.qpts = a.qpts;
  la.qbeg = a.qbeg;
  la.qin = a.qin;
  la.leaf_ce = leaf_ce;
  la.par_leaf = a.par_leaf;
  la.par_ce = par_ce;
  la.ispl = a.il->ispl;
  la.isrc = a.il->isrc;
  la.rlow = a.il->rlow;
  la.rmax2 = a.rmax2;
  la.item_par = item_par;
  la.item_q0 = item_q0;
  la.nitems = nitems;
  la.item_off = 0;
  la.Lmax = Lmax;
  la.ldo = a.k;
  la.order = a.order;
  la.early = !(a.flags & JZ_FLAG_NO_EARLY_EXIT);
  la.sorted = !(a.flags & (JZ_FLAG_NO_SEGSORT | JZ_FLAG_NO_EARLY_EXIT));
  la.out_idx = a.out_idx;
  la.out_d2 = a.out_d2;
  la.out_row_gidx = a.out_row_gidx;
  la.stats = a.evals;
  la.self = a.spts == a.qpts;
  la.counter = nullptr;
  unsigned long long *counters = nullptr;
  if (nitems > 0) {
    // chunked launches (a.on_rows: rows of the finished z-order query range after each chunk,
    // e.g. to stream them to the host while the next chunk runs); k <= k_max only
    const int nch = (a.on_rows && a.k <= kMaxK && a.chunks > 1) ? a.chunks : 1;
    std::vector<int32_t> q0h;
    if (nch > 1) {
      q0h.resize(nitems);
      JZ_CUDA(cudaMemcpyAsync(q0h.data(), item_q0, nitems * sizeof(int32_t), cudaMemcpyDeviceToHost, st));
      JZ_CUDA(cudaStreamSynchronize(st));
    }
    const int npass = (a.k + kMaxK - 1) / kMaxK;
    if (JZ_PERSIST) {  // one zeroed work-item counter per launch
      JZ_CUDA(cudaMallocAsync(&counters, (size_t)nch * npass * sizeof(unsigned long long), st));
      JZ_CUDA(cudaMemsetAsync(counters, 0, (size_t)nch * npass * sizeof(unsigned long long), st));
    }
    for (int ch = 0; ch < nch; ++ch) {
      const int64_t i0 = nitems * ch / nch, i1 = nitems * (ch + 1) / nch;
      if (i1 <= i0) continue;
      la.item_off = i0;
      la.nitems = i1;
      const unsigned blocks = (unsigned)ceil_div(i1 - i0, kLWarps);
      // k > k_max: ceil(k / k_max) passes over the same interaction list (built for R_max(k));
      // pass c keeps only keys after the last (d2, index) of pass c-1.
      for (int c0 = 0; c0 < a.k; c0 += kMaxK) {
        la.col0 = c0;
        la.k = a.k - c0 < kMaxK ? a.k - c0 : kMaxK;
        if (counters) la.counter = counters + (size_t)ch * npass + c0 / kMaxK;
        if (la.k <= 8) launch_l<8>(la, D, blocks, st);
        else if (la.k <= 16) launch_l<16>(la, D, blocks, st);
        else launch_l<32>(la, D, blocks, st);
        JZ_LAUNCH_CHECK();
      }
      if (nch > 1) a.on_rows(q0h[i0], i1 < nitems ? (int64_t)q0h[i1] : a.nq);
    }
  }
  if (counters) JZ_CUDA(cudaFreeAsync(counters, st));
  JZ_CUDA(cudaFreeAsync(cnt, st));
  JZ_CUDA(cudaFreeAsync(off, st));
  JZ_CUDA(cudaFreeAsync(item_par, st));
  JZ_CUDA(cudaFreeAsync(item_q0, st));
#ifdef JZ_DIAG_WALK
  {
    unsigned long long h[8];
    JZ_CUDA(cudaMemcpyFromSymbolAsync(h, g_diag, sizeof(h), 0, cudaMemcpyDeviceToHost, st));
    JZ_CUDA(cudaStreamSynchronize(st));
    const double it = h[5] ? (double)h[5] : 1.0;
    fprintf(stderr, "JZ_DIAG per item: entries %.1f passing %.1f chunks %.1f leaves_warp %.1f staged %.1f (items %llu) "
            "walk pair-evals needed %.1f of %.1f\n",
            h[0] / it, h[1] / it, h[2] / it, h[3] / it, h[4] / it, h[5], h[6] / it, h[7] / it);
    const unsigned long long z[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    JZ_CUDA(cudaMemcpyToSymbolAsync(g_diag, z, sizeof(z), 0, cudaMemcpyHostToDevice, st));
  }
#endif
  JZ_CUDA(cudaFreeAsync(leaf_ce, st));
  if (par_ce) JZ_CUDA(cudaFreeAsync(par_ce, st));
}

void fof_leaf(const LeafArgs &a, const Dom &D, float b2, int32_t *par, cudaStream_t st) {
  if (a.npar == 0) return;
  int32_t *cnt = nullptr;
  int64_t *off = nullptr;
  JZ_CUDA(cudaMallocAsync(&cnt, a.npar * sizeof(int32_t), st));
  JZ_CUDA(cudaMallocAsync(&off, (a.npar + 1) * sizeof(int64_t), st));
  k_item_count<<<grid_for(a.npar, 256), 256, 0, st>>>(a.par_leaf, a.sbeg, a.npar, 32, cnt);
  JZ_LAUNCH_CHECK();
  exclusive_scan_i32_to_i64(cnt, off, a.npar, st);
  const int64_t nitems = read_i64(off + a.npar, st);
  int32_t *item_par = nullptr, *item_q0 = nullptr;
  JZ_CUDA(cudaMallocAsync(&item_par, (nitems + 1) * sizeof(int32_t), st));
  JZ_CUDA(cudaMallocAsync(&item_q0, (nitems + 1) * sizeof(int32_t), st));
  k_item_fill<<<grid_for(a.npar, 256), 256, 0, st>>>(a.par_leaf, a.sbeg, a.npar, 32, off, item_par, item_q0);
  JZ_LAUNCH_CHECK();
  const float Lmax = D.periodic ? fmaxf(fmaxf(D.L[0], D.L[1]), D.L[2]) : 0.f;
  CE *leaf_ce = nullptr, *par_ce = nullptr;
  JZ_CUDA(cudaMallocAsync(&leaf_ce, (a.nleaf > 0 ? a.nleaf : 1) * sizeof(CE), st));
  k_box_ce<<<grid_for(a.nleaf, 256), 256, 0, st>>>(a.leaf_box, a.nleaf, Lmax, leaf_ce);
  JZ_LAUNCH_CHECK();
  if (a.par_box) {
    JZ_CUDA(cudaMallocAsync(&par_ce, a.npar * sizeof(CE), st));
    k_box_ce<<<grid_for(a.npar, 256), 256, 0, st>>>(a.par_box, a.npar, Lmax, par_ce);
    JZ_LAUNCH_CHECK();
  }
  FofPK f;
  f.spts = a.spts;
  f.sbeg = a.sbeg;
  f.leaf_ce = leaf_ce;
  f.leaf_box = a.leaf_box;
  f.par_leaf = a.par_leaf;
  f.par_ce = par_ce;
  f.ispl = a.il->ispl;
  f.isrc = a.il->isrc;
  f.rlow = a.il->rlow;
  f.item_par = item_par;
  f.item_q0 = item_q0;
  f.nitems = nitems;
  f.b2 = b2;
  f.Lmax = Lmax;
  f.sorted = !(a.flags & (JZ_FLAG_NO_SEGSORT | JZ_FLAG_NO_EARLY_EXIT));
  f.par = par;
  f.stats = a.evals;
  f.counter = nullptr;
  unsigned long long *fcnt = nullptr;
  if (nitems > 0) {
    unsigned blocks = (unsigned)ceil_div(nitems, kLWarps);
    if (JZ_PERSIST) {
      JZ_CUDA(cudaMallocAsync(&fcnt, sizeof(unsigned long long), st));
      JZ_CUDA(cudaMemsetAsync(fcnt, 0, sizeof(unsigned long long), st));
      f.counter = fcnt;
      int nb = 0, dev = 0, sms = 0;
      if (D.periodic) JZ_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k_fof_leaf<true>, kLThreads, 0));
      else JZ_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k_fof_leaf<false>, kLThreads, 0));
      JZ_CUDA(cudaGetDevice(&dev));
      JZ_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
      if (nb * sms > 0 && blocks > (unsigned)(nb * sms)) blocks = (unsigned)(nb * sms);
    }
    if (D.periodic) k_fof_leaf<true><<<blocks, kLThreads, 0, st>>>(f, D);
    else k_fof_leaf<false><<<blocks, kLThreads, 0, st>>>(f, D);
    JZ_LAUNCH_CHECK();
  }
  JZ_CUDA(cudaFreeAsync(cnt, st));
  JZ_CUDA(cudaFreeAsync(off, st));
  JZ_CUDA(cudaFreeAsync(item_par, st));
  JZ_CUDA(cudaFreeAsync(item_q0, st));
  JZ_CUDA(cudaFreeAsync(leaf_ce, st));
  if (par_ce) JZ_CUDA(cudaFreeAsync(par_ce, st));
  if (fcnt) JZ_CUDA(cudaFreeAsync(fcnt, st));
}

}  // namespace jz
