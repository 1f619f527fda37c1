// jz_leaf.cu -- LeafToLeaf (Alg. 1 line 6 L321, L386, L398).
//
// B200 design:
//  * Work item = 32 consecutive (z-order) query points of one receiving plane-1 node J, one
//    query per lane, one warp per item; warps are independent (no CTA barriers).
//    The item walks J's plane-1 interaction list (sorted by r_low): the leaf-level
//    NodeToNode pass is not materialised. Leaf pairs are pruned on the fly: the bounding box
//    of the warp's queries is tested against each source node S and then, one lane per child
//    leaf, against S's child leaves (a ballot gives the survivors), with the exact monotone
//    d_low^2 bound against the warp's current max k-th distance (the early exit of P:L398).
//  * Surviving leaves are staged by the warp into its own shared-memory slot as separate
//    x / y / z / gidx arrays (coalesced 16-byte loads, leaf starts aligned to 4, tails padded
//    with NaN coordinates so their d2 is NaN and never passes a comparison).
//  * Distances: two sources per packed f32x2 instruction, query coordinate as the broadcast
//    operand: FADD2 x3, FMUL2, FFMA2 x2 per source pair = the canonical scalar formula with
//    per-element round-to-nearest (bit-identical). Periodic leaf pairs whose pairs all wrap
//    the same way get one extra exact FADD2 per axis; straddling pairs use the per-pair select.
//  * Filtering: per group of 4 sources the lane compares min(d2) with its k-th distance; the
//    insertion slow path runs only when some lane passes. Top-k: sorted register list of
//    64-bit keys (d2_bits << 32 | gidx + 1): unsigned order == (d2, index) order (R2),
//    initialised with sentinels at R_max^2 of J (bounds every contained query's k-th distance).
//  * Rows are written straight to their final place (input or z order): no reorder pass.
#include "jz_common.cuh"
#include "jz_internal.h"

namespace jz {

constexpr int kLWarps = 2;
constexpr int kLThreads = kLWarps * 32;
constexpr int kLCap = 256;  // staged source points per warp (4 KB SoA)
constexpr int kQCap = 16;   // per-lane candidate queue (4 KB per warp)

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

// Sorted insert of `key` (known to be < a[K-1]) into a[0..K). The list is cut into quarters;
// a quarter is touched only if key < its last element, so the common late insertion near the
// tail costs one quarter of the compare/select network.
template <int K>
__device__ __forceinline__ void topk_insert(u64 (&a)[K], u64 key) {
  constexpr int Q = K / 4;
#pragma unroll
  for (int q = 3; q >= 0; --q) {
    if (key < a[q * Q + Q - 1]) {
#pragma unroll
      for (int j = q * Q + Q - 1; j >= q * Q; --j) {
        const bool mv = j > 0 && key < a[j > 0 ? j - 1 : 0];
        a[j] = mv ? a[j > 0 ? j - 1 : 0] : (key < a[j] ? key : a[j]);
      }
    }
  }
}

struct LeafPK {
  const float4 *spts;        // source points, z order (type-separated)
  const int32_t *sbeg;       // [nleaf+1] first source of each leaf
  const float4 *qpts;        // query points, z order
  const int32_t *qbeg;       // [nleaf+1] first query of each leaf
  const int32_t *qin;        // [nq] input row of each query
  const NodeBox *leaf_box;   // [nleaf]
  const int32_t *par_leaf;   // [npar+1] first leaf of each receiving parent
  const NodeBox *par_box;    // [npar] or nullptr
  const int64_t *ispl;       // parent-level interaction list
  const int32_t *isrc;
  const float *rlow;
  const float *rmax2;        // [npar] or nullptr (= +inf)
  const int32_t *item_par;   // [nitems] receiving parent of each 32-query work item
  const int32_t *item_q0;    // [nitems] first query (sorted position) of the item
  int64_t nitems;
  int k;      // neighbours found by this pass (<= K)
  int col0;   // first output column of this pass (k > k_max chunking)
  int ldo;    // output row stride (total k)
  int order;
  int early;
  int sorted;
  int32_t *out_idx;
  float *out_d2;
  int32_t *out_row_gidx;
  unsigned long long *stats;  // [0] distance evaluations, [1] top-k insertions (or nullptr)
};

// per-axis shift class of a (query box, source box) pair: 0 = no wrap for any pair,
// 1 = every pair wraps by -L, 2 = every pair wraps by +L (shift returned in sh),
// 3 = straddles (per-pair select)
__device__ __forceinline__ int shift_class(float qlo, float qhi, float slo, float shi, float L, float h, float &sh) {
  const float tmin = __fsub_rn(qlo, shi), tmax = __fsub_rn(qhi, slo);
  sh = 0.f;
  if (tmin >= h) {
    sh = -L;
    return 1;
  }
  if (tmax < -h) {
    sh = L;
    return 2;
  }
  if (tmin >= -h && tmax < h) return 0;
  return 3;
}

__device__ __forceinline__ bool any_straddle(int c) {
  return ((c & 3) == 3) || (((c >> 2) & 3) == 3) || (((c >> 4) & 3) == 3);
}

struct WarpBuf {
  float x[kLCap], y[kLCap], z[kLCap];
  int g[kLCap];
  u64 q[kQCap][32];  // candidate queue, lane-minor
};

template <int K, bool LB>
struct Lane {
  u64 tk[K];
  u64 lb;    // keys <= lb were found by earlier passes (0 on the first pass)
  float kth;
  unsigned ins;
  int qn;    // queued candidates
  bool act;  // lane holds a query (inactive lanes keep kth = -1)
};

// Insert the lane's queued candidates: all lanes drain their queues in parallel, so the
// warp runs max(queue length) insertion rounds instead of one per candidate group.
template <int K, bool LB>
__device__ __forceinline__ void flush(WarpBuf &B, Lane<K, LB> &L) {
  const int lane = threadIdx.x & 31;
  const int mx = __reduce_max_sync(0xffffffffu, (unsigned)L.qn);
  for (int i = 0; i < mx; ++i) {
    if (i < L.qn) {
      const u64 key = B.q[i][lane];
      if (key < L.tk[K - 1]) {
        topk_insert<K>(L.tk, key);
        ++L.ins;
      }
    }
  }
  L.kth = L.act ? __uint_as_float((unsigned)(L.tk[K - 1] >> 32)) : -1.f;
  L.qn = 0;
}

template <int K, bool LB>
__device__ __forceinline__ void cand(Lane<K, LB> &L, float d2, int g) {
  if (d2 <= L.kth) {
    const u64 key = ((u64)__float_as_uint(d2) << 32) | (unsigned)(g + 1);
    if (key < L.tk[K - 1] && (!LB || key > L.lb)) {
      topk_insert<K>(L.tk, key);
      L.kth = __uint_as_float((unsigned)(L.tk[K - 1] >> 32));
      ++L.ins;
    }
  }
}

template <int K, bool LB>
__device__ __forceinline__ void enqueue(WarpBuf &B, Lane<K, LB> &L, float d2, int g) {
  if (d2 <= L.kth) {
    const u64 key = ((u64)__float_as_uint(d2) << 32) | (unsigned)(g + 1);
    if (!LB || key > L.lb) {
      B.q[L.qn][threadIdx.x & 31] = key;
      ++L.qn;
    }
  }
}

// evaluate staged sources [0, n) (n multiple of 4, NaN padded) against the lane's query
template <int K, bool LB, bool SHIFT>
__device__ __forceinline__ void eval_block(WarpBuf &B, int n, float qx, float qy, float qz, float shx, float shy,
                                           float shz, Lane<K, LB> &L) {
  const u64 QX = pk(qx, qx), QY = pk(qy, qy), QZ = pk(qz, qz);
  const u64 SX = pk(shx, shx), SY = pk(shy, shy), SZ = pk(shz, shz);
  for (int j = 0; j < n; j += 4) {
    const float4 X = *reinterpret_cast<const float4 *>(&B.x[j]);
    const float4 Y = *reinterpret_cast<const float4 *>(&B.y[j]);
    const float4 Z = *reinterpret_cast<const float4 *>(&B.z[j]);
    u64 tx0 = sub2(QX, pk(X.x, X.y)), tx1 = sub2(QX, pk(X.z, X.w));
    u64 ty0 = sub2(QY, pk(Y.x, Y.y)), ty1 = sub2(QY, pk(Y.z, Y.w));
    u64 tz0 = sub2(QZ, pk(Z.x, Z.y)), tz1 = sub2(QZ, pk(Z.z, Z.w));
    if (SHIFT) {
      tx0 = add2(tx0, SX);
      tx1 = add2(tx1, SX);
      ty0 = add2(ty0, SY);
      ty1 = add2(ty1, SY);
      tz0 = add2(tz0, SZ);
      tz1 = add2(tz1, SZ);
    }
    const u64 d0 = fma2(tz0, tz0, fma2(ty0, ty0, mul2(tx0, tx0)));
    const u64 d1 = fma2(tz1, tz1, fma2(ty1, ty1, mul2(tx1, tx1)));
    float a0, a1, a2, a3;
    upk(d0, a0, a1);
    upk(d1, a2, a3);
    const float m = fminf(fminf(a0, a1), fminf(a2, a3));  // NaN padding is ignored by min
    if (__any_sync(0xffffffffu, m <= L.kth)) {
      const int4 G = *reinterpret_cast<const int4 *>(&B.g[j]);
      enqueue<K, LB>(B, L, a0, G.x);
      enqueue<K, LB>(B, L, a1, G.y);
      enqueue<K, LB>(B, L, a2, G.z);
      enqueue<K, LB>(B, L, a3, G.w);
      if (__any_sync(0xffffffffu, L.qn > kQCap - 4)) flush<K, LB>(B, L);
    }
  }
  if (__any_sync(0xffffffffu, L.qn > 0)) flush<K, LB>(B, L);
}

template <int K, bool LB>
__device__ __forceinline__ void eval_generic(const WarpBuf &B, int n, float qx, float qy, float qz, const Dom &D,
                                             Lane<K, LB> &L) {
  for (int j = 0; j < n; ++j) {
    const float d2 = canon_d2_per(qx, qy, qz, B.x[j], B.y[j], B.z[j], D);  // NaN padding -> NaN
    cand<K, LB>(L, d2, B.g[j]);
  }
}

// Visit the child leaves [la, lb) of one source node, skipping [xa, xb): one lane tests one
// leaf (exact box bound vs the warp's current max k-th distance), then every lane tests its own
// query against each surviving leaf (skip unless some lane needs it); survivors are staged in
// batches of one periodic shift class and evaluated.
template <int K, bool LB, bool PER>
__device__ __forceinline__ void visit_leaves(const LeafPK &a, const Dom &D, WarpBuf &B, const NodeBox &wbox, float wmax,
                                             int la, int lb, int xa, int xb, float qx, float qy, float qz, bool act,
                                             Lane<K, LB> &L, unsigned long long &nev) {
  const int lane = threadIdx.x & 31;
  for (int l0 = la; l0 < lb; l0 += 32) {
    const int l = l0 + lane;
    bool pass = false;
    int cls = 0;
    if (l < lb && (l < xa || l >= xb)) {
      const NodeBox lbx = a.leaf_box[l];
      pass = box_dlow2(wbox, lbx, D) <= wmax;
      if (PER && pass) {
        float shd;
        cls |= shift_class(wbox.lo.x, wbox.hi.x, lbx.lo.x, lbx.hi.x, D.L[0], D.h[0], shd) << 0;
        cls |= shift_class(wbox.lo.y, wbox.hi.y, lbx.lo.y, lbx.hi.y, D.L[1], D.h[1], shd) << 2;
        cls |= shift_class(wbox.lo.z, wbox.hi.z, lbx.lo.z, lbx.hi.z, D.L[2], D.h[2], shd) << 4;
      }
    }
    unsigned bal = __ballot_sync(0xffffffffu, pass);
    while (bal) {
      // batch consecutive surviving leaves of one shift class into the warp buffer
      const int first = __ffs(bal) - 1;
      const int c0 = __shfl_sync(0xffffffffu, cls, first);
      int n = 0;
      while (bal) {
        const int src = __ffs(bal) - 1;
        if (__shfl_sync(0xffffffffu, cls, src) != c0) break;
        // per-lane test: does any lane's query reach this leaf within its own k-th distance?
        {
          const NodeBox lbx = a.leaf_box[l0 + src];
          const bool need = L.act && pt_box_dlow2(qx, qy, qz, lbx, D) <= L.kth;
          if (!__any_sync(0xffffffffu, need)) {
            bal &= bal - 1;
            continue;
          }
        }
        const int lp = a.sbeg[l0 + src], m = a.sbeg[l0 + src + 1] - lp;
        if (n + ((m + 3) & ~3) > kLCap) break;
        bal &= bal - 1;
        for (int t = lane; t < ((m + 3) & ~3); t += 32) {
          float4 p = make_float4(__int_as_float(0x7fc00000), __int_as_float(0x7fc00000), __int_as_float(0x7fc00000),
                                 0.f);
          if (t < m) p = a.spts[lp + t];
          B.x[n + t] = p.x;
          B.y[n + t] = p.y;
          B.z[n + t] = p.z;
          B.g[n + t] = __float_as_int(p.w);
        }
        nev += act ? (unsigned)m : 0u;
        n += (m + 3) & ~3;
      }
      __syncwarp();
      if (n == 0) continue;
      if (!PER || c0 == 0) {
        eval_block<K, LB, false>(B, n, qx, qy, qz, 0.f, 0.f, 0.f, L);
      } else if (!any_straddle(c0)) {  // no axis straddles: uniform exact shift
        float s0, s1, s2;
        const NodeBox lbx = a.leaf_box[l0 + first];
        shift_class(wbox.lo.x, wbox.hi.x, lbx.lo.x, lbx.hi.x, D.L[0], D.h[0], s0);
        shift_class(wbox.lo.y, wbox.hi.y, lbx.lo.y, lbx.hi.y, D.L[1], D.h[1], s1);
        shift_class(wbox.lo.z, wbox.hi.z, lbx.lo.z, lbx.hi.z, D.L[2], D.h[2], s2);
        eval_block<K, LB, true>(B, n, qx, qy, qz, s0, s1, s2, L);
      } else {
        eval_generic<K, LB>(B, n, qx, qy, qz, D, L);
      }
      __syncwarp();
    }
  }
}

__device__ __forceinline__ float warp_max_kth(float kth) {
  return __uint_as_float(__reduce_max_sync(0xffffffffu, __float_as_uint(fmaxf(kth, 0.f))));
}

template <int K, bool LB, bool PER>
__global__ void __launch_bounds__(kLThreads) k_leaf(LeafPK a, Dom D) {
  __shared__ __align__(16) WarpBuf s_buf[kLWarps];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t item = (int64_t)blockIdx.x * kLWarps + warp;
  if (item >= a.nitems) return;
  WarpBuf &B = s_buf[warp];
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
  NodeBox wbox;
  wbox.lo = make_float4(blo[0], blo[1], blo[2], 0.f);
  wbox.hi = make_float4(bhi[0], bhi[1], bhi[2], 0.f);

  const float R0 = a.rmax2 ? a.rmax2[J] : INFINITY;
  Lane<K, LB> L;
  {
    const u64 sentinel = ((u64)__float_as_uint(R0) << 32) | 0xffffffffull;
#pragma unroll
    for (int j = 0; j < K; ++j) L.tk[j] = (j < K - a.k) ? 0ull : sentinel;
    L.kth = act ? R0 : -1.f;  // inactive lanes never pass a comparison
    L.lb = 0;
    if (LB && act) {  // continue after the last (d2, index) of the previous pass
      const int64_t o = row * a.ldo + a.col0 - 1;
      L.lb = ((u64)__float_as_uint(a.out_d2[o]) << 32) | (unsigned)(a.out_idx[o] + 1);
    }
    L.ins = 0;
    L.qn = 0;
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
    visit_leaves<K, LB, PER>(a, D, B, wbox, INFINITY, xa, xb, 0, 0, qx, qy, qz, act, L, nev);
  }
  const int64_t eb = a.ispl[J], ee = a.ispl[J + 1];
  for (int64_t e = eb; e < ee; ++e) {
    const int S = a.isrc[e];
    const float wmax = a.early ? warp_max_kth(L.kth) : INFINITY;
    if (a.rlow[e] > wmax) {
      if (a.sorted) break;
      continue;
    }
    if (a.par_box && box_dlow2(wbox, a.par_box[S], D) > wmax) continue;
    visit_leaves<K, LB, PER>(a, D, B, wbox, wmax, a.par_leaf[S], a.par_leaf[S + 1], S == J ? xa : 0, S == J ? xb : 0, qx,
                         qy, qz, act, L, nev);
  }
  if (a.stats) {
    unsigned long long tot = nev, ins = L.ins;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      tot += __shfl_xor_sync(0xffffffffu, tot, o);
      ins += __shfl_xor_sync(0xffffffffu, ins, o);
    }
    if (lane == 0) {
      atomicAdd(&a.stats[0], tot);
      atomicAdd(&a.stats[1], ins);
    }
  }
  if (act) {
    int32_t *oi = a.out_idx + row * a.ldo + a.col0;
    float *od = a.out_d2 + row * a.ldo + a.col0;
#pragma unroll
    for (int j = 0; j < K; ++j) {
      if (j >= K - a.k) {
        oi[j - (K - a.k)] = (int32_t)((unsigned)(L.tk[j] & 0xffffffffu) - 1u);
        od[j - (K - a.k)] = __uint_as_float((unsigned)(L.tk[j] >> 32));
      }
    }
    if (a.out_row_gidx) a.out_row_gidx[row] = __float_as_int(qw);
  }
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

template <int K>
static void launch_l(const LeafPK &la, const Dom &D, unsigned blocks, cudaStream_t st) {
  if (la.col0 > 0) {  // later pass of a k > k_max query
    if (D.periodic) k_leaf<K, true, true><<<blocks, kLThreads, 0, st>>>(la, D);
    else k_leaf<K, true, false><<<blocks, kLThreads, 0, st>>>(la, D);
  } else {
    if (D.periodic) k_leaf<K, false, true><<<blocks, kLThreads, 0, st>>>(la, D);
    else k_leaf<K, false, false><<<blocks, kLThreads, 0, st>>>(la, D);
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

  LeafPK la;
  la.spts = a.spts;
  la.sbeg = a.sbeg;
  la.qpts = a.qpts;
  la.qbeg = a.qbeg;
  la.qin = a.qin;
  la.leaf_box = a.leaf_box;
  la.par_leaf = a.par_leaf;
  la.par_box = a.par_box;
  la.ispl = a.il->ispl;
  la.isrc = a.il->isrc;
  la.rlow = a.il->rlow;
  la.rmax2 = a.rmax2;
  la.item_par = item_par;
  la.item_q0 = item_q0;
  la.nitems = nitems;
  la.ldo = a.k;
  la.order = a.order;
  la.early = !(a.flags & JZ_FLAG_NO_EARLY_EXIT);
  la.sorted = !(a.flags & (JZ_FLAG_NO_SEGSORT | JZ_FLAG_NO_EARLY_EXIT));
  la.out_idx = a.out_idx;
  la.out_d2 = a.out_d2;
  la.out_row_gidx = a.out_row_gidx;
  la.stats = a.evals;
  if (nitems > 0) {
    const unsigned blocks = (unsigned)ceil_div(nitems, kLWarps);
    // k > k_max: ceil(k / k_max) passes over the same interaction list (built for R_max(k));
    // pass c keeps only keys after the last (d2, index) of pass c-1.
    for (int c0 = 0; c0 < a.k; c0 += kMaxK) {
      la.col0 = c0;
      la.k = a.k - c0 < kMaxK ? a.k - c0 : kMaxK;
      if (la.k <= 8) launch_l<8>(la, D, blocks, st);
      else if (la.k <= 16) launch_l<16>(la, D, blocks, st);
      else launch_l<32>(la, D, blocks, st);
      JZ_LAUNCH_CHECK();
    }
  }
  JZ_CUDA(cudaFreeAsync(cnt, st));
  JZ_CUDA(cudaFreeAsync(off, st));
  JZ_CUDA(cudaFreeAsync(item_par, st));
  JZ_CUDA(cudaFreeAsync(item_q0, st));
}

}  // namespace jz
