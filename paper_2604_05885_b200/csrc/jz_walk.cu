// jz_walk.cu -- dual tree walk down the plane hierarchy (
// PAPER.md Alg. 1 lines 1-5 L309-322, Alg. 2 NodeToNode L337-352, Alg. 3 FindRmax L354-384,
// early exit on sorted r_low L395-398).
//
// Layout: an interaction list at plane level p is (ispl [nrecv+1] int64, isrc int32, rlow f32)
// with rlow = d_low^2 of the (receiver, source) pair. Receivers at level p+1 are "parents";
// the kernels below move the list one plane down:
//   k_n2n<RMAX>   one warp per receiving parent, one lane per child: a register
//                 count-heap of N_r = 8 (d_up^2, count) entries over the children of
//                 every source parent in the segment, staged in shared memory -> R_max^2.
//   k_n2n<COUNT>  #source children with d_low^2 <= R_max^2
//   scan          CumulativeSumPrep0 (jz_scan.cu)
//   k_n2n<INSERT> write isrc / rlow at the scanned offsets
//   k_segsort     sort each receiver's segment by (rlow, isrc) (P:L396 bitonic network).
// All bounds are squared FP32 values that bound the canonical d2 exactly (jz_common.cuh).
#include <climits>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "jz_common.cuh"
#include "jz_internal.h"

namespace jz {

constexpr int kHeap = 8;        // N_r (R13)

enum { RMAX = 0, COUNT = 1, INSERT = 2 };

void IList::release(cudaStream_t st) {
  if (ispl) cudaFreeAsync(ispl, st);
  if (isrc) cudaFreeAsync(isrc, st);
  if (rlow) cudaFreeAsync(rlow, st);
  ispl = nullptr;
  isrc = nullptr;
  rlow = nullptr;
  nrecv = total = 0;
}

__global__ void k_dense_init(int64_t S, int64_t *__restrict__ ispl, int32_t *__restrict__ isrc,
                             float *__restrict__ rlow) {
  // ispl_i = S i, isrc_j = j mod S; r_low = 0 at the top
  const int64_t m = S * S > S + 1 ? S * S : S + 1;
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < m; j += (int64_t)gridDim.x * blockDim.x) {
    if (j < S * S) {
      isrc[j] = (int32_t)(j % S);
      rlow[j] = 0.f;
    }
    if (j <= S) ispl[j] = S * j;
  }
}

__global__ void k_super_beg(int64_t S, int64_t ntop, int ngr, int32_t *__restrict__ beg) {
  // Alg. 1 line 1: spl^(P) = Range(0, N_top, NGR)
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j <= S; j += (int64_t)gridDim.x * blockDim.x)
    beg[j] = (int32_t)min(j * ngr, ntop);
}

// ---- count heap: 8 slots sorted by radius, empty slots = (+inf, 0)
struct CountHeap {
  float r[kHeap];
  int c[kHeap];
  int tot;
};

__device__ __forceinline__ float heap_radius(const CountHeap &h, int k) {
  int cum = 0;
  float R = INFINITY;
  bool found = false;
#pragma unroll
  for (int j = 0; j < kHeap; ++j) {
    cum += h.c[j];
    if (!found && cum >= k) {
      R = h.r[j];
      found = true;
    }
  }
  return R;
}

__device__ __forceinline__ void heap_insert(CountHeap &h, float r, int c, int k) {
  if (h.c[kHeap - 1] == 0 || h.tot - h.c[kHeap - 1] + c >= k) {
    // ordered insert after equal radii, discarding the last slot
    h.tot += c - h.c[kHeap - 1];
#pragma unroll
    for (int j = kHeap - 1; j > 0; --j) {
      const bool mv = h.r[j - 1] > r;
      const bool here = !mv && h.r[j] > r;
      h.r[j] = mv ? h.r[j - 1] : (here ? r : h.r[j]);
      h.c[j] = mv ? h.c[j - 1] : (here ? c : h.c[j]);
    }
    if (h.r[0] > r) {
      h.r[0] = r;
      h.c[0] = c;
    }
  } else {
    // dropping the last would leave < k: add the count to the first larger radius
    bool done = false;
#pragma unroll
    for (int j = 0; j < kHeap; ++j) {
      if (!done && h.r[j] > r) {
        h.c[j] += c;
        done = true;
      }
    }
    if (!done) {  // no larger radius: the last slot absorbs it at radius r (R13)
      h.r[kHeap - 1] = r;
      h.c[kHeap - 1] += c;
    }
    h.tot += c;
  }
}

// One warp per receiving parent (4 parents per CTA), one lane per child; the source
// parent's children are staged in the warp's shared-memory slot. Warps are independent
// (no CTA barriers); the RMAX early exit is a warp vote.
#ifndef JZ_N2N_WARPS
#define JZ_N2N_WARPS 1
#endif
constexpr int kN2NWarps = JZ_N2N_WARPS;
constexpr int kN2NWStage = 128;  // staged source children per warp (4 KB)

template <int MODE>
__global__ void __launch_bounds__(kN2NWarps * 32) k_n2n(const int32_t *__restrict__ pbeg, int64_t npar,
                                                       const int64_t *__restrict__ ispl,
                                                       const int32_t *__restrict__ isrc, const float *__restrict__ rlow,
                                                       const NodeBox *__restrict__ cbox, Dom D, int k, int sorted,
                                                       int early, float *__restrict__ rmax2, int32_t *__restrict__ cnt,
                                                       const int64_t *__restrict__ ispl_out,
                                                       int32_t *__restrict__ isrc_out, float *__restrict__ rlow_out,
                                                       const uint8_t *__restrict__ qf) {
  // qf (optional): receivers holding at least one query; the others get no list (joint trees
  // of separate / partial query sets: source-only nodes never receive)
  __shared__ NodeBox s_box[kN2NWarps][kN2NWStage];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t J = (int64_t)blockIdx.x * kN2NWarps + warp;
  if (J >= npar) return;
  NodeBox *sb = s_box[warp];
  const int cb = pbeg[J], ce = pbeg[J + 1];
  const int64_t eb = ispl[J], ee = ispl[J + 1];
  for (int c0 = cb; c0 < ce; c0 += 32) {
    const int i = c0 + lane;
    const bool inrange = i < ce;
    const bool valid = inrange && (!qf || qf[i]);
    NodeBox mb;
    if (valid) mb = cbox[i];
    CountHeap h;
    float R = INFINITY;
    int count = 0;
    int64_t wp = 0;
    float Rchunk = 0.f;
    if (MODE == RMAX) {
#pragma unroll
      for (int j = 0; j < kHeap; ++j) {
        h.r[j] = INFINITY;
        h.c[j] = 0;
      }
      h.tot = 0;
    } else {
      R = valid ? rmax2[i] : 0.f;
      if (MODE == INSERT && valid) wp = ispl_out[i];
      Rchunk = R;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) Rchunk = fmaxf(Rchunk, __shfl_xor_sync(0xffffffffu, Rchunk, o));
    }
    for (int64_t e = eb; e < ee; ++e) {
      const int S = isrc[e];
      const float rl = rlow[e];
      if (early) {
        // early exit: no child can use this entry (d_low of children >= rl)
        const bool need = MODE == RMAX ? __any_sync(0xffffffffu, valid && rl < R) : rl <= Rchunk;
        if (!need) {
          if (sorted) break;
          continue;
        }
      }
      const int sb0 = pbeg[S], se = pbeg[S + 1];
      for (int s0 = sb0; s0 < se; s0 += kN2NWStage) {
        const int sn = min(kN2NWStage, se - s0);
        __syncwarp();
        for (int t = lane; t < sn; t += 32) sb[t] = cbox[s0 + t];
        __syncwarp();
        if (valid) {
          for (int t = 0; t < sn; ++t) {
            const NodeBox sbx = sb[t];
            if (MODE == RMAX) {
              const float r2 = box_dup2(mb, sbx, D);
              if (r2 < R) {
                heap_insert(h, r2, box_count(sbx), k);
                R = heap_radius(h, k);
              }
            } else {
              const float dl = box_dlow2(mb, sbx, D);
              if (dl <= R) {
                if (MODE == COUNT) ++count;
                else {
                  isrc_out[wp] = s0 + t;
                  rlow_out[wp] = dl;
                  ++wp;
                }
              }
            }
          }
        }
      }
    }
    if (inrange) {
      if (MODE == RMAX) rmax2[i] = valid ? R : 0.f;
      if (MODE == COUNT) cnt[i] = valid ? count : 0;
    }
  }
}

// ---- flat variant: one thread per receiving child (all lanes busy whatever the fan-out c); the
// source boxes come through L1 (consecutive children share their parent's list, so a warp mostly
// reads the same boxes). Same decisions as k_n2n, per child instead of per 32-child chunk.
#ifndef JZ_N2N_WC
#define JZ_N2N_WC 1  // warp per receiving child (k_n2n_wc) instead of a thread per child (k_n2n_flat)
#endif
#ifndef JZ_N2N_WC_MAX
#define JZ_N2N_WC_MAX (1 << 19)  // planes with at least this many children: a thread per child
#endif
#ifndef JZ_N2N_FLAT
#define JZ_N2N_FLAT 1
#endif
__global__ void k_child_parent(const int32_t *__restrict__ pbeg, int64_t npar, int32_t *__restrict__ cpar) {
  for (int64_t P = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; P < npar; P += (int64_t)gridDim.x * blockDim.x)
    for (int c = pbeg[P]; c < pbeg[P + 1]; ++c) cpar[c] = (int32_t)P;
}

template <int MODE>
__global__ void __launch_bounds__(256) k_n2n_flat(const int32_t *__restrict__ cpar, int64_t nchild,
                                                  const int32_t *__restrict__ pbeg, const int64_t *__restrict__ ispl,
                                                  const int32_t *__restrict__ isrc, const float *__restrict__ rlow,
                                                  const NodeBox *__restrict__ cbox, Dom D, int k, int sorted, int early,
                                                  float *__restrict__ rmax2, int32_t *__restrict__ cnt,
                                                  const int64_t *__restrict__ ispl_out, int32_t *__restrict__ isrc_out,
                                                  float *__restrict__ rlow_out, const uint8_t *__restrict__ qf) {
  for (int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; c < nchild; c += (int64_t)gridDim.x * blockDim.x) {
    if (qf && !qf[c]) {  // no queries below: no list
      if (MODE == RMAX) rmax2[c] = 0.f;
      if (MODE == COUNT) cnt[c] = 0;
      continue;
    }
    const int J = cpar[c];
    const NodeBox mb = cbox[c];
    CountHeap h;
    float R = INFINITY;
    if (MODE == RMAX) {
#pragma unroll
      for (int j = 0; j < kHeap; ++j) {
        h.r[j] = INFINITY;
        h.c[j] = 0;
      }
      h.tot = 0;
    } else {
      R = rmax2[c];
    }
    int count = 0;
    int64_t wp = MODE == INSERT ? ispl_out[c] : 0;
    const int64_t eb = ispl[J], ee = ispl[J + 1];
    for (int64_t e = eb; e < ee; ++e) {
      const float rl = rlow[e];
      if (early && (MODE == RMAX ? !(rl < R) : !(rl <= R))) {
        if (sorted) break;
        continue;
      }
      const int S = isrc[e];
      for (int s = pbeg[S]; s < pbeg[S + 1]; ++s) {
        const NodeBox sbx = cbox[s];
        if (MODE == RMAX) {
          const float r2 = box_dup2(mb, sbx, D);
          if (r2 < R) {
            heap_insert(h, r2, box_count(sbx), k);
            R = heap_radius(h, k);
          }
        } else {
          const float dl = box_dlow2(mb, sbx, D);
          if (dl <= R) {
            if (MODE == COUNT) ++count;
            else {
              isrc_out[wp] = s;
              rlow_out[wp] = dl;
              ++wp;
            }
          }
        }
      }
    }
    if (MODE == RMAX) rmax2[c] = R;
    if (MODE == COUNT) cnt[c] = count;
  }
}

// ---- warp-per-child variant (JZ_N2N_WC): one warp per receiving child, lanes over the children of
// each list entry (box loads and bounds in parallel, 32x the threads of k_n2n_flat). RMAX runs the
// same sequential count heap as the flat kernel, every lane redundantly on the shuffled candidates in
// list order, so R, the counts and the list order are identical (results bit-identical).
template <int MODE>
__global__ void __launch_bounds__(256) k_n2n_wc(const int32_t *__restrict__ cpar, int64_t nchild,
                                                const int32_t *__restrict__ pbeg, const int64_t *__restrict__ ispl,
                                                const int32_t *__restrict__ isrc, const float *__restrict__ rlow,
                                                const NodeBox *__restrict__ cbox, Dom D, int k, int sorted, int early,
                                                float *__restrict__ rmax2, int32_t *__restrict__ cnt,
                                                const int64_t *__restrict__ ispl_out, int32_t *__restrict__ isrc_out,
                                                float *__restrict__ rlow_out, const uint8_t *__restrict__ qf) {
  const int lane = threadIdx.x & 31;
  const int64_t nw = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t c = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); c < nchild; c += nw) {
    if (qf && !qf[c]) {
      if (lane == 0) {
        if (MODE == RMAX) rmax2[c] = 0.f;
        if (MODE == COUNT) cnt[c] = 0;
      }
      continue;
    }
    const int J = cpar[c];
    const NodeBox mb = cbox[c];
    CountHeap h;
    float R = INFINITY;
    if (MODE == RMAX) {
#pragma unroll
      for (int j = 0; j < kHeap; ++j) {
        h.r[j] = INFINITY;
        h.c[j] = 0;
      }
      h.tot = 0;
    } else {
      R = rmax2[c];
    }
    int count = 0;
    int64_t wp = MODE == INSERT ? ispl_out[c] : 0;
    const int64_t eb = ispl[J], ee = ispl[J + 1];
    for (int64_t e = eb; e < ee; ++e) {
      const float rl = rlow[e];
      if (early && (MODE == RMAX ? !(rl < R) : !(rl <= R))) {
        if (sorted) break;
        continue;
      }
      const int S = isrc[e];
      const int s0 = pbeg[S], s1 = pbeg[S + 1];
      for (int b = s0; b < s1; b += 32) {
        const int s = b + lane;
        const bool in = s < s1;
        if (MODE == RMAX) {
          float r2 = INFINITY;
          int bc = 0;
          if (in) {
            const NodeBox sbx = cbox[s];
            r2 = box_dup2(mb, sbx, D);
            bc = box_count(sbx);
          }
          unsigned m = __ballot_sync(0xffffffffu, in && r2 < R);
          while (m) {  // list order, the same test against the running radius as the flat kernel
            const int j = __ffs(m) - 1;
            m &= m - 1;
            const float rj = __shfl_sync(0xffffffffu, r2, j);
            const int cj = __shfl_sync(0xffffffffu, bc, j);
            if (rj < R) {
              heap_insert(h, rj, cj, k);
              R = heap_radius(h, k);
            }
          }
        } else {
          float dl = INFINITY;
          if (in) dl = box_dlow2(mb, cbox[s], D);
          const bool ok = in && dl <= R;
          const unsigned bal = __ballot_sync(0xffffffffu, ok);
          if (MODE == INSERT && ok) {
            const int64_t o = wp + __popc(bal & ((1u << lane) - 1u));
            isrc_out[o] = s;
            rlow_out[o] = dl;
          }
          wp += __popc(bal);
          count += __popc(bal);
        }
      }
    }
    if (lane == 0) {
      if (MODE == RMAX) rmax2[c] = R;
      if (MODE == COUNT) cnt[c] = count;
    }
  }
}

// receivers holding queries: leaves from the query leaf starts, upper planes by OR over children
__global__ void k_qflag_leaf(const int32_t *__restrict__ qbeg, int64_t n, uint8_t *__restrict__ f) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    f[i] = qbeg[i + 1] > qbeg[i];
}
__global__ void k_qflag_up(const int32_t *__restrict__ beg, int64_t n, const uint8_t *__restrict__ fc,
                           uint8_t *__restrict__ f) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    uint8_t v = 0;
    for (int c = beg[i]; c < beg[i + 1] && !v; ++c) v = fc[c];
    f[i] = v;
  }
}

// ---- segment sort: one warp per receiver, bitonic network in shared memory
constexpr int kSegMax = 1024;
constexpr int kSegWarps = 4;

__global__ void __launch_bounds__(kSegWarps * 32) k_segsort(const int64_t *__restrict__ ispl, int64_t nrecv,
                                                          int32_t *__restrict__ isrc, float *__restrict__ rlow) {
  __shared__ unsigned long long s_k[kSegWarps][kSegMax];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  unsigned long long *sk = s_k[w];
  for (int64_t seg = (int64_t)blockIdx.x * kSegWarps + w; seg < nrecv; seg += (int64_t)gridDim.x * kSegWarps) {
    const int64_t b = ispl[seg];
    const int m = (int)(ispl[seg + 1] - b);
    if (m <= 1) continue;
    if (m > kSegMax) {
      // too long to sort here: r_low = 0 is a valid lower bound and trivially sorted
      for (int i = lane; i < m; i += 32) rlow[b + i] = 0.f;
      continue;
    }
    int P = 32;
    while (P < m) P <<= 1;
    for (int i = lane; i < P; i += 32)
      sk[i] = i < m ? (((unsigned long long)__float_as_uint(rlow[b + i]) << 32) | (unsigned)isrc[b + i]) : ~0ull;
    __syncwarp();
    for (int size = 2; size <= P; size <<= 1) {
      for (int stride = size >> 1; stride > 0; stride >>= 1) {
        for (int i = lane; i < (P >> 1); i += 32) {
          const int lo = 2 * stride * (i / stride) + (i % stride);
          const int hi = lo + stride;
          const bool asc = (lo & size) == 0;
          unsigned long long x = sk[lo], y = sk[hi];
          if ((x > y) == asc) {
            sk[lo] = y;
            sk[hi] = x;
          }
        }
        __syncwarp();
      }
    }
    for (int i = lane; i < m; i += 32) {
      unsigned long long v = sk[i];
      isrc[b + i] = (int32_t)(v & 0xffffffffu);
      rlow[b + i] = __uint_as_float((unsigned)(v >> 32));
    }
    __syncwarp();
  }
}

__global__ void k_fill_f32(float *__restrict__ a, int64_t m, float v) {
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < m; j += (int64_t)gridDim.x * blockDim.x) a[j] = v;
}

void walk_to(const std::vector<Plane> &planes, const Dom &D, int k, int ngr, unsigned flags, int stop, IList &out_il,
             float **rmax2_out, int32_t **superbeg_out, cudaStream_t st, float fixed_r2, const int32_t *qbeg) {
  const int P = (int)planes.size();
  // query-holding receivers per plane (only when the queries are a subset of the points)
  std::vector<uint8_t *> qf(P, nullptr);
  if (qbeg) {
    for (int p = 0; p < P; ++p) {
      JZ_CUDA(cudaMallocAsync(&qf[p], planes[p].nnodes > 0 ? planes[p].nnodes : 1, st));
      if (p == 0) k_qflag_leaf<<<grid_for(planes[0].nnodes, 256), 256, 0, st>>>(qbeg, planes[0].nnodes, qf[0]);
      else k_qflag_up<<<grid_for(planes[p].nnodes, 256), 256, 0, st>>>(planes[p].beg, planes[p].nnodes, qf[p - 1], qf[p]);
      JZ_LAUNCH_CHECK();
    }
  }
  const int top = P - 1;
  const int64_t ntop = planes[top].nnodes;
  const int64_t S = ceil_div(ntop, ngr);
  const bool early = !(flags & JZ_FLAG_NO_EARLY_EXIT);
  const bool do_sort = !(flags & JZ_FLAG_NO_SEGSORT);
  int32_t *superbeg = nullptr;
  JZ_CUDA(cudaMallocAsync(&superbeg, (S + 1) * sizeof(int32_t), st));
  k_super_beg<<<grid_for(S + 1, 256), 256, 0, st>>>(S, ntop, ngr, superbeg);
  JZ_LAUNCH_CHECK();
  IList il;
  il.nrecv = S;
  il.total = S * S;
  JZ_CUDA(cudaMallocAsync(&il.ispl, (S + 1) * sizeof(int64_t), st));
  JZ_CUDA(cudaMallocAsync(&il.isrc, il.total * sizeof(int32_t), st));
  JZ_CUDA(cudaMallocAsync(&il.rlow, il.total * sizeof(float), st));
  k_dense_init<<<grid_for(S * S + 2, 256), 256, 0, st>>>(S, il.ispl, il.isrc, il.rlow);
  JZ_LAUNCH_CHECK();
  float *rmax2 = nullptr;
  for (int p = top; p >= stop; --p) {
    const int32_t *pbeg = (p == top) ? superbeg : planes[p + 1].beg;
    const int64_t npar = (p == top) ? S : planes[p + 1].nnodes;
    const Plane &pl = planes[p];
    int32_t *cnt = nullptr;
    if (rmax2) JZ_CUDA(cudaFreeAsync(rmax2, st));
    JZ_CUDA(cudaMallocAsync(&rmax2, pl.nnodes * sizeof(float), st));
    JZ_CUDA(cudaMallocAsync(&cnt, pl.nnodes * sizeof(int32_t), st));
    const int srt = do_sort ? 1 : 0;
    const int ee = early ? 1 : 0;
    int32_t *cpar = nullptr;
    const bool flat = JZ_N2N_FLAT && !getenv("JZ_N2N_WARP");
    if (flat) {
      JZ_CUDA(cudaMallocAsync(&cpar, (pl.nnodes > 0 ? pl.nnodes : 1) * sizeof(int32_t), st));
      k_child_parent<<<grid_for(npar, 256), 256, 0, st>>>(pbeg, npar, cpar);
      JZ_LAUNCH_CHECK();
    }
    const unsigned fb = (unsigned)grid_for(pl.nnodes, 256);
    // warp per child while the plane is small enough that a thread per child leaves the chip idle
    // (10^8 C4 plane 1: 1.4e5 children, 7.4 -> 4.7 ms); the 2^30 C5 plane 1 (1.7e6 children) is
    // faster with a thread per child (20.6 vs 32.9 ms)
    const bool wc = JZ_N2N_WC && !getenv("JZ_N2N_THREAD") && pl.nnodes < JZ_N2N_WC_MAX;
    const unsigned wb = (unsigned)grid_for(pl.nnodes, 8, 148 * 64);  // 8 warps per CTA
    if (fixed_r2 >= 0.f) {  // fixed-radius walk (friends-of-friends): every node keeps r^2
      k_fill_f32<<<grid_for(pl.nnodes, 256), 256, 0, st>>>(rmax2, pl.nnodes, fixed_r2);
    } else if (flat) {
      (wc ? k_n2n_wc<RMAX> : k_n2n_flat<RMAX>)<<<wc ? wb : fb, 256, 0, st>>>(cpar, pl.nnodes, pbeg, il.ispl, il.isrc, il.rlow, pl.box, D, k, srt, ee, rmax2,
                                             nullptr, nullptr, nullptr, nullptr, qf[p]);
    } else {
      k_n2n<RMAX><<<(unsigned)ceil_div(npar, kN2NWarps), kN2NWarps * 32, 0, st>>>(pbeg, npar, il.ispl, il.isrc, il.rlow,
                                                                                pl.box, D, k, srt, ee, rmax2, nullptr,
                                                                                nullptr, nullptr, nullptr, qf[p]);
    }
    JZ_LAUNCH_CHECK();
    if (flat)
      (wc ? k_n2n_wc<COUNT> : k_n2n_flat<COUNT>)<<<wc ? wb : fb, 256, 0, st>>>(cpar, pl.nnodes, pbeg, il.ispl, il.isrc, il.rlow, pl.box, D, k, srt, ee,
                                              rmax2, cnt, nullptr, nullptr, nullptr, qf[p]);
    else
      k_n2n<COUNT><<<(unsigned)ceil_div(npar, kN2NWarps), kN2NWarps * 32, 0, st>>>(pbeg, npar, il.ispl, il.isrc, il.rlow, pl.box, D, k, srt, ee,
                                                           rmax2, cnt, nullptr, nullptr, nullptr, qf[p]);
    JZ_LAUNCH_CHECK();
    IList nl;
    nl.nrecv = pl.nnodes;
    JZ_CUDA(cudaMallocAsync(&nl.ispl, (pl.nnodes + 1) * sizeof(int64_t), st));
    exclusive_scan_i32_to_i64(cnt, nl.ispl, pl.nnodes, st);
    nl.total = read_i64(nl.ispl + pl.nnodes, st);
    JZ_CUDA(cudaMallocAsync(&nl.isrc, (nl.total > 0 ? nl.total : 1) * sizeof(int32_t), st));
    JZ_CUDA(cudaMallocAsync(&nl.rlow, (nl.total > 0 ? nl.total : 1) * sizeof(float), st));
    if (flat)
      (wc ? k_n2n_wc<INSERT> : k_n2n_flat<INSERT>)<<<wc ? wb : fb, 256, 0, st>>>(cpar, pl.nnodes, pbeg, il.ispl, il.isrc, il.rlow, pl.box, D, k, srt, ee,
                                               rmax2, nullptr, nl.ispl, nl.isrc, nl.rlow, qf[p]);
    else
      k_n2n<INSERT><<<(unsigned)ceil_div(npar, kN2NWarps), kN2NWarps * 32, 0, st>>>(pbeg, npar, il.ispl, il.isrc, il.rlow, pl.box, D, k, srt, ee,
                                                            rmax2, nullptr, nl.ispl, nl.isrc, nl.rlow, qf[p]);
    JZ_LAUNCH_CHECK();
    if (cpar) JZ_CUDA(cudaFreeAsync(cpar, st));
    if (do_sort) {
      k_segsort<<<grid_for(pl.nnodes, kSegWarps, 148 * 16), kSegWarps * 32, 0, st>>>(nl.ispl, nl.nrecv, nl.isrc,
                                                                                     nl.rlow);
      JZ_LAUNCH_CHECK();
    }
    il.release(st);
    il = nl;
    JZ_CUDA(cudaFreeAsync(cnt, st));
  }
  for (auto *f : qf)
    if (f) JZ_CUDA(cudaFreeAsync(f, st));
  out_il = il;
  *rmax2_out = rmax2;
  if (stop > top) {
    *superbeg_out = superbeg;
  } else {
    JZ_CUDA(cudaFreeAsync(superbeg, st));
    *superbeg_out = nullptr;
  }
}


// ---------------------------------------------------------------- friends-of-friends walk (F4)
// PAPER.md §5 "Implementation" (L477-490): a group pointer per node is carried down the planes.
// ParentToNode: a node whose parent's group is linked points to the first child of that group's
// root, else to itself; a node is (self-)linked if its group is linked or its diagonal
// is <= R_link (d_up(A, A)^2 <= b2). NodeToNode distinguishes three cases:
// (1) same linked group or d_low^2 > b2: discarded; (2) d_up^2 <= b2: the two nodes are linked
// (union of their groups, lower root wins, CAS + retry); (3) otherwise the pair goes to
// the list of the next plane. After the links the pointers are contracted to their roots.
// Bounds are the exact monotone box bounds of jz_common.cuh (R8): d_up^2 <= b2 means every point
// pair of the two nodes has canonical d2 <= b2.
__device__ __forceinline__ int gfind(int32_t *g, int x) {
  while (true) {
    const int p = __ldcg(&g[x]);
    if (p == x) return x;
    const int pp = __ldcg(&g[p]);
    if (pp == p) return p;
    __stcg(&g[x], pp);  // path halving: pp is an ancestor of x (benign race)
    x = pp;
  }
}

__device__ __forceinline__ void gunion(int32_t *g, int a, int b) {
  while (true) {
    a = gfind(g, a);
    b = gfind(g, b);
    if (a == b) return;
    if (a > b) {
      const int t = a;
      a = b;
      b = t;
    }
    const int old = atomicCAS(&g[b], b, a);
    if (old == b) return;
    b = old;
  }
}

// top plane (no linked parent): own pointer, self-linked iff the diagonal is <= R_link
__global__ void k_fof_top(const NodeBox *__restrict__ box, int64_t n, Dom D, float b2, int32_t *__restrict__ g,
                          uint8_t *__restrict__ lk) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const NodeBox b = box[i];
    g[i] = (int32_t)i;
    lk[i] = box_dup2(b, b, D) <= b2;
  }
}

// ParentToNode: children of parent P (plane p+1, child ranges pbeg) on plane p
__global__ void k_fof_p2n(const int32_t *__restrict__ pbeg, int64_t npar, const int32_t *__restrict__ gp,
                          const uint8_t *__restrict__ lkp, const NodeBox *__restrict__ box, Dom D, float b2,
                          int32_t *__restrict__ g, uint8_t *__restrict__ lk) {
  for (int64_t P = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; P < npar; P += (int64_t)gridDim.x * blockDim.x) {
    const bool linked = lkp[P];
    const int first = linked ? pbeg[gp[P]] : 0;  // first child of the root of the parent's group
    for (int c = pbeg[P]; c < pbeg[P + 1]; ++c) {
      const NodeBox b = box[c];
      g[c] = linked ? first : c;
      lk[c] = linked || box_dup2(b, b, D) <= b2;
    }
  }
}

// smallest quarter squared diagonal of the plane's nodes (float bits, atomicMin): a pair (c, s) can
// only be fully linked if d_up(c, s)^2 <= b2, and d_up(c, s) >= max(diag c, diag s) / 2
__global__ void k_fof_mindiag(const NodeBox *__restrict__ box, int64_t n, Dom D, unsigned *__restrict__ out) {
  unsigned m = 0x7f800000u;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const NodeBox b = box[i];
    m = min(m, __float_as_uint(__fmul_rd(box_dup2(b, b, D), 0.25f)));
  }
  m = __reduce_min_sync(0xffffffffu, m);
  if ((threadIdx.x & 31) == 0) atomicMin(out, m);
}

__global__ void k_fof_contract(int32_t *__restrict__ g, int64_t n) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    g[i] = gfind(g, (int)i);
}

enum { FLINK = 0, FCOUNT = 1, FINSERT = 2 };

// one warp per receiving parent J, one lane per child c; source children of every entry of J's list
// staged in shared memory (as k_n2n); MODE FLINK: case (2) links; FCOUNT / FINSERT: case (3) pairs
template <int MODE, bool LINKS>
__global__ void __launch_bounds__(kN2NWarps * 32) k_fof_n2n(const int32_t *__restrict__ pbeg, int64_t npar,
                                                           const int64_t *__restrict__ ispl,
                                                           const int32_t *__restrict__ isrc,
                                                           const NodeBox *__restrict__ cbox, Dom D, float b2,
                                                           int32_t *__restrict__ g, uint8_t *__restrict__ lk,
                                                           int32_t *__restrict__ cnt,
                                                           const int64_t *__restrict__ ispl_out,
                                                           int32_t *__restrict__ isrc_out, float *__restrict__ rlow_out) {
  __shared__ NodeBox s_box[kN2NWarps][kN2NWStage];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t J = (int64_t)blockIdx.x * kN2NWarps + warp;
  if (J >= npar) return;
  NodeBox *sb = s_box[warp];
  const int cb = pbeg[J], ce = pbeg[J + 1];
  const int64_t eb = ispl[J], ee = ispl[J + 1];
  for (int c0 = cb; c0 < ce; c0 += 32) {
    const int c = c0 + lane;
    const bool valid = c < ce;
    NodeBox mb;
    int rc = 0;
    bool lc = false;
    if (valid) {
      mb = cbox[c];
      if (MODE != FLINK) {
        rc = g[c];  // contracted
        lc = lk[c];
      }
    }
    int count = 0;
    int64_t wp = (MODE == FINSERT && valid) ? ispl_out[c] : 0;
    for (int64_t e = eb; e < ee; ++e) {
      const int S = isrc[e];
      const int sb0 = pbeg[S], se = pbeg[S + 1];
      for (int s0 = sb0; s0 < se; s0 += kN2NWStage) {
        const int sn = min(kN2NWStage, se - s0);
        __syncwarp();
        for (int t = lane; t < sn; t += 32) sb[t] = cbox[s0 + t];
        __syncwarp();
        if (valid) {
          for (int t = 0; t < sn; ++t) {
            const int s = s0 + t;
            const NodeBox sbx = sb[t];
            const float dl = box_dlow2(mb, sbx, D);
            if (dl > b2) continue;                                   // case (1): too far
            const bool full = LINKS && box_dup2(mb, sbx, D) <= b2;  // case (2): every pair within R_link
            if (MODE == FLINK) {
              if (full && s != c) {
                gunion(g, c, s);
                lk[c] = 1;
                lk[s] = 1;
              }
            } else {
              if (full) continue;
              if (LINKS && lc && g[s] == rc) continue;  // case (1): same linked group
              if (MODE == FCOUNT) ++count;
              else {
                isrc_out[wp] = s;
                rlow_out[wp] = dl;
                ++wp;
              }
            }
          }
        }
      }
    }
    if (valid && MODE == FCOUNT) cnt[c] = count;
  }
}

// the same three cases with one warp per receiving child and lanes over the children of each
// list entry (as k_n2n_wc): many more threads on the coarse planes; unions are concurrent-safe
// (CAS) and the written lists keep the (entry, child) order
template <int MODE, bool LINKS>
__global__ void __launch_bounds__(256) k_fof_wc(const int32_t *__restrict__ cpar, int64_t nchild,
                                                const int32_t *__restrict__ pbeg, const int64_t *__restrict__ ispl,
                                                const int32_t *__restrict__ isrc, const NodeBox *__restrict__ cbox,
                                                Dom D, float b2, int32_t *__restrict__ g, uint8_t *__restrict__ lk,
                                                int32_t *__restrict__ cnt, const int64_t *__restrict__ ispl_out,
                                                int32_t *__restrict__ isrc_out, float *__restrict__ rlow_out) {
  const int lane = threadIdx.x & 31;
  const int64_t nw = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t c = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); c < nchild; c += nw) {
    const int J = cpar[c];
    const NodeBox mb = cbox[c];
    const int rc = MODE != FLINK ? g[c] : 0;
    const bool lc = MODE != FLINK ? lk[c] != 0 : false;
    int count = 0;
    int64_t wp = MODE == FINSERT ? ispl_out[c] : 0;
    const int64_t eb = ispl[J], ee = ispl[J + 1];
    for (int64_t e = eb; e < ee; ++e) {
      const int S = isrc[e];
      const int s1 = pbeg[S + 1];
      for (int b = pbeg[S]; b < s1; b += 32) {
        const int s = b + lane;
        bool ok = false;
        float dl = 0.f;
        if (s < s1) {
          const NodeBox sbx = cbox[s];
          dl = box_dlow2(mb, sbx, D);
          if (dl <= b2) {                                            // else case (1): too far
            const bool full = LINKS && box_dup2(mb, sbx, D) <= b2;  // case (2): every pair within R_link
            if (MODE == FLINK) {
              if (full && s != (int)c) {
                gunion(g, (int)c, s);
                lk[c] = 1;
                lk[s] = 1;
              }
            } else {
              ok = !full && !(LINKS && lc && g[s] == rc);  // case (1): same linked group
            }
          }
        }
        if (MODE != FLINK) {
          const unsigned bal = __ballot_sync(0xffffffffu, ok);
          if (MODE == FINSERT && ok) {
            const int64_t o = wp + __popc(bal & ((1u << lane) - 1u));
            isrc_out[o] = s;
            rlow_out[o] = dl;
          }
          wp += __popc(bal);
          count += __popc(bal);
        }
      }
    }
    if (MODE == FCOUNT && lane == 0) cnt[c] = count;
  }
}

__global__ void k_fof_point_init(const int32_t *__restrict__ beg, int64_t nleaf, const int32_t *__restrict__ g,
                                 const uint8_t *__restrict__ lk, int32_t *__restrict__ par) {
  for (int64_t l = blockIdx.x; l < nleaf; l += gridDim.x) {
    const bool linked = lk[l];
    const int first = linked ? beg[g[l]] : 0;
    for (int x = beg[l] + threadIdx.x; x < beg[l + 1]; x += blockDim.x) par[x] = linked ? first : x;
  }
}

// the walk of friends-of-friends down to plane 1 (receivers of the leaf stage) with node links;
// writes the point-level union-find initialisation: par[x] = first point of the root leaf of x's
// group when x's leaf is linked (all its points are in that component), else x
void fof_walk(const std::vector<Plane> &planes, const Dom &D, int ngr, float b2, IList &out_il,
              int32_t **superbeg_out, int32_t *par, int64_t npts, cudaStream_t st) {
  const int P = (int)planes.size();
  const int top = P - 1;
  if (P < 2) {  // one plane: the dense super-node list, no node links (par stays the identity)
    float *rmax2 = nullptr;
    walk_to(planes, D, 1, ngr, 0, 1, out_il, &rmax2, superbeg_out, st, b2);
    if (rmax2) JZ_CUDA(cudaFreeAsync(rmax2, st));
    return;
  }
  const int64_t ntop = planes[top].nnodes;
  const int64_t S = ceil_div(ntop, ngr);
  int32_t *superbeg = nullptr;
  JZ_CUDA(cudaMallocAsync(&superbeg, (S + 1) * sizeof(int32_t), st));
  k_super_beg<<<grid_for(S + 1, 256), 256, 0, st>>>(S, ntop, ngr, superbeg);
  JZ_LAUNCH_CHECK();
  IList il;
  il.nrecv = S;
  il.total = S * S;
  JZ_CUDA(cudaMallocAsync(&il.ispl, (S + 1) * sizeof(int64_t), st));
  JZ_CUDA(cudaMallocAsync(&il.isrc, il.total * sizeof(int32_t), st));
  JZ_CUDA(cudaMallocAsync(&il.rlow, il.total * sizeof(float), st));
  k_dense_init<<<grid_for(S * S + 2, 256), 256, 0, st>>>(S, il.ispl, il.isrc, il.rlow);
  JZ_LAUNCH_CHECK();
  int32_t *gp = nullptr;
  uint8_t *lkp = nullptr;
  unsigned *mind = nullptr;
  JZ_CUDA(cudaMallocAsync(&mind, sizeof(unsigned), st));
  for (int p = top; p >= 0; --p) {
    const Plane &pl = planes[p];
    int32_t *g = nullptr;
    uint8_t *lk = nullptr;
    JZ_CUDA(cudaMallocAsync(&g, (pl.nnodes > 0 ? pl.nnodes : 1) * sizeof(int32_t), st));
    JZ_CUDA(cudaMallocAsync(&lk, pl.nnodes > 0 ? pl.nnodes : 1, st));
    if (p == top) {
      k_fof_top<<<grid_for(pl.nnodes, 256), 256, 0, st>>>(pl.box, pl.nnodes, D, b2, g, lk);
    } else {
      k_fof_p2n<<<grid_for(planes[p + 1].nnodes, 256), 256, 0, st>>>(planes[p + 1].beg, planes[p + 1].nnodes, gp, lkp,
                                                                      pl.box, D, b2, g, lk);
    }
    JZ_LAUNCH_CHECK();
    if (gp) JZ_CUDA(cudaFreeAsync(gp, st));
    if (lkp) JZ_CUDA(cudaFreeAsync(lkp, st));
    gp = g;
    lkp = lk;
    if (p == 0) break;  // leaves: pairs are the leaf stage's (plane-1 lists)
    const int32_t *pbeg = (p == top) ? superbeg : planes[p + 1].beg;
    const int64_t npar = (p == top) ? S : planes[p + 1].nnodes;
    const unsigned blocks = (unsigned)ceil_div(npar, kN2NWarps);
    // node links are only possible if some node of the plane is small enough (quarter squared
    // diagonal <= b2); otherwise the plane is walked with the plain fixed-radius test
    JZ_CUDA(cudaMemsetAsync(mind, 0x7f, sizeof(unsigned), st));
    k_fof_mindiag<<<grid_for(pl.nnodes, 256, 148 * 4), 256, 0, st>>>(pl.box, pl.nnodes, D, mind);
    JZ_LAUNCH_CHECK();
    unsigned mh = 0;
    JZ_CUDA(cudaMemcpyAsync(&mh, mind, sizeof(unsigned), cudaMemcpyDeviceToHost, st));
    JZ_CUDA(cudaStreamSynchronize(st));
    float mdq;
    memcpy(&mdq, &mh, 4);
    const bool links = mdq <= b2;
    const bool fwc = JZ_N2N_WC && !getenv("JZ_N2N_THREAD") && pl.nnodes < JZ_N2N_WC_MAX;
    int32_t *cpar = nullptr;
    const unsigned wb = (unsigned)grid_for(pl.nnodes, 8, 148 * 64);
    if (fwc) {
      JZ_CUDA(cudaMallocAsync(&cpar, (pl.nnodes > 0 ? pl.nnodes : 1) * sizeof(int32_t), st));
      k_child_parent<<<grid_for(npar, 256), 256, 0, st>>>(pbeg, npar, cpar);
      JZ_LAUNCH_CHECK();
    }
    if (links && fwc) {
      k_fof_wc<FLINK, true><<<wb, 256, 0, st>>>(cpar, pl.nnodes, pbeg, il.ispl, il.isrc, pl.box, D, b2, g, lk, nullptr,
                                                nullptr, nullptr, nullptr);
      JZ_LAUNCH_CHECK();
      k_fof_contract<<<grid_for(pl.nnodes, 256), 256, 0, st>>>(g, pl.nnodes);
      JZ_LAUNCH_CHECK();
    } else if (links) {
      k_fof_n2n<FLINK, true><<<blocks, kN2NWarps * 32, 0, st>>>(pbeg, npar, il.ispl, il.isrc, pl.box, D, b2, g, lk,
                                                                 nullptr, nullptr, nullptr, nullptr);
      JZ_LAUNCH_CHECK();
      k_fof_contract<<<grid_for(pl.nnodes, 256), 256, 0, st>>>(g, pl.nnodes);
      JZ_LAUNCH_CHECK();
    }
    int32_t *cnt = nullptr;
    JZ_CUDA(cudaMallocAsync(&cnt, pl.nnodes * sizeof(int32_t), st));
    if (fwc && links)
      k_fof_wc<FCOUNT, true><<<wb, 256, 0, st>>>(cpar, pl.nnodes, pbeg, il.ispl, il.isrc, pl.box, D, b2, g, lk, cnt,
                                                 nullptr, nullptr, nullptr);
    else if (fwc)
      k_fof_wc<FCOUNT, false><<<wb, 256, 0, st>>>(cpar, pl.nnodes, pbeg, il.ispl, il.isrc, pl.box, D, b2, g, lk, cnt,
                                                  nullptr, nullptr, nullptr);
    else if (links)
      k_fof_n2n<FCOUNT, true><<<blocks, kN2NWarps * 32, 0, st>>>(pbeg, npar, il.ispl, il.isrc, pl.box, D, b2, g, lk, cnt,
                                                                  nullptr, nullptr, nullptr);
    else
      k_fof_n2n<FCOUNT, false><<<blocks, kN2NWarps * 32, 0, st>>>(pbeg, npar, il.ispl, il.isrc, pl.box, D, b2, g, lk,
                                                                   cnt, nullptr, nullptr, nullptr);
    JZ_LAUNCH_CHECK();
    IList nl;
    nl.nrecv = pl.nnodes;
    JZ_CUDA(cudaMallocAsync(&nl.ispl, (pl.nnodes + 1) * sizeof(int64_t), st));
    exclusive_scan_i32_to_i64(cnt, nl.ispl, pl.nnodes, st);
    nl.total = read_i64(nl.ispl + pl.nnodes, st);
    JZ_CUDA(cudaMallocAsync(&nl.isrc, (nl.total > 0 ? nl.total : 1) * sizeof(int32_t), st));
    JZ_CUDA(cudaMallocAsync(&nl.rlow, (nl.total > 0 ? nl.total : 1) * sizeof(float), st));
    if (fwc && links)
      k_fof_wc<FINSERT, true><<<wb, 256, 0, st>>>(cpar, pl.nnodes, pbeg, il.ispl, il.isrc, pl.box, D, b2, g, lk,
                                                  nullptr, nl.ispl, nl.isrc, nl.rlow);
    else if (fwc)
      k_fof_wc<FINSERT, false><<<wb, 256, 0, st>>>(cpar, pl.nnodes, pbeg, il.ispl, il.isrc, pl.box, D, b2, g, lk,
                                                   nullptr, nl.ispl, nl.isrc, nl.rlow);
    else if (links)
      k_fof_n2n<FINSERT, true><<<blocks, kN2NWarps * 32, 0, st>>>(pbeg, npar, il.ispl, il.isrc, pl.box, D, b2, g, lk,
                                                                   nullptr, nl.ispl, nl.isrc, nl.rlow);
    else
      k_fof_n2n<FINSERT, false><<<blocks, kN2NWarps * 32, 0, st>>>(pbeg, npar, il.ispl, il.isrc, pl.box, D, b2, g, lk,
                                                                    nullptr, nl.ispl, nl.isrc, nl.rlow);
    JZ_LAUNCH_CHECK();
    if (cpar) JZ_CUDA(cudaFreeAsync(cpar, st));
    // segments in (d_low, source) order, as the kNN walk: nearby source nodes first
    k_segsort<<<grid_for(pl.nnodes, kSegWarps, 148 * 16), kSegWarps * 32, 0, st>>>(nl.ispl, nl.nrecv, nl.isrc, nl.rlow);
    JZ_LAUNCH_CHECK();
    il.release(st);
    il = nl;
    JZ_CUDA(cudaFreeAsync(cnt, st));
    if (p == 1) out_il = il;
  }
  // gp / lkp: leaf groups (ParentToNode from plane 1) -> point-level initialisation
  k_fof_point_init<<<grid_for(planes[0].nnodes, 128), 128, 0, st>>>(planes[0].beg, planes[0].nnodes, gp, lkp, par);
  JZ_LAUNCH_CHECK();
  JZ_CUDA(cudaFreeAsync(gp, st));
  JZ_CUDA(cudaFreeAsync(lkp, st));
  JZ_CUDA(cudaFreeAsync(mind, st));
  JZ_CUDA(cudaFreeAsync(superbeg, st));
  *superbeg_out = nullptr;
  (void)npts;
}

}  // namespace jz
