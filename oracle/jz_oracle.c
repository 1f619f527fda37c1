/*
 * jz_oracle.c -- CPU ORACLE for exact k-nearest-neighbour search (TEST INFRASTRUCTURE).
 *
 * This file is test infrastructure. Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load it. It shares no
 * code, header, table or constant generator with the CUDA path in
 * paper_2604_05885_b200/ (DESIGN.md "Oracle").
 *
 * What it computes ("guarantee that all candidate neighbours
 * required for an exact k-nearest neighbour search are considered", L432/L453
 * self-query "query points equal to the source points", L454 periodic wrapping;
 * SURVEY.md §8(c) "Definition of record"):
 *
 *   for every point i, the k smallest pairs (d2(p_i, p_j), j) over all
 *   j in [0, N) -- j = i included -- in lexicographic order, where
 *     t_d  = RN(q_d - s_d)                                  (FP32 subtraction)
 *     if periodic: t_d >= L_d/2 -> t_d = RN(t_d - L_d);
 *                  t_d < -L_d/2 -> t_d = RN(t_d + L_d)      (minimal image, [-L/2, L/2))
 *     d2  = fmaf(t_z, t_z, fmaf(t_y, t_y, t_x * t_x))       (FP32, no FTZ/DAZ)
 *   (readings R1-R3: FP32 canonical formula, ties -> lower index,
 *    self included.)
 *
 * Two implementations of the same definition:
 *   oracle_knn_brute : the definition written out, O(N^2), j scanned ascending.
 *   oracle_knn_grid  : uniform-grid shell search with a conservative stop rule;
 *                      returns the same bits (pinned against brute in tests).
 * Both may run a subset of query rows (rows != NULL) for sampled checks.
 *
 * Separate query points ("query the tree using a set of query points
 * x_query distinct from the source points x"): the *_q entry
 * points take a query array; row r is then the k smallest (d2(x_query[i], x_j), j)
 * over the sources j, i = rows ? rows[r] : r. Any k <= N works (PAPER.md L386:
 * k > k_max is the kernel's business, not the definition's).
 *
 * Build: gcc -O2 -fopenmp -ffp-contract=off -fPIC -shared (no -ffast-math).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#if defined(__FAST_MATH__)
#error "oracle must not be built with -ffast-math"
#endif

typedef struct {
  int periodic;
  float L[3];
  float h[3]; /* 0.5 * L, exact */
} domain_t;

/* One coordinate difference, wrapped to the minimal image when periodic. */
static inline float wrap_diff(float q, float s, const domain_t *dom, int d) {
  float t = q - s; /* RN, FP32 (x86-64 SSE: no excess precision) */
  if (dom->periodic) {
    if (t >= dom->h[d])
      t = t - dom->L[d];
    else if (t < -dom->h[d])
      t = t + dom->L[d];
  }
  return t;
}

/* Canonical squared distance (one FMUL, then two FMA). */
static inline float canon_d2(const float *q, const float *s, const domain_t *dom) {
  float tx = wrap_diff(q[0], s[0], dom, 0);
  float ty = wrap_diff(q[1], s[1], dom, 1);
  float tz = wrap_diff(q[2], s[2], dom, 2);
  return fmaf(tz, tz, fmaf(ty, ty, tx * tx));
}

/* (d2, j) lexicographic "less than" */
static inline int pair_less(float da, int32_t ja, float db, int32_t jb) {
  return da < db || (da == db && ja < jb);
}

/* Sorted top-k list; insert (d, j) if it beats the current k-th entry. */
typedef struct {
  int k, cnt;
  float *d;
  int32_t *j;
} topk_t;

static inline void topk_insert(topk_t *t, float d, int32_t j) {
  int pos;
  if (t->cnt == t->k) {
    if (!pair_less(d, j, t->d[t->k - 1], t->j[t->k - 1])) return;
    pos = t->k - 1;
  } else {
    pos = t->cnt++;
  }
  while (pos > 0 && pair_less(d, j, t->d[pos - 1], t->j[pos - 1])) {
    t->d[pos] = t->d[pos - 1];
    t->j[pos] = t->j[pos - 1];
    --pos;
  }
  t->d[pos] = d;
  t->j[pos] = j;
}

static void make_domain(domain_t *dom, const float *box) {
  memset(dom, 0, sizeof(*dom));
  if (box) {
    dom->periodic = 1;
    for (int d = 0; d < 3; ++d) {
      dom->L[d] = box[d];
      dom->h[d] = 0.5f * box[d];
    }
  }
}

static void set_threads(int nthreads) {
#ifdef _OPENMP
  if (nthreads > 0) omp_set_num_threads(nthreads);
#else
  (void)nthreads;
#endif
}

int oracle_max_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}

/*
 * Brute force: rows r in [0, nrows) query point q = rows ? rows[r] : r.
 * out_idx/out_d2 are [nrows][k] row-major. Returns 0, or 2 on bad args.
 */
int oracle_knn_brute_q(const float *pos, int64_t n, const float *qry, const float *box, int k,
                       const int64_t *rows, int64_t nrows, int32_t *out_idx, float *out_d2, int nthreads) {
  if (n < 1 || k < 1 || k > n || !qry) return 2;
  domain_t dom;
  make_domain(&dom, box);
  set_threads(nthreads);
#pragma omp parallel for schedule(dynamic, 64)
  for (int64_t r = 0; r < nrows; ++r) {
    int64_t i = rows ? rows[r] : r;
    const float *q = qry + 3 * i;
    topk_t t = {k, 0, out_d2 + r * k, out_idx + r * k};
    for (int64_t j = 0; j < n; ++j) {
      float d2 = canon_d2(q, pos + 3 * j, &dom);
      /* j ascending: strict "<" against the k-th keeps lower indices on ties */
      if (t.cnt < k || d2 < t.d[k - 1]) topk_insert(&t, d2, (int32_t)j);
    }
  }
  return 0;
}

/* Self-query: the query points are the sources. */
int oracle_knn_brute(const float *pos, int64_t n, const float *box, int k, const int64_t *rows,
                     int64_t nrows, int32_t *out_idx, float *out_d2, int nthreads) {
  return oracle_knn_brute_q(pos, n, pos, box, k, rows, nrows, out_idx, out_d2, nthreads);
}

/* ------------------------------------------------------------------------- */
/* Uniform grid                                                               */
/* ------------------------------------------------------------------------- */

typedef struct {
  int G[3];
  double lo[3], w[3]; /* cell d spans [lo + c*w, lo + (c+1)*w) */
  int64_t *start;     /* [ncell+1] */
  int32_t *order;     /* point ids sorted by cell (stable: ascending id within a cell) */
} grid_t;

static inline int cell_coord(const grid_t *g, float x, int d) {
  double c = floor(((double)x - g->lo[d]) / g->w[d]);
  if (c < 0) c = 0;
  if (c > g->G[d] - 1) c = g->G[d] - 1;
  return (int)c;
}

static int grid_build(grid_t *g, const float *pos, int64_t n, const domain_t *dom, double per_cell) {
  double lo[3], hi[3];
  if (dom->periodic) {
    for (int d = 0; d < 3; ++d) {
      lo[d] = 0.0;
      hi[d] = dom->L[d];
    }
  } else {
    for (int d = 0; d < 3; ++d) {
      lo[d] = INFINITY;
      hi[d] = -INFINITY;
    }
    for (int64_t i = 0; i < n; ++i)
      for (int d = 0; d < 3; ++d) {
        double v = pos[3 * i + d];
        if (v < lo[d]) lo[d] = v;
        if (v > hi[d]) hi[d] = v;
      }
  }
  double vol = 1.0;
  for (int d = 0; d < 3; ++d) vol *= fmax(hi[d] - lo[d], 1e-30);
  double w = cbrt(vol * per_cell / (double)n);
  int64_t ncell = 1;
  for (int d = 0; d < 3; ++d) {
    double span = hi[d] - lo[d];
    int G = (int)floor(span / w);
    if (G < 1) G = 1;
    if (G > 2048) G = 2048;
    g->G[d] = G;
    g->lo[d] = lo[d];
    /* open: widen the last cell slightly so max coordinates fall inside */
    g->w[d] = span > 0 ? span / G : 1.0;
    ncell *= G;
  }
  g->start = (int64_t *)calloc((size_t)ncell + 1, sizeof(int64_t));
  g->order = (int32_t *)malloc((size_t)n * sizeof(int32_t));
  int32_t *cell = (int32_t *)malloc((size_t)n * sizeof(int32_t));
  if (!g->start || !g->order || !cell) {
    free(cell);
    return 7;
  }
  for (int64_t i = 0; i < n; ++i) {
    const float *p = pos + 3 * i;
    int cx = cell_coord(g, p[0], 0), cy = cell_coord(g, p[1], 1), cz = cell_coord(g, p[2], 2);
    int64_t c = ((int64_t)cx * g->G[1] + cy) * g->G[2] + cz;
    cell[i] = (int32_t)c;
    g->start[c + 1]++;
  }
  for (int64_t c = 0; c < ncell; ++c) g->start[c + 1] += g->start[c];
  int64_t *fill = (int64_t *)malloc((size_t)ncell * sizeof(int64_t));
  memcpy(fill, g->start, (size_t)ncell * sizeof(int64_t));
  for (int64_t i = 0; i < n; ++i) g->order[fill[cell[i]]++] = (int32_t)i;
  free(fill);
  free(cell);
  return 0;
}

static void grid_free(grid_t *g) {
  free(g->start);
  free(g->order);
}

static inline void scan_cell(const grid_t *g, const float *pos, const float *q, const domain_t *dom,
                             int64_t c, topk_t *t) {
  for (int64_t a = g->start[c]; a < g->start[c + 1]; ++a) {
    int32_t j = g->order[a];
    float d2 = canon_d2(q, pos + 3 * (int64_t)j, dom);
    if (t->cnt < t->k || pair_less(d2, j, t->d[t->k - 1], t->j[t->k - 1])) topk_insert(t, d2, j);
  }
}

/*
 * Grid shell search. After finishing Chebyshev shell s around the query's cell
 * the visited region is the cube of cells [c-s, c+s]^3 (wrapped when periodic).
 * r_s = distance (float64) from q to the outside of that cube, minus a slack
 * of 1e-12 * extent, minus (periodic only) the wrap slack sqrt(3) * 2^-24 * L_max.
 * Stop once cnt == k and d2_k < r_s^2 (1 - 1e-6). Why that is safe: an unvisited
 * point s has an exact minimal-image displacement t_e with |t_e| >= r_s (before
 * the slacks). The canonical per-axis value is RN(q_d - s_d), wrapped by an exact
 * +-L_d (R1, "periodic wrapping in the distance
 * calculation"):
 *   - no wrap: |RN(q-s)| >= |q-s| (1 - 2^-24)          (relative error only);
 *   - wrap:    RN(q-s) +- L differs from q-s +- L by |RN(q-s) - (q-s)|
 *              <= ulp(|q-s|)/2 <= 2^-24 L_d               (ABSOLUTE error: the
 *              rounding happens before the wrap, so it is not relative to |t|).
 * Hence |t_canon| >= |t_e| (1 - 2^-24) - sqrt(3) 2^-24 L_max, and the FP32 sum of
 * squares loses at most another 3 * 2^-24 relative: canonical d2 >=
 * (r_s - sqrt(3) 2^-24 L_max)^2 (1 - 6 * 2^-24) > d2_k, so no unvisited point can
 * enter the list (not even on a tie). Also stop once every cell has been visited.
 * (Round-1 bug: without the absolute wrap slack, cells < ~0.06 L could stop early
 * on a wrapped pair; tests/test_oracle_knn.py::test_grid_periodic_wrap_slack.)
 */
static void grid_query(const grid_t *g, const float *pos, const float *q, const domain_t *dom, topk_t *t) {
  int c[3];
  for (int d = 0; d < 3; ++d) c[d] = cell_coord(g, q[d], d);
  int smax = 0;
  for (int d = 0; d < 3; ++d) {
    int need = dom->periodic ? (g->G[d] / 2 + 1) : (g->G[d]);
    if (need > smax) smax = need;
  }
  double ext = fmax(fmax(g->w[0] * g->G[0], g->w[1] * g->G[1]), g->w[2] * g->G[2]);
  double lmax = fmax(fmax((double)dom->L[0], (double)dom->L[1]), (double)dom->L[2]);
  for (int s = 0; s <= smax; ++s) {
    /* visit the cells with Chebyshev distance exactly s (deduplicated when wrapped) */
    int lo[3], hi[3];
    for (int d = 0; d < 3; ++d) {
      lo[d] = c[d] - s;
      hi[d] = c[d] + s;
      if (dom->periodic) {
        if (2 * s + 1 >= g->G[d]) { /* whole axis covered: visit each index once */
          lo[d] = c[d] - (g->G[d] - 1) / 2;
          hi[d] = lo[d] + g->G[d] - 1;
        }
      } else {
        if (lo[d] < 0) lo[d] = 0;
        if (hi[d] > g->G[d] - 1) hi[d] = g->G[d] - 1;
      }
    }
    for (int x = lo[0]; x <= hi[0]; ++x)
      for (int y = lo[1]; y <= hi[1]; ++y)
        for (int z = lo[2]; z <= hi[2]; ++z) {
          int dx = abs(x - c[0]), dy = abs(y - c[1]), dz = abs(z - c[2]);
          int cheb = dx > dy ? dx : dy;
          if (dz > cheb) cheb = dz;
          /* shell membership; with a clipped / folded axis a cell whose clipped
           * coordinate distance is < s on all axes was visited in an earlier shell */
          if (cheb != s) continue;
          int cx = x, cy = y, cz = z;
          if (dom->periodic) {
            cx = ((x % g->G[0]) + g->G[0]) % g->G[0];
            cy = ((y % g->G[1]) + g->G[1]) % g->G[1];
            cz = ((z % g->G[2]) + g->G[2]) % g->G[2];
          }
          int64_t cell = ((int64_t)cx * g->G[1] + cy) * g->G[2] + cz;
          scan_cell(g, pos, q, dom, cell, t);
        }
    /* stop rule */
    double rs = INFINITY;
    int all_covered = 1;
    for (int d = 0; d < 3; ++d) {
      int covered = dom->periodic ? (2 * s + 1 >= g->G[d]) : (c[d] - s <= 0 && c[d] + s >= g->G[d] - 1);
      if (covered) continue;
      all_covered = 0;
      double face_lo = g->lo[d] + (double)(c[d] - s) * g->w[d];
      double face_hi = g->lo[d] + (double)(c[d] + s + 1) * g->w[d];
      double dist = fmin((double)q[d] - face_lo, face_hi - (double)q[d]);
      if (!dom->periodic) {
        /* a clipped side has no points beyond it */
        if (c[d] - s <= 0) dist = face_hi - (double)q[d];
        if (c[d] + s >= g->G[d] - 1) dist = (double)q[d] - face_lo;
      }
      if (dist < rs) rs = dist;
    }
    if (all_covered) break;
    rs -= 1e-12 * ext;
    if (dom->periodic) rs -= 1.7320508075688772 * 0x1p-24 * lmax;
    if (t->cnt == t->k && rs > 0 && (double)t->d[t->k - 1] < rs * rs * (1.0 - 1e-6)) break;
  }
}

int oracle_knn_grid_q(const float *pos, int64_t n, const float *qry, const float *box, int k, const int64_t *rows,
                      int64_t nrows, int32_t *out_idx, float *out_d2, int nthreads, double per_cell) {
  if (n < 1 || k < 1 || k > n || !qry) return 2;
  domain_t dom;
  make_domain(&dom, box);
  set_threads(nthreads);
  grid_t g;
  memset(&g, 0, sizeof(g));
  int rc = grid_build(&g, pos, n, &dom, per_cell > 0 ? per_cell : 2.0);
  if (rc) {
    grid_free(&g);
    return rc;
  }
#pragma omp parallel for schedule(dynamic, 256)
  for (int64_t r = 0; r < nrows; ++r) {
    int64_t i = rows ? rows[r] : r;
    topk_t t = {k, 0, out_d2 + r * k, out_idx + r * k};
    grid_query(&g, pos, qry + 3 * i, &dom, &t);
  }
  grid_free(&g);
  return 0;
}

int oracle_knn_grid(const float *pos, int64_t n, const float *box, int k, const int64_t *rows, int64_t nrows,
                    int32_t *out_idx, float *out_d2, int nthreads, double per_cell) {
  return oracle_knn_grid_q(pos, n, pos, box, k, rows, nrows, out_idx, out_d2, nthreads, per_cell);
}

/* Canonical d2 of explicit pairs (for invariant tests: symmetry, stored-d2 recomputation). */
void oracle_pair_d2(const float *a, const float *b, int64_t m, const float *box, float *out) {
  domain_t dom;
  make_domain(&dom, box);
  for (int64_t i = 0; i < m; ++i) out[i] = canon_d2(a + 3 * i, b + 3 * i, &dom);
}

/* ------------------------------------------------------------------------- */
/* Friends-of-friends (§5)              */
/* ------------------------------------------------------------------------- */
/*
 * Groups are the connected components of the graph with an edge between i != j
 * iff the canonical FP32 d2(p_i, p_j) (above) is <= b2, b2 = RN32(r_link * r_link)
 * (R21). label[i] = the smallest index of i's component: the union-find
 * below always links the larger root under the smaller one ("update the
 * higher index root to point towards the lower index root"), so every root is its
 * component's minimum.
 *   oracle_fof_brute : every pair i < j, O(N^2).
 *   oracle_fof_grid  : cells of width >= 1.0001 r_link (+ 2 * 2^-24 L_max when
 *                      periodic), pairs in the 27 neighbouring cells (a linked pair
 *                      is closer than one cell width on every axis); same labels
 *                      (pinned against brute in tests).
 * Why the periodic term: a linked pair has canonical |t_d| <= sqrt(b2)(1 + 2^-23),
 * but a wrapped t_d = RN(q-s) +- L carries an absolute error up to 2^-24 L_d
 * (the rounding precedes the exact wrap, see grid_query), so the exact
 * per-axis separation can exceed r_link by that much.
 */
static int32_t uf_find(int32_t *par, int32_t x) {
  while (par[x] != x) {
    par[x] = par[par[x]];
    x = par[x];
  }
  return x;
}

static void uf_union(int32_t *par, int32_t a, int32_t b) {
  a = uf_find(par, a);
  b = uf_find(par, b);
  if (a == b) return;
  if (a < b)
    par[b] = a;
  else
    par[a] = b;
}

static void uf_labels(int32_t *par, int64_t n) {
  for (int64_t i = 0; i < n; ++i) par[i] = uf_find(par, (int32_t)i);
}

int oracle_fof_brute(const float *pos, int64_t n, const float *box, float b2, int32_t *label) {
  domain_t dom;
  make_domain(&dom, box);
  for (int64_t i = 0; i < n; ++i) label[i] = (int32_t)i;
  for (int64_t i = 0; i < n; ++i)
    for (int64_t j = i + 1; j < n; ++j)
      if (canon_d2(pos + 3 * i, pos + 3 * j, &dom) <= b2) uf_union(label, (int32_t)i, (int32_t)j);
  uf_labels(label, n);
  return 0;
}

int oracle_fof_grid(const float *pos, int64_t n, const float *box, float b2, int32_t *label) {
  domain_t dom;
  make_domain(&dom, box);
  double w = sqrt((double)b2) * 1.0001;
  if (dom.periodic) w += 2.0 * 0x1p-24 * fmax(fmax((double)dom.L[0], (double)dom.L[1]), (double)dom.L[2]);
  double lo[3], span[3];
  for (int d = 0; d < 3; ++d) {
    lo[d] = dom.periodic ? 0.0 : INFINITY;
    span[d] = dom.periodic ? dom.L[d] : -INFINITY;
  }
  if (!dom.periodic) {
    double hi[3] = {-INFINITY, -INFINITY, -INFINITY};
    for (int64_t i = 0; i < n; ++i)
      for (int d = 0; d < 3; ++d) {
        if (pos[3 * i + d] < lo[d]) lo[d] = pos[3 * i + d];
        if (pos[3 * i + d] > hi[d]) hi[d] = pos[3 * i + d];
      }
    for (int d = 0; d < 3; ++d) span[d] = hi[d] - lo[d];
  }
  int G[3];
  int64_t ncell = 1;
  for (int d = 0; d < 3; ++d) {
    double g = floor(span[d] / w);
    if (g < 1) g = 1;
    if (g > 1024) g = 1024; /* coarser cells stay correct (width only grows) */
    G[d] = (int)g;
    ncell *= G[d];
    if (dom.periodic && G[d] < 3) return oracle_fof_brute(pos, n, box, b2, label);
  }
  grid_t g;
  g.start = (int64_t *)calloc((size_t)ncell + 1, sizeof(int64_t));
  g.order = (int32_t *)malloc((size_t)(n > 0 ? n : 1) * sizeof(int32_t));
  int32_t *cell = (int32_t *)malloc((size_t)(n > 0 ? n : 1) * sizeof(int32_t));
  int64_t *fill = (int64_t *)malloc((size_t)ncell * sizeof(int64_t));
  if (!g.start || !g.order || !cell || !fill) {
    free(g.start);
    free(g.order);
    free(cell);
    free(fill);
    return 7;
  }
  for (int d = 0; d < 3; ++d) {
    g.G[d] = G[d];
    g.lo[d] = lo[d];
    g.w[d] = span[d] > 0 ? span[d] / G[d] : 1.0;
  }
  for (int64_t i = 0; i < n; ++i) {
    const float *p = pos + 3 * i;
    int64_t c = ((int64_t)cell_coord(&g, p[0], 0) * G[1] + cell_coord(&g, p[1], 1)) * G[2] + cell_coord(&g, p[2], 2);
    cell[i] = (int32_t)c;
    g.start[c + 1]++;
  }
  for (int64_t c = 0; c < ncell; ++c) g.start[c + 1] += g.start[c];
  memcpy(fill, g.start, (size_t)ncell * sizeof(int64_t));
  for (int64_t i = 0; i < n; ++i) g.order[fill[cell[i]]++] = (int32_t)i;
  for (int64_t i = 0; i < n; ++i) label[i] = (int32_t)i;
  for (int64_t i = 0; i < n; ++i) {
    const float *p = pos + 3 * i;
    const int c0[3] = {cell_coord(&g, p[0], 0), cell_coord(&g, p[1], 1), cell_coord(&g, p[2], 2)};
    for (int dx = -1; dx <= 1; ++dx)
      for (int dy = -1; dy <= 1; ++dy)
        for (int dz = -1; dz <= 1; ++dz) {
          int cc[3] = {c0[0] + dx, c0[1] + dy, c0[2] + dz};
          int skip = 0;
          for (int d = 0; d < 3; ++d) {
            if (cc[d] < 0 || cc[d] >= G[d]) {
              if (dom.periodic)
                cc[d] = (cc[d] + G[d]) % G[d];
              else
                skip = 1;
            }
          }
          if (skip) continue;
          const int64_t c = ((int64_t)cc[0] * G[1] + cc[1]) * G[2] + cc[2];
          for (int64_t a = g.start[c]; a < g.start[c + 1]; ++a) {
            const int32_t j = g.order[a];
            if (j > i && canon_d2(p, pos + 3 * (int64_t)j, &dom) <= b2) uf_union(label, (int32_t)i, j);
          }
        }
  }
  uf_labels(label, n);
  free(cell);
  free(fill);
  grid_free(&g);
  return 0;
}
