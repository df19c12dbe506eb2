/*
 * ORACLE — test infrastructure only.  Never linked into, loaded by, or
 * called from the product path (paper_2507_01110_b200/).  Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference
 * leg may use it, and only as the checker / CPU baseline.
 *
 * Plain-C restatement of the reference's LoD selection for the per-view hot
 * path, evaluated in IEEE fp64 with the exact operation order numpy and
 * OpenBLAS use on the reference's CPU path (pinned against
 * golden vectors generated from the reference in tests/golden/):
 *
 *   np.linalg.norm(v)          1-D  -> BLAS ddot:  sqrt(fma(z,z,fma(y,y,x*x)))
 *   np.linalg.norm(v, axis=1)  2-D  -> add.reduce: sqrt((x*x+y*y)+z*z)
 *   c @ P[:, :3].T + P[:, 3]   n>=2 -> dgemm:      fma(c2,p2,fma(c1,p1,c0*p0)) + d
 *                              n==1 -> dgemv:      fma(c2,p2,fma(c0,p0,c1*p1)) + d
 *
 * Functions (reference file:line, /root/reference/pkg/src/glod/):
 *   oracle_bfs_cut   hierarchy.py:244-266 (bfs_cut)
 *   oracle_cut_spt   spt.py:67-75         (cut_spt)
 *   oracle_cut_hspt  hspt.py:104-158      (cut_hspt)
 *
 * Build: oracle/Makefile (gcc -O2 -ffp-contract=off; fma() from libm).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define NONE (-1)

static double norm_ddot(double x, double y, double z) { return sqrt(fma(z, z, fma(y, y, x * x))); }
static double norm_rows(double x, double y, double z) { return sqrt((x * x + y * y) + z * z); }

static double npmax3(double a, double b, double c) {
  /* np.max along an axis propagates NaN */
  if (a != a || b != b || c != c) return NAN;
  double m = a;
  if (b > m) m = b;
  if (c > m) m = c;
  return m;
}

/* core.py:356-361 */
static double min_distance(double T, int metric, const double* s) {
  if (metric == 0) return T / npmax3(s[0], s[1], s[2]);
  return T / sqrt(s[0] * s[1] + s[0] * s[2] + s[1] * s[2]);
}

/* core.py:364-372 with hspt.py:125 radius = 3 * max(scale) */
static int sphere_in(const double* P, const double* c, double r, int64_t frontier_n) {
  for (int k = 0; k < 6; ++k) {
    const double* p = P + 4 * k;
    double s = frontier_n == 1 ? fma(c[2], p[2], fma(c[0], p[0], c[1] * p[1]))
                               : fma(c[2], p[2], fma(c[1], p[1], c[0] * p[0]));
    s = s + p[3];
    if (!(s <= r)) return 0;
  }
  return 1;
}

static int cmp_i64(const void* a, const void* b) {
  int64_t x = *(const int64_t*)a, y = *(const int64_t*)b;
  return (x > y) - (x < y);
}

typedef struct { int64_t* v; int64_t n, cap; } vec;
static void push(vec* a, int64_t x) {
  if (a->n == a->cap) {
    a->cap = a->cap ? 2 * a->cap : 64;
    a->v = (int64_t*)realloc(a->v, sizeof(int64_t) * a->cap);
  }
  a->v[a->n++] = x;
}

/* hierarchy.py:244-266.  Appends the (unsorted) cut to *sel. */
static void bfs_cut_into(const int32_t* children, const double* means, const double* scales,
                         int64_t start, const double* pos, const double* planes, double T,
                         int metric, vec* sel) {
  vec cur = {0}, nxt = {0};
  push(&cur, start);
  while (cur.n) {
    int64_t n = cur.n;
    nxt.n = 0;
    for (int64_t i = 0; i < n; ++i) {
      int64_t v = cur.v[i];
      const double* m = means + 3 * v;
      const double* s = scales + 3 * v;
      if (planes && !sphere_in(planes, m, 3.0 * npmax3(s[0], s[1], s[2]), n)) continue;
      double dist = norm_rows(m[0] - pos[0], m[1] - pos[1], m[2] - pos[2]);
      double md = min_distance(T, metric, s);
      int leaf = children[2 * v] == NONE;
      if (dist >= md || leaf) {
        push(sel, v);
      } else {
        push(&nxt, children[2 * v]);
        push(&nxt, children[2 * v + 1]);
      }
    }
    vec t = cur; cur = nxt; nxt = t;
  }
  free(cur.v);
  free(nxt.v);
}

int64_t oracle_bfs_cut(const int32_t* children, const double* means, const double* scales,
                       int64_t start, const double* pos, const double* planes, double T,
                       int metric, int64_t* out) {
  vec sel = {0};
  bfs_cut_into(children, means, scales, start, pos, planes, T, metric, &sel);
  qsort(sel.v, sel.n, sizeof(int64_t), cmp_i64);
  if (sel.n) memcpy(out, sel.v, sizeof(int64_t) * sel.n);
  int64_t n = sel.n;
  free(sel.v);
  return n;
}

/* spt.py:67-75.  Returns the number of selected nodes written to out. */
int64_t oracle_cut_spt(const double* key_self, const double* key_parent, const int64_t* nodes,
                       int64_t count, int64_t root, double d, int64_t* prefix_len,
                       int64_t* out) {
  /* n = searchsorted(-key_parent, -d, 'left'): first i with -kp[i] >= -d */
  int64_t lo = 0, hi = count;
  while (lo < hi) {
    int64_t mid = (lo + hi) / 2;
    if (-key_parent[mid] < -d) lo = mid + 1; else hi = mid;
  }
  *prefix_len = lo;
  int64_t root_rec = 0;
  for (int64_t i = 0; i < count; ++i)
    if (nodes[i] == root) { root_rec = i; break; }
  if (d >= key_self[root_rec]) {
    out[0] = root;
    return 1;
  }
  int64_t k = 0;
  for (int64_t i = 0; i < lo; ++i)
    if (key_self[i] <= d) out[k++] = nodes[i];
  return k;
}

/*
 * hspt.py:104-158.  kind[node] = spt_id (>=0) of an SPT root, -2 for a
 * passthrough root, -1 otherwise.  SPT tables are per spt_id.
 * Outputs: upper/pass (sorted), per selected SPT in ascending root order:
 * spt_id, d_root, prefix_len, count; and the concatenated selections.
 * counts_out = {n_upper, n_pass, n_spt, n_sel}.
 */
int oracle_cut_hspt(int64_t cap, int64_t root, const int32_t* children, const int32_t* kind,
                    const double* means, const double* scales, const int64_t* spt_offset,
                    const int64_t* spt_count, const int64_t* spt_root, const double* spt_center,
                    const double* key_self, const double* key_parent, const int64_t* rec_node,
                    const double* pos, const double* planes, double T, int metric,
                    int64_t* upper_out, int64_t* pass_out, int64_t* spt_id_out,
                    double* d_root_out, int64_t* prefix_out, int64_t* sel_count_out,
                    int64_t* sel_out, int64_t* counts_out) {
  (void)cap;
  vec upper = {0}, pass = {0}, spts = {0}, cur = {0}, nxt = {0};
  push(&cur, root);
  while (cur.n) {
    int64_t n = cur.n;
    nxt.n = 0;
    for (int64_t i = 0; i < n; ++i) {
      int64_t v = cur.v[i];
      const double* m = means + 3 * v;
      const double* s = scales + 3 * v;
      if (planes && !sphere_in(planes, m, 3.0 * npmax3(s[0], s[1], s[2]), n)) continue;
      int32_t k = kind[v];
      if (k >= 0) { push(&spts, v); continue; }
      if (k == -2) {
        bfs_cut_into(children, means, scales, v, pos, planes, T, metric, &pass);
        continue;
      }
      double dist = norm_rows(m[0] - pos[0], m[1] - pos[1], m[2] - pos[2]);
      double md = min_distance(T, metric, s);
      int leaf = children[2 * v] == NONE;
      if (dist >= md || leaf) {
        push(&upper, v);
      } else {
        push(&nxt, children[2 * v]);
        push(&nxt, children[2 * v + 1]);
      }
    }
    vec t = cur; cur = nxt; nxt = t;
  }
  qsort(upper.v, upper.n, sizeof(int64_t), cmp_i64);
  qsort(pass.v, pass.n, sizeof(int64_t), cmp_i64);
  qsort(spts.v, spts.n, sizeof(int64_t), cmp_i64);  /* sorted(selected_spts) by root id */
  if (upper.n) memcpy(upper_out, upper.v, 8 * upper.n);
  if (pass.n) memcpy(pass_out, pass.v, 8 * pass.n);
  int64_t nsel = 0;
  for (int64_t j = 0; j < spts.n; ++j) {
    int32_t sid = kind[spts.v[j]];
    const double* c = spt_center + 3 * sid;
    double d = norm_ddot(c[0] - pos[0], c[1] - pos[1], c[2] - pos[2]);
    int64_t off = spt_offset[sid], pl = 0;
    int64_t got = oracle_cut_spt(key_self + off, key_parent + off, rec_node + off,
                                 spt_count[sid], spt_root[sid], d, &pl, sel_out + nsel);
    spt_id_out[j] = sid;
    d_root_out[j] = d;
    prefix_out[j] = pl;
    sel_count_out[j] = got;
    nsel += got;
  }
  counts_out[0] = upper.n;
  counts_out[1] = pass.n;
  counts_out[2] = spts.n;
  counts_out[3] = nsel;
  free(upper.v); free(pass.v); free(spts.v); free(cur.v); free(nxt.v);
  return 0;
}
