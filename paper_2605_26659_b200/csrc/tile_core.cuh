// tile_core.cuh -- warp-tile building blocks of the FINOM scan kernels.
//
// A tile is a run of <= TILE+1 consecutive elements of the merged order of
// the row mesh R and the column mesh C of one half-iteration (column before
// row on ties).  One WARP owns one tile: no block-level barriers, so the 16
// independent warps an SM holds hide each other's latencies.  Inside a tile
// the reference's two recurrences (_kernels.py:59-88) become scans of
// 2-state affine maps
//     column j: (p, acc) -> (p, acc + c_j)
//     row i:    (p, acc) -> (r_i p + acc, 0)
// composed as (p, acc) -> (A p + B acc + C, D acc + E): sequential per lane
// (EPT elements), shuffle scan across the warp.
#pragma once
#include <cuda_runtime.h>

#include "fexp.cuh"

namespace fb {

#ifndef FB_EPT
#define FB_EPT 8
#endif
constexpr int EPT = FB_EPT;             // merged elements per lane
constexpr int NSLOT = 32 * EPT;         // slots per warp tile
constexpr int TILE = NSLOT - 1;         // merged elements per tile (+1 tie slack)
constexpr int RPT = EPT;                // rows per lane in the epilogue (upper bound)
constexpr int WPC = 4;                  // warps (tiles) per CTA
constexpr int NTHR = 32 * WPC;
constexpr int FAN = 32;                 // resolve-tree fan-out
constexpr int NLEV = 5;                 // tiles + 4 levels (32^4 tiles per problem)
static_assert(EPT <= 32 && 32 % EPT == 0, "walk mask is 32 bits, lane chunks word-aligned");

enum { ST_OK = 0, ST_ZD = 1, ST_NF = 2 };

struct Tf {
  double A, B, C, D, E;
};
__device__ __forceinline__ Tf tf_id() { return Tf{1.0, 0.0, 0.0, 1.0, 0.0}; }

// g o f (f first).  In-tile compositions: products of at most TILE ratios of
// an absorbed kernel stay far inside the double range, so no guards.
__device__ __forceinline__ Tf tf_cat(const Tf &f, const Tf &g) {
  Tf h;
  h.A = g.A * f.A;
  h.B = fma(g.A, f.B, g.B * f.D);
  h.C = fma(g.A, f.C, fma(g.B, f.E, g.C));
  h.D = g.D * f.D;
  h.E = fma(g.D, f.E, g.E);
  return h;
}
__device__ __forceinline__ void tf_apply(const Tf &f, double &p, double &acc) {
  double np = fma(f.A, p, fma(f.B, acc, f.C));
  double na = fma(f.D, acc, f.E);
  p = np;
  acc = na;
}
// Cross-tile compositions: a structurally zero state stays zero even if a
// composite ratio overflowed (hard part 4).
__device__ __forceinline__ double gm(double a, double b) {
  return (a == 0.0 || b == 0.0) ? 0.0 : a * b;
}
__device__ __forceinline__ Tf tf_cat_g(const Tf &f, const Tf &g) {
  Tf h;
  h.A = gm(g.A, f.A);
  h.B = gm(g.A, f.B) + gm(g.B, f.D);
  h.C = (gm(g.A, f.C) + gm(g.B, f.E)) + g.C;
  h.D = gm(g.D, f.D);
  h.E = gm(g.D, f.E) + g.E;
  return h;
}
__device__ __forceinline__ void tf_apply_g(const Tf &f, double &p, double &acc) {
  double np = (gm(f.A, p) + gm(f.B, acc)) + f.C;
  double na = gm(f.D, acc) + f.E;
  p = np;
  acc = na;
}
__device__ __forceinline__ Tf tf_shfl(const Tf &f, int src) {
  return Tf{__shfl_sync(0xffffffffu, f.A, src), __shfl_sync(0xffffffffu, f.B, src),
            __shfl_sync(0xffffffffu, f.C, src), __shfl_sync(0xffffffffu, f.D, src),
            __shfl_sync(0xffffffffu, f.E, src)};
}
__device__ __forceinline__ Tf tf_shfl_up(const Tf &f, int d) {
  return Tf{__shfl_up_sync(0xffffffffu, f.A, d), __shfl_up_sync(0xffffffffu, f.B, d),
            __shfl_up_sync(0xffffffffu, f.C, d), __shfl_up_sync(0xffffffffu, f.D, d),
            __shfl_up_sync(0xffffffffu, f.E, d)};
}
__device__ __forceinline__ Tf tf_shfl_down(const Tf &f, int d) {
  return Tf{__shfl_down_sync(0xffffffffu, f.A, d), __shfl_down_sync(0xffffffffu, f.B, d),
            __shfl_down_sync(0xffffffffu, f.C, d), __shfl_down_sync(0xffffffffu, f.D, d),
            __shfl_down_sync(0xffffffffu, f.E, d)};
}

__device__ __forceinline__ bool tf_finite(const Tf &f) {
  return isfinite(f.A) && isfinite(f.B) && isfinite(f.C) && isfinite(f.D) && isfinite(f.E);
}

// g o f, guarded only if an input is not finite (the guard matters for 0 * inf only).
__device__ __forceinline__ Tf tf_cat_f(const Tf &f, const Tf &g) {
  if (tf_finite(f) && tf_finite(g)) return tf_cat(f, g);
  return tf_cat_g(f, g);
}

// Warp scans of per-lane maps.  Exclusive results: xf = maps of lanes < lane
// (lane 0 first), xb = maps of lanes > lane (lane 31 first); inclusive totals
// returned in all lanes.  G selects the guarded composition; the guarded
// scan first tries the plain one, which agrees with it (up to fma
// contraction) whenever nothing is infinite: the guard only matters for
// 0 * inf, so it is kept for warps whose inputs or results are not finite.
template <bool G>
__device__ __forceinline__ void warp_scan2(const Tf &f, const Tf &b, Tf &xf, Tf &xb, Tf &totf,
                                           Tf &totb) {
  const int lane = threadIdx.x & 31;
  if (G && __all_sync(0xffffffffu, tf_finite(f) && tf_finite(b))) {
    warp_scan2<false>(f, b, xf, xb, totf, totb);
    if (__all_sync(0xffffffffu, tf_finite(xf) && tf_finite(xb) && tf_finite(totf) &&
                                    tf_finite(totb)))
      return;
  }
  Tf incf = f, incb = b;
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    Tf of = tf_shfl_up(incf, off);
    Tf ob = tf_shfl_down(incb, off);
    if (lane >= off) incf = G ? tf_cat_g(of, incf) : tf_cat(of, incf);
    if (lane + off < 32) incb = G ? tf_cat_g(ob, incb) : tf_cat(ob, incb);
  }
  xf = tf_shfl_up(incf, 1);
  xb = tf_shfl_down(incb, 1);
  if (lane == 0) xf = tf_id();
  if (lane == 31) xb = tf_id();
  totf = tf_shfl(incf, 31);
  totb = tf_shfl(incb, 0);
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
  return v;
}
__device__ __forceinline__ double warp_max(double v) {
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, off));
  return v;
}
__device__ __forceinline__ double warp_min(double v) {
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) v = fmin(v, __shfl_xor_sync(0xffffffffu, v, off));
  return v;
}

// Predicated in-place fp64 update (plain selects would cost two 32-bit
// selects per value on top of the arithmetic).
__device__ __forceinline__ void p_fma_mul(bool p, double &c, double &a, double co, double ao) {
  // if p: c = a * co + c; a = a * ao (c first: it uses the old a)
  asm("{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %4, 0;\n\t@q fma.rn.f64 %0, %1, %2, %0;\n\t"
      "@q mul.rn.f64 %1, %1, %3;\n\t}"
      : "+d"(c), "+d"(a) : "d"(co), "d"(ao), "r"((int)p));
}

// Max / min over the warp of non-negative doubles (no NaN): the IEEE bit
// patterns order like the values, so two 32-bit warp reductions suffice.
__device__ __forceinline__ double warp_max_pos(double v) {
  const unsigned hi = (unsigned)__double2hiint(v), lo = (unsigned)__double2loint(v);
  const unsigned mh = __reduce_max_sync(0xffffffffu, hi);
  const unsigned ml = __reduce_max_sync(0xffffffffu, hi == mh ? lo : 0u);
  return __hiloint2double((int)mh, (int)ml);
}
__device__ __forceinline__ double warp_min_pos(double v) {
  const unsigned hi = (unsigned)__double2hiint(v), lo = (unsigned)__double2loint(v);
  const unsigned mh = __reduce_min_sync(0xffffffffu, hi);
  const unsigned ml = __reduce_min_sync(0xffffffffu, hi == mh ? lo : 0xffffffffu);
  return __hiloint2double((int)mh, (int)ml);
}

// Warp sums of four quantities by reduce-scatter in a fixed order: on return
// lane 0 holds the sum of q0, lane 8 of q1, lane 16 of q2, lane 24 of q3
// (lanes 0-7, 8-15, ... hold the same value).
__device__ __forceinline__ double warp_sum4(double q0, double q1, double q2, double q3) {
  const int lane = threadIdx.x & 31;
  const bool b4 = lane & 16, b3 = lane & 8;
  double k0 = b4 ? q2 : q0, k1 = b4 ? q3 : q1;
  const double s0 = b4 ? q0 : q2, s1 = b4 ? q1 : q3;
  k0 = __dadd_rn(k0, __shfl_xor_sync(0xffffffffu, s0, 16));
  k1 = __dadd_rn(k1, __shfl_xor_sync(0xffffffffu, s1, 16));
  double k = b3 ? k1 : k0;
  const double s = b3 ? k0 : k1;
  k = __dadd_rn(k, __shfl_xor_sync(0xffffffffu, s, 8));
#pragma unroll
  for (int off = 4; off > 0; off >>= 1) k = __dadd_rn(k, __shfl_xor_sync(0xffffffffu, k, off));
  return k;
}

// ---------------------------------------------------------------------------
// Wait-free carry resolution tree.  Level 0 nodes are tiles, level L+1 nodes
// group FAN consecutive level-L nodes of one problem; the single level-3
// node is the problem.  A producer warp writes its tile node and arrives;
// the last child to arrive at a node scans the node's children (one warp,
// shuffles), stores each child's exclusive maps within the node, reduces
// the children's partials in a fixed order, and arrives one level up.  The
// warp completing the problem node runs the per-problem epilogue (control
// logic).  A consumer's carry is the composition of <= 3 exclusive maps.
// Timing experiment (FB_DBG_RES builds only): globaltimer stamps of the
// resolve chain for one iteration, max (or min, stored complemented) over
// the warps that reach the point.
#ifdef FB_DBG_RES
__device__ unsigned long long g_phase[16];
__device__ __forceinline__ void res_stamp(int slot, bool is_min) {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  atomicMax(&g_phase[slot], is_min ? ~t : t);
}
#define RES_STAMP(cond, slot, mn) \
  do {                             \
    if (cond) res_stamp(slot, mn); \
  } while (0)
#else
#define RES_STAMP(cond, slot, mn)
#endif
struct Node {
  Tf tf, tb;   // totals over the subtree (forward / backward)
  Tf xf, xb;   // exclusive maps within the parent
  double err, vmax, vmin, fail;  // partial reductions over the subtree
  int cnt, pad;
};
struct Resolve {
  Node *lev[NLEV];
};
struct TreeGeo {  // per problem: node base and count per level
  int base[NLEV], n[NLEV];
};

__device__ __forceinline__ Tf ldcg_tf(const Tf *p) {
  return Tf{__ldcg(&p->A), __ldcg(&p->B), __ldcg(&p->C), __ldcg(&p->D), __ldcg(&p->E)};
}

// Level-0 arrival of tile lt (lane 0 issues the release atomic on the parent
// counter and gets its old value; the caller may do independent work before
// handing it to tree_arrive_from).
__device__ __forceinline__ int tree_arrive_begin(const Resolve &R, const TreeGeo &tg, int lt) {
  int old = 0;
  if ((threadIdx.x & 31) == 0) {
    Node *pn = R.lev[1] + tg.base[1] + lt / FAN;
    asm volatile("atom.add.release.gpu.global.s32 %0, [%1], 1;" : "=r"(old) : "l"(&pn->cnt) : "memory");
  }
  return old;
}

// Continues an arrival whose level-0 atomic returned old0 (lane 0).  Returns
// true in the warp that completed the problem; then `top` holds the
// problem's reduced partials.
// (L0 > 0: continue from level L0, lt then indexes that level's nodes)
__device__ __forceinline__ bool tree_arrive_from(const Resolve &R, const TreeGeo &tg, int lt,
                                                 int old0, double (&top)[4], int L0 = 0) {
  const int lane = threadIdx.x & 31;
  int idx = lt;
#pragma unroll 1
  for (int L = L0; L + 1 < NLEV; ++L) {
    const int parent = idx / FAN;
    const int nchild = min(FAN, tg.n[L] - parent * FAN);
    Node *pn = R.lev[L + 1] + tg.base[L + 1] + parent;
    int last = 0;
    if (lane == 0) {
      int old = old0;
      if (L > 0)
#ifdef FB_ACQREL
        asm volatile("atom.add.acq_rel.gpu.global.s32 %0, [%1], 1;"
                     : "=r"(old) : "l"(&pn->cnt) : "memory");
#else
        asm volatile("atom.add.release.gpu.global.s32 %0, [%1], 1;"
                     : "=r"(old) : "l"(&pn->cnt) : "memory");
#endif
      last = old == nchild - 1;
    }
    last = __shfl_sync(0xffffffffu, last, 0);
    if (!last) return false;
    RES_STAMP(lane == 0 && L < 3 && g_phase[10] != 0 && g_phase[14] == 0, 11 + L, false);
#ifndef FB_ACQREL
    __threadfence();
#endif
    Node *ch = R.lev[L] + tg.base[L] + parent * FAN;
    const bool have = lane < nchild;
    Tf f = tf_id(), b = tf_id();
    double e = 0.0, mx = 0.0, mn = INFINITY, fl = -1.0;
    if (have) {
      f = ldcg_tf(&ch[lane].tf);
      b = ldcg_tf(&ch[lane].tb);
      e = __ldcg(&ch[lane].err);
      mx = __ldcg(&ch[lane].vmax);
      mn = __ldcg(&ch[lane].vmin);
      fl = __ldcg(&ch[lane].fail);
    }
    Tf xf, xb, totf, totb;
    warp_scan2<true>(f, b, xf, xb, totf, totb);
    if (have) {
      ch[lane].xf = xf;
      ch[lane].xb = xb;
    }
    e = warp_sum(e);
    mx = warp_max(mx);
    mn = warp_min(mn);
    fl = warp_max(fl);
    if (lane == 0) {
      pn->tf = totf;
      pn->tb = totb;
      pn->err = e;
      pn->vmax = mx;
      pn->vmin = mn;
      pn->fail = fl;
      pn->cnt = 0;
    }
    top[0] = e;
    top[1] = mx;
    top[2] = mn;
    top[3] = fl;
    idx = parent;
  }
  return true;
}

// Called by a full warp after lane 0 wrote its tile node (maps + partials).
__device__ __forceinline__ bool tree_arrive(const Resolve &R, const TreeGeo &tg, int lt,
                                            double (&top)[4]) {
  return tree_arrive_from(R, tg, lt, tree_arrive_begin(R, tg, lt), top);
}

// Incoming forward state (from the left) and backward state (from the right)
// of tile lt of a problem.
// init (nullable): per problem incoming states (p, acc, q, accb) of the
// problem's first / last tile (a row shard's carries from the other shards).
__device__ __forceinline__ void tree_carry(const Resolve &R, const TreeGeo &tg, int lt, double &p,
                                           double &acc, double &q, double &accb,
                                           const double *init = nullptr, int prob = 0) {
  p = acc = q = accb = 0.0;
  if (init) {
    p = init[4 * prob];
    acc = init[4 * prob + 1];
    q = init[4 * prob + 2];
    accb = init[4 * prob + 3];
  }
  int id[NLEV - 1];
  id[0] = lt;
  for (int L = 1; L < NLEV - 1; ++L) id[L] = id[L - 1] / FAN;
  for (int L = NLEV - 2; L >= 0; --L) {
    const Node &nd = R.lev[L][tg.base[L] + id[L]];
    tf_apply_g(nd.xf, p, acc);
    tf_apply_g(nd.xb, q, accb);
  }
}

// ---------------------------------------------------------------------------
// Shared-memory image of one warp tile.  R* = rows of the half, C* =
// columns (Rc/Ra/Cc/Ca carry one halo element on each side, [-1] and [n]).
// vf/vb hold the walk operand of every merged element in slot order:
// element k of lane l's chunk lives at slot k*32 + l (conflict-free walks).
//   row i:    vf = r_lo into row i,   vb = r_hi out of row i
//   column j: vf = c_lo(j),           vb = c_hi(j)
struct Sm {
  double *Rc, *Ra, *Ro, *Ro2;
  double *Cc, *Ca, *Cv;
  double *vf, *vb;
  int *rslot, *cslot, *cown;
};
// doubles per warp: rows 4.5 nr + 4 (second output incl.), columns 4 nc + 4,
// slots 2 NSLOT; nr + nc <= TILE + 1 = NSLOT
constexpr int WSM = (9 * NSLOT) / 2 + 2 * NSLOT + 16;

__device__ __forceinline__ Sm sm_carve(double *p, int nr, int nc, bool two_out) {
  Sm s;
  s.Rc = p + 1; p += nr + 2;
  s.Ra = p + 1; p += nr + 2;
  s.Ro = p; p += nr;
  s.Ro2 = two_out ? p : s.Ro; p += two_out ? nr : 0;
  s.Cc = p + 1; p += nc + 2;
  s.Ca = p + 1; p += nc + 2;
  s.Cv = p; p += nc;
  s.vf = p; p += NSLOT;
  s.vb = p; p += NSLOT;
  int *q = reinterpret_cast<int *>(p);
  s.rslot = q; q += nr;
  s.cslot = q; q += nc;
  s.cown = q;
  return s;
}

__device__ __forceinline__ void load_tab(double2 *tab) {
  for (int k = threadIdx.x; k < 64; k += blockDim.x)
    tab[k] = make_double2(EXP_TAB_C[k][0], EXP_TAB_C[k][1]);
}

__device__ __forceinline__ void cp_async8(double *dst, const double *src) {
  unsigned sa = (unsigned)__cvta_generic_to_shared(dst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(sa), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.commit_group;\n\tcp.async.wait_group 0;" ::: "memory");
}
// asynchronous dst[-1 .. cnt] <- src[lo-1 .. lo+cnt]; completes at cp_async_wait()
__device__ __forceinline__ void load_halo_async(double *dst, const double *src, int lo, int cnt,
                                                int N, bool zero) {
  const int lane = threadIdx.x & 31;
  if (zero) {
    for (int k = lane - 1; k <= cnt; k += 32) dst[k] = 0.0;
    return;
  }
  for (int k = lane; k < cnt; k += 32) cp_async8(dst + k, src + lo + k);
  if (lane == 0) {
    if (lo > 0) cp_async8(dst - 1, src + lo - 1); else dst[-1] = 0.0;
  }
  if (lane == 1) {
    if (lo + cnt < N) cp_async8(dst + cnt, src + lo + cnt); else dst[cnt] = 0.0;
  }
}

// dst[-1 .. cnt] <- src[lo-1 .. lo+cnt] (halo entries only where they exist)
// (indices outside [w0, N) read as 0: mesh ends, or the edges of a row
// shard's data window)
__device__ __forceinline__ void load_halo(double *dst, const double *src, int lo, int cnt, int N,
                                          bool zero, int w0 = 0) {
  const int lane = threadIdx.x & 31;
  if (zero) {
    for (int k = lane - 1; k <= cnt; k += 32) dst[k] = 0.0;
    return;
  }
  for (int k = lane; k < cnt; k += 32) dst[k] = __ldg(src + lo + k);
  if (lane == 0) dst[-1] = lo > w0 ? __ldg(src + lo - 1) : 0.0;
  if (lane == 1) dst[cnt] = lo + cnt < N ? __ldg(src + lo + cnt) : 0.0;
}

// number of columns among the first `diag` merged elements (column first on ties)
__device__ __forceinline__ int merge_path(int diag, const double *Rc, int nr, const double *Cc,
                                          int nc) {
  int lo = max(0, diag - nr), hi = min(diag, nc);
  while (lo < hi) {
    int mid = (lo + hi + 1) >> 1;
    int i = diag - mid;
    if (i >= nr || Cc[mid - 1] <= Rc[i]) lo = mid; else hi = mid - 1;
  }
  return lo;
}

// Lane chunk: start (ib, jb), end (ie, je), element-type mask (bit set =
// column); writes every element's slot and each column's lower owner.
struct Walk {
  int ib, jb, ie, je, cnt;
  unsigned mask;
};
__device__ __forceinline__ Walk walk0(const Sm &s, int nr, int nc) {
  const int lane = threadIdx.x & 31;
  const int M = nr + nc;
  const int E = (M + 31) / 32;
  Walk w;
  const int pos0 = min(lane * E, M), pos1 = min(pos0 + E, M);
  w.cnt = pos1 - pos0;
  w.jb = merge_path(pos0, s.Rc, nr, s.Cc, nc);
  w.ib = pos0 - w.jb;
  int i = w.ib, j = w.jb;
  unsigned mask = 0;
  for (int k = 0; k < w.cnt; ++k) {
    const int slot = k * 32 + lane;
    bool isc = (j < nc) && (i >= nr || s.Cc[j] <= s.Rc[i]);
    if (isc) {
      mask |= 1u << k;
      s.cown[j] = i;
      s.cslot[j] = slot;
      ++j;
    } else {
      s.rslot[i] = slot;
      ++i;
    }
  }
  w.ie = i;
  w.je = j;
  w.mask = mask;
  return w;
}

// Same chunk from the precomputed merged-order mask of the tile (8 words,
// bit k = 1 iff merged element k is a column): no coordinate comparisons.
__device__ __forceinline__ Walk walk_mask(const Sm &s, const unsigned *mw, int nr, int nc) {
  const int lane = threadIdx.x & 31;
  const int M = nr + nc;
  Walk w;
  const int pos0 = min(lane * EPT, M);
  w.cnt = min(EPT, M - pos0);
  unsigned bits = (__ldg(mw + (lane * EPT) / 32) >> ((lane * EPT) % 32)) & ((1u << EPT) - 1u);
  bits &= w.cnt >= 32 ? 0xffffffffu : ((1u << w.cnt) - 1u);
  const int pc = __popc(bits);
  int incl = pc;
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    int o = __shfl_up_sync(0xffffffffu, incl, off);
    if (lane >= off) incl += o;
  }
  w.jb = incl - pc;
  w.ib = pos0 - w.jb;
  int i = w.ib, j = w.jb;
  for (int k = 0; k < w.cnt; ++k) {
    const int slot = k * 32 + lane;
    if ((bits >> k) & 1u) {
      s.cown[j] = i;
      s.cslot[j] = slot;
      ++j;
    } else {
      s.rslot[i] = slot;
      ++i;
    }
  }
  w.ie = i;
  w.je = j;
  w.mask = bits;
  return w;
}

struct Geo {  // roles of one half within a tile
  int r0, r1, nR, c0, c1, nC;
  double cfirst, clast, rfirst, rlast;
};

// Row ratios (kernel1d.py:127-147) with the structural-zero predicates of
// _kernels.py:64-69 / :81-86 folded in: gap i joins rows i-1 and i;
//   vf[row i]   = r_lo into row i     (0 if no column <= row i-1)
//   vb[row i-1] = r_hi out of row i-1 (0 if no column >  row i)
__device__ __forceinline__ void tile_ratios(const Sm &s, const Geo &g, int nr, bool absorbed,
                                            double eps, double inv, const double2 *tab,
                                            bool dyn = false) {
  const int lane = threadIdx.x & 31;
#pragma unroll 2
  for (int i = lane; i <= nr; i += 32) {
    const int gi = g.r0 + i;
    const bool have = gi > 0 && gi < g.nR;
    const double gap = have ? s.Rc[i] - s.Rc[i - 1] : 0.0;
    const double da = (have && absorbed) ? s.Ra[i] - s.Ra[i - 1] : 0.0;
    const bool pf = have && (i < nr) && (g.cfirst <= s.Rc[i - 1]);
    const bool pb = have && (i > 0) && (g.clast > s.Rc[i]);
    const double ef = ratio_x(dyn, gap, da, true, eps, inv, tab);
    const double eb = absorbed ? ratio_x(dyn, gap, da, false, eps, inv, tab) : ef;
    if (i < nr) s.vf[s.rslot[i]] = pf ? ef : 0.0;
    if (i > 0) s.vb[s.rslot[i - 1]] = pb ? eb : 0.0;
  }
}

// Column contributions c_lo = K'_{o,j} v_j and c_hi = K'_{o-1,j} v_j with
// o = cown[j] (kernel1d.py:148; edge times value as in _kernels.py:283/:288).
// v_j = Cv[j] (times the column coordinate if ymul).
__device__ __forceinline__ void tile_contrib(const Sm &s, const Geo &g, int nc, bool ymul,
                                             double eps, double inv, const double2 *tab,
                                             bool dyn = false) {
  const int lane = threadIdx.x & 31;
#pragma unroll 2
  for (int j = lane; j < nc; j += 32) {
    const double c = s.Cc[j], ca = s.Ca[j];
    double v = s.Cv[j];
    if (ymul) v = c * v;
    const int o = s.cown[j];
    const int og = g.r0 + o;
    // both exponentials unconditionally (independent chains interleave);
    // the halo entries beyond the mesh ends are finite placeholders
    const double elo = edge_x(dyn, s.Rc[o] - c, s.Ra[o], ca, eps, inv, tab);
    const double ehi = edge_x(dyn, c - s.Rc[o - 1], s.Ra[o - 1], ca, eps, inv, tab);
    const int sl = s.cslot[j];
    s.vf[sl] = og < g.nR ? elo * v : 0.0;
    s.vb[sl] = og > 0 ? ehi * v : 0.0;
  }
}

// Local maps of the lane's chunk, branch-free over the element types.
__device__ __forceinline__ void walk_maps(const Sm &s, const Walk &w, Tf &f, Tf &b) {
  const int lane = threadIdx.x & 31;
  f = tf_id();
  for (int k = 0; k < w.cnt; ++k) {
    const double v = s.vf[k * 32 + lane];
    const bool col = (w.mask >> k) & 1u;
    const double nA = v * f.A, nB = fma(v, f.B, f.D), nC = fma(v, f.C, f.E), nE = f.E + v;
    f.A = col ? f.A : nA;
    f.B = col ? f.B : nB;
    f.C = col ? f.C : nC;
    f.D = col ? f.D : 0.0;
    f.E = col ? nE : 0.0;
  }
  b = tf_id();
  for (int k = w.cnt - 1; k >= 0; --k) {
    const double v = s.vb[k * 32 + lane];
    const bool col = (w.mask >> k) & 1u;
    const double nA = v * b.A, nB = fma(v, b.B, b.D), nC = fma(v, b.C, b.E), nE = b.E + v;
    b.A = col ? b.A : nA;
    b.B = col ? b.B : nB;
    b.C = col ? b.C : nC;
    b.D = col ? b.D : 0.0;
    b.E = col ? nE : 0.0;
  }
}

// Final recurrences with the true incoming states (reference operation
// order: p = (r * p) + acc, _kernels.py:65-67; out = p + q, :87).
__device__ __forceinline__ void walk_apply(const Sm &s, const Walk &w, double p, double acc,
                                           double q, double accb, bool sum) {
  const int lane = threadIdx.x & 31;
  int i = w.ib;
  for (int k = 0; k < w.cnt; ++k) {
    const double v = s.vf[k * 32 + lane];
    const bool col = (w.mask >> k) & 1u;
    const double np = __dadd_rn(v == 0.0 ? 0.0 : __dmul_rn(v, p), acc);
    const double na = __dadd_rn(acc, v);
    if (!col) s.Ro[i] = np;
    p = col ? p : np;
    acc = col ? na : 0.0;
    i += col ? 0 : 1;
  }
  i = w.ie;
  for (int k = w.cnt - 1; k >= 0; --k) {
    const double v = s.vb[k * 32 + lane];
    const bool col = (w.mask >> k) & 1u;
    const double nq = __dadd_rn(v == 0.0 ? 0.0 : __dmul_rn(v, q), accb);
    const double na = __dadd_rn(accb, v);
    i -= col ? 0 : 1;
    if (!col) {
      if (sum) s.Ro[i] = __dadd_rn(s.Ro[i], nq); else s.Ro2[i] = nq;
    }
    q = col ? q : nq;
    accb = col ? na : 0.0;
  }
}

// Local maps -> the lane's incoming states given the tile's incoming states.
__device__ __forceinline__ void tile_states(const Sm &s, const Walk &w, double &p, double &acc,
                                            double &q, double &accb) {
  Tf f, b, xf, xb, tf_, tb_;
  walk_maps(s, w, f, b);
  warp_scan2<false>(f, b, xf, xb, tf_, tb_);
  tf_apply(xf, p, acc);
  tf_apply(xb, q, accb);
}

// One contribution to the next-half tile maps (both directions), for one
// next-half column (a row of the current half) with coordinate c, shift ca,
// value v.  Next-half rows are the current columns: coords Nc, shifts Na, nn
// of them, global range [c0, c1) of nNR; halos at [-1] and [nn].
//   fwd: columns before the last next row add K'_{last,i} v (-> fC), the
//        others K'_{c1,i} v (-> fE, owner = first next row after the tile);
//   bwd: columns after the first next row add K'_{first,i} v (-> bC), the
//        others K'_{c0-1,i} v (-> bE).
__device__ __forceinline__ void next_contrib2(const double *Nc, const double *Na, int nn, int c0,
                                              int c1, int nNR, double c, double ca, double v,
                                              double eps, double inv, const double2 *tab,
                                              double &fC, double &fE, double &bC, double &bE,
                                              bool dyn = false) {
  const bool fin = nn > 0 && c <= Nc[nn - 1];  // before the last next row
  const bool bin = nn > 0 && c > Nc[0];        // after the first next row
  const int fk = fin ? nn - 1 : nn, bk = bin ? 0 : -1;
  const double ef = edge_x(dyn, Nc[fk] - c, Na[fk], ca, eps, inv, tab) * v;
  const double eb = edge_x(dyn, c - Nc[bk], Na[bk], ca, eps, inv, tab) * v;
  if (fin) fC += ef;
  else if (c1 < nNR) fE += ef;
  if (bin) bC += eb;
  else if (c0 > 0) bE += eb;
}

// Composite coefficients of the next-half maps (each the product the
// reference's per-row ratios telescope to, kernel1d.py:133/:140), one
// exponential per lane 0..3, gathered in every lane.
//   fwd: A = ratio (c0-1 -> c1-1) [0 if structurally zero], B = (c0 -> c1-1)
//   bwd: A = ratio (c1 -> c0)     [0 if structurally zero], B = (c1-1 -> c0)
__device__ __forceinline__ void next_maps(const double *Nc, const double *Na, int nn, int c0,
                                          int c1, int nNR, double kfirst, double klast, double fC,
                                          double fE, double bC, double bE, double eps, double inv,
                                          const double2 *tab, Tf &mf, Tf &mb, bool dyn = false) {
  const int lane = threadIdx.x & 31;
  if (nn == 0) {
    mf = Tf{1.0, 0.0, 0.0, 1.0, fE};
    mb = Tf{1.0, 0.0, 0.0, 1.0, bE};
    return;
  }
  // lane 0: fB (c0 -> c1-1), 1: fA (c0-1 -> c1-1), 2: bB (c1-1 -> c0), 3: bA (c1 -> c0)
  const int hi = (lane == 3) ? nn : nn - 1;
  const int lo = (lane == 1) ? -1 : 0;
  const bool use = lane < 4 && (lane == 0 || lane == 2 || (lane == 1 && c0 > 0 && kfirst <= Nc[-1]) ||
                                (lane == 3 && c1 < nNR && klast > Nc[nn]));
  double e = 0.0;
  if (use) e = ratio_x(dyn, Nc[hi] - Nc[lo], Na[hi] - Na[lo], lane < 2, eps, inv, tab);
  const double fB = __shfl_sync(0xffffffffu, e, 0), fA = __shfl_sync(0xffffffffu, e, 1);
  const double bB = __shfl_sync(0xffffffffu, e, 2), bA = __shfl_sync(0xffffffffu, e, 3);
  mf = Tf{fA, fB, fC, 0.0, fE};
  mb = Tf{bA, bB, bC, 0.0, bE};
}

}  // namespace fb
