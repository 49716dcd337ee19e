// tile_core.cuh -- per-tile building blocks of the FINOM scan kernels.
//
// A tile is a run of <= TILE+1 consecutive elements of the merged order of
// the row mesh R and the column mesh C of one half-iteration (column before
// row on ties).  Inside a tile the reference's two recurrences
// (_kernels.py:59-88) become scans of 2-state affine maps
//     column j: (p, acc) -> (p, acc + c_j)
//     row i:    (p, acc) -> (r_i p + acc, 0)
// composed as (p, acc) -> (A p + B acc + C, D acc + E).
#pragma once
#include <cuda_runtime.h>

#include "fexp.cuh"

namespace fb {

constexpr int TILE = 2048;  // merged elements per tile (+1 tie slack)
constexpr int NT = 256;     // threads per tile CTA
constexpr int NW = NT / 32;
constexpr int EMAX = (TILE + 1 + NT - 1) / NT;  // merged elements per thread
constexpr int RPT = EMAX;                       // epilogue rows per thread (upper bound)
static_assert(EMAX <= 32, "walk mask is 32 bits");

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
// Cross-tile compositions (look-back): a structurally zero state stays zero
// even if a composite ratio overflowed (hard part 4).
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

// Scan scratch: warp totals and warp-exclusive maps for both directions.
struct ScanSm {
  Tf wf[NW], wb[NW];   // inclusive warp totals
  Tf pf[NW], pb[NW];   // warp-exclusive maps (fwd: from tile start; bwd: from tile end)
  Tf totf, totb;       // tile totals
};

// Exclusive per-thread maps in both directions plus the tile totals.
//   xf: T_{k-1} o ... o T_0 restricted to this warp (apply after ss.pf[warp])
//   xb: T_{k+1} o ... o T_31 restricted to this warp (apply after ss.pb[warp])
__device__ __forceinline__ void block_scan2(const Tf &f, const Tf &b, Tf &xf, Tf &xb,
                                            ScanSm &ss) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  Tf incf = f, incb = b;
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    Tf of = tf_shfl_up(incf, off);
    Tf ob = tf_shfl_down(incb, off);
    if (lane >= off) incf = tf_cat(of, incf);
    if (lane + off < 32) incb = tf_cat(ob, incb);
  }
  xf = tf_shfl_up(incf, 1);
  xb = tf_shfl_down(incb, 1);
  if (lane == 0) xf = tf_id();
  if (lane == 31) xb = tf_id();
  if (lane == 31) ss.wf[warp] = incf;
  if (lane == 0) ss.wb[warp] = incb;
  __syncthreads();
  if (threadIdx.x == 0) {
    Tf acc = tf_id();
    for (int w = 0; w < NW; ++w) {
      ss.pf[w] = acc;
      acc = tf_cat(acc, ss.wf[w]);
    }
    ss.totf = acc;
  } else if (threadIdx.x == 32) {
    Tf acc = tf_id();
    for (int w = NW - 1; w >= 0; --w) {
      ss.pb[w] = acc;
      acc = tf_cat(acc, ss.wb[w]);
    }
    ss.totb = acc;
  }
  __syncthreads();
}

// Fixed-order block reduction of up to 8 values per thread (ops: 0 sum,
// 1 max, 2 min).  Deterministic for a fixed NT.  Result valid in thread 0.
template <int K>
__device__ __forceinline__ void block_reduce(double (&v)[K], const int (&op)[K], double *red) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int k = 0; k < K; ++k) {
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
      double o = __shfl_xor_sync(0xffffffffu, v[k], off);
      v[k] = op[k] == 0 ? v[k] + o : (op[k] == 1 ? fmax(v[k], o) : fmin(v[k], o));
    }
    if (lane == 0) red[warp * K + k] = v[k];
  }
  __syncthreads();
  if (threadIdx.x == 0) {
#pragma unroll
    for (int k = 0; k < K; ++k) {
      double s = red[k];
      for (int w = 1; w < NW; ++w) {
        double o = red[w * K + k];
        s = op[k] == 0 ? s + o : (op[k] == 1 ? fmax(s, o) : fmin(s, o));
      }
      v[k] = s;
    }
  }
  __syncthreads();
}

// ---------------------------------------------------------------------------
// Wait-free carry resolution.  Producers (the previous half's epilogue, the
// absorb and precompute kernels) publish per-tile maps for both scan
// directions.  The last CTA to finish a group of GROUP consecutive tiles
// scans the group (one warp, shuffles) into in-group exclusive maps; the
// last group of a problem scans the group totals into group incoming
// states.  A consumer's carry is then O(1): one map applied to one state.
constexpr int GROUP = 32;

struct TileMaps {  // produced per tile
  Tf f, b;
};
struct ResTile {   // in-group exclusive maps (fwd: from group start, bwd: from group end)
  Tf f, b;
};
struct ResGroup {  // group totals, then group incoming states
  Tf tf, tb;
  double pf, af, pb, ab;
};
struct Resolve {
  TileMaps *maps;
  ResTile *tile;
  ResGroup *group;
  int *gcnt;  // per group arrival counter
  int *pcnt;  // per problem group-arrival counter
};

__device__ __forceinline__ Tf ldcg_tf(const Tf *p) {
  return Tf{__ldcg(&p->A), __ldcg(&p->B), __ldcg(&p->C), __ldcg(&p->D), __ldcg(&p->E)};
}

// Warp-wide exclusive scans of n <= 32 maps per chunk, sequential over chunks.
// in(k) gives the maps of element k; out(k, xf, xb) receives the exclusive
// maps; returns the totals.  Forward: element 0 first.  Backward: element n-1
// first.  All 32 lanes must call.
template <class In, class Out>
__device__ __forceinline__ void warp_scan_maps(int n, In in, Out out, Tf &totf, Tf &totb) {
  const int lane = threadIdx.x & 31;
  Tf cf = tf_id(), cb = tf_id();  // carried totals of processed chunks
  const int nch = (n + 31) / 32;
  // forward: chunks in order
  for (int c = 0; c < nch; ++c) {
    int k = c * 32 + lane;
    Tf f = tf_id(), bb;
    if (k < n) in(k, f, bb);
    Tf inc = f;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      Tf o = tf_shfl_up(inc, off);
      if (lane >= off) inc = tf_cat_g(o, inc);
    }
    Tf ex = tf_shfl_up(inc, 1);
    if (lane == 0) ex = tf_id();
    Tf xf = tf_cat_g(cf, ex);  // carried chunks first
    if (k < n) out(k, xf, true);
    Tf last;
    last.A = __shfl_sync(0xffffffffu, inc.A, 31);
    last.B = __shfl_sync(0xffffffffu, inc.B, 31);
    last.C = __shfl_sync(0xffffffffu, inc.C, 31);
    last.D = __shfl_sync(0xffffffffu, inc.D, 31);
    last.E = __shfl_sync(0xffffffffu, inc.E, 31);
    cf = tf_cat_g(cf, last);
  }
  // backward: chunks in reverse order, lanes reversed
  for (int c = nch - 1; c >= 0; --c) {
    int k = c * 32 + lane;
    Tf ff, b = tf_id();
    if (k < n) in(k, ff, b);
    Tf inc = b;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      Tf o = tf_shfl_down(inc, off);
      if (lane + off < 32) inc = tf_cat_g(o, inc);
    }
    Tf ex = tf_shfl_down(inc, 1);
    if (lane == 31) ex = tf_id();
    Tf xb = tf_cat_g(cb, ex);
    if (k < n) out(k, xb, false);
    Tf first;
    first.A = __shfl_sync(0xffffffffu, inc.A, 0);
    first.B = __shfl_sync(0xffffffffu, inc.B, 0);
    first.C = __shfl_sync(0xffffffffu, inc.C, 0);
    first.D = __shfl_sync(0xffffffffu, inc.D, 0);
    first.E = __shfl_sync(0xffffffffu, inc.E, 0);
    cb = tf_cat_g(cb, first);
  }
  totf = cf;
  totb = cb;
}

// Called by warp 0 of a producer CTA after thread 0 wrote R.maps[t] (and
// fenced).  t: global tile; tile0/ntiles: the problem's tiles; grp0: the
// problem's first group; prob: problem index.
__device__ __forceinline__ void resolve_arrive(const Resolve &R, int t, int tile0, int ntiles,
                                               int grp0, int prob) {
  const int lane = threadIdx.x & 31;
  const int lt = t - tile0, gl = lt / GROUP, g = grp0 + gl;
  const int gt0 = tile0 + gl * GROUP, gn = min(GROUP, ntiles - gl * GROUP);
  const int ngroups = (ntiles + GROUP - 1) / GROUP;
  int last = 0;
  if (lane == 0) {
    __threadfence();
    last = atomicAdd(R.gcnt + g, 1) == gn - 1;
  }
  last = __shfl_sync(0xffffffffu, last, 0);
  if (!last) return;
  __threadfence();
  Tf totf, totb;
  warp_scan_maps(
      gn,
      [&](int k, Tf &f, Tf &b) {
        f = ldcg_tf(&R.maps[gt0 + k].f);
        b = ldcg_tf(&R.maps[gt0 + k].b);
      },
      [&](int k, const Tf &x, bool fwd) {
        if (fwd) R.tile[gt0 + k].f = x; else R.tile[gt0 + k].b = x;
      },
      totf, totb);
  if (lane == 0) {
    R.group[g].tf = totf;
    R.group[g].tb = totb;
    R.gcnt[g] = 0;
    __threadfence();
    last = atomicAdd(R.pcnt + prob, 1) == ngroups - 1;
  }
  last = __shfl_sync(0xffffffffu, last, 0);
  if (!last) return;
  __threadfence();
  Tf pf, pb;
  warp_scan_maps(
      ngroups,
      [&](int k, Tf &f, Tf &b) {
        f = ldcg_tf(&R.group[grp0 + k].tf);
        b = ldcg_tf(&R.group[grp0 + k].tb);
      },
      [&](int k, const Tf &x, bool fwd) {
        double p = 0.0, a = 0.0;
        tf_apply_g(x, p, a);  // incoming state of group k from the problem boundary
        if (fwd) {
          R.group[grp0 + k].pf = p;
          R.group[grp0 + k].af = a;
        } else {
          R.group[grp0 + k].pb = p;
          R.group[grp0 + k].ab = a;
        }
      },
      pf, pb);
  if (lane == 0) R.pcnt[prob] = 0;
}

// Carry of tile t (incoming forward state from the left, backward from the right).
__device__ __forceinline__ void resolve_carry(const Resolve &R, int t, int tile0, int grp0,
                                              double &p, double &acc, double &q, double &accb) {
  const int g = grp0 + (t - tile0) / GROUP;
  const ResGroup &G = R.group[g];
  p = G.pf;
  acc = G.af;
  q = G.pb;
  accb = G.ab;
  tf_apply_g(R.tile[t].f, p, acc);
  tf_apply_g(R.tile[t].b, q, accb);
}

// ---------------------------------------------------------------------------
// Shared-memory tile image.  R* = rows of the half, C* = columns (Rc/Ra/Cc/Ca
// carry one halo element on each side, [-1] and [n]).  vf/vb hold the walk
// operand of every merged element in "slot" order: element k of thread t's
// chunk lives at slot k*NT + t, so the walks read conflict-free.
//   row i:    vf = r_lo into row i,   vb = r_hi out of row i
//   column j: vf = c_lo(j),           vb = c_hi(j)
struct Sm {
  double *Rc, *Ra, *Ro, *Ro2;
  double *Cc, *Ca;
  double *vf, *vb;
  int *rslot, *cslot, *cown;
};
// slots run up to EMAX*NT (chunks are E = ceil(M/NT) long, the last ones short)
constexpr int NSLOT = EMAX * NT;
// doubles: rows 3.5 nr + 4 (+ nr with a second output), columns 3 nc + 4,
// merged 2 NSLOT; nr + nc <= cap
__host__ __device__ constexpr int sm_doubles(int cap) { return (9 * cap) / 2 + 2 * NSLOT + 16; }

__device__ __forceinline__ Sm sm_carve(double *p, int nr, int nc, bool two_out) {
  Sm s;
  s.Rc = p + 1; p += nr + 2;
  s.Ra = p + 1; p += nr + 2;
  s.Ro = p; p += nr;
  s.Ro2 = two_out ? p : s.Ro; p += two_out ? nr : 0;
  s.Cc = p + 1; p += nc + 2;
  s.Ca = p + 1; p += nc + 2;
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

// dst[-1 .. cnt] <- src[lo-1 .. lo+cnt] (halo entries only where they exist)
__device__ __forceinline__ void load_halo(double *dst, const double *src, int lo, int cnt, int N,
                                          bool zero) {
  if (zero) {
    for (int k = threadIdx.x - 1; k <= cnt; k += blockDim.x) dst[k] = 0.0;
    return;
  }
  for (int k = threadIdx.x; k < cnt; k += blockDim.x) dst[k] = __ldg(src + lo + k);
  if (threadIdx.x == 0) {
    dst[-1] = lo > 0 ? __ldg(src + lo - 1) : 0.0;
    dst[cnt] = lo + cnt < N ? __ldg(src + lo + cnt) : 0.0;
  }
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

// Per-thread merged chunk: start (ib, jb), end (ie, je), element-type mask
// (bit set = column); writes every element's slot and each column's lower
// owner (first row >= column).
struct Walk {
  int ib, jb, ie, je, cnt;
  unsigned mask;
};
__device__ __forceinline__ Walk walk0(const Sm &s, int nr, int nc) {
  const int M = nr + nc;
  const int E = (M + NT - 1) / NT;
  Walk w;
  const int pos0 = min((int)threadIdx.x * E, M), pos1 = min(pos0 + E, M);
  w.cnt = pos1 - pos0;
  w.jb = merge_path(pos0, s.Rc, nr, s.Cc, nc);
  w.ib = pos0 - w.jb;
  int i = w.ib, j = w.jb;
  unsigned mask = 0;
  for (int k = 0; k < w.cnt; ++k) {
    const int slot = k * NT + threadIdx.x;
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

struct Geo {  // roles of one half within a tile
  int r0, r1, nR, c0, c1, nC;
  double cfirst, clast, rfirst, rlast;
};

// Row ratios (kernel1d.py:127-147) with the structural-zero predicates of
// _kernels.py:64-69 / :81-86 folded in: gap i joins rows i-1 and i;
//   vf[row i]   = r_lo into row i     (0 if no column <= row i-1)
//   vb[row i-1] = r_hi out of row i-1 (0 if no column >  row i)
__device__ __forceinline__ void tile_ratios(const Sm &s, const Geo &g, int nr, bool absorbed,
                                            double eps, double inv, const double2 *tab) {
  for (int i = threadIdx.x; i <= nr; i += NT) {
    int gi = g.r0 + i;
    double f = 0.0, b = 0.0;
    if (gi > 0 && gi < g.nR) {
      double gap = s.Rc[i] - s.Rc[i - 1];
      bool pf = (i < nr) && (g.cfirst <= s.Rc[i - 1]);
      bool pb = (i > 0) && (g.clast > s.Rc[i]);
      if (absorbed) {
        double da = s.Ra[i] - s.Ra[i - 1];
        if (pf) f = ratio_exp(gap, da, true, eps, inv, tab);
        if (pb) b = ratio_exp(gap, da, false, eps, inv, tab);
      } else if (pf || pb) {
        double e = ratio_exp(gap, 0.0, true, eps, inv, tab);
        f = pf ? e : 0.0;
        b = pb ? e : 0.0;
      }
    }
    if (i < nr) s.vf[s.rslot[i]] = f;
    if (i > 0) s.vb[s.rslot[i - 1]] = b;
  }
}

// Column contributions c_lo = K'_{o,j} v_j and c_hi = K'_{o-1,j} v_j with
// o = cown[j] (kernel1d.py:148; edge times value as in _kernels.py:283/:288).
// v_j = vin[c0 + j] (times the column coordinate if ymul).
__device__ __forceinline__ void tile_contrib(const Sm &s, const Geo &g, int nc, const double *vin,
                                             bool one, bool ymul, double eps, double inv,
                                             const double2 *tab) {
  for (int j = threadIdx.x; j < nc; j += NT) {
    double c = s.Cc[j], ca = s.Ca[j];
    double v = one ? 1.0 : vin[g.c0 + j];
    if (ymul) v = c * v;
    int o = s.cown[j];
    int og = g.r0 + o;
    double lo = 0.0, hi = 0.0;
    if (og < g.nR) lo = edge_exp(s.Rc[o] - c, s.Ra[o], ca, eps, inv, tab) * v;
    if (og > 0) hi = edge_exp(c - s.Rc[o - 1], s.Ra[o - 1], ca, eps, inv, tab) * v;
    const int sl = s.cslot[j];
    s.vf[sl] = lo;
    s.vb[sl] = hi;
  }
}

// Local maps of the thread's chunk, branch-free over the element types.
__device__ __forceinline__ void walk_maps(const Sm &s, const Walk &w, Tf &f, Tf &b) {
  f = tf_id();
  for (int k = 0; k < w.cnt; ++k) {
    const double v = s.vf[k * NT + threadIdx.x];
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
    const double v = s.vb[k * NT + threadIdx.x];
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
  int i = w.ib;
  for (int k = 0; k < w.cnt; ++k) {
    const double v = s.vf[k * NT + threadIdx.x];
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
    const double v = s.vb[k * NT + threadIdx.x];
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

// One contribution to a next-half tile map (fwd or bwd), for one next-half
// column (a row of the current half) with coordinate c, shift ca, value v.
// Next-half rows are the current columns: coords Nc, shifts Na, nn of them,
// global range [c0, c1) of nNR; halos at [-1] and [nn].
//   fwd: columns before the last next row add K'_{last,i} v (-> C), the
//        others K'_{c1,i} v (-> E, owner = first next row after the tile);
//   bwd: columns after the first next row add K'_{first,i} v (-> C), the
//        others K'_{c0-1,i} v (-> E).
template <bool FWD>
__device__ __forceinline__ void next_contrib(const double *Nc, const double *Na, int nn, int c0,
                                             int c1, int nNR, double c, double ca, double v,
                                             double eps, double inv, const double2 *tab,
                                             double &C, double &E) {
  if (FWD) {
    if (nn > 0 && c <= Nc[nn - 1])
      C += edge_exp(Nc[nn - 1] - c, Na[nn - 1], ca, eps, inv, tab) * v;
    else if (c1 < nNR)
      E += edge_exp(Nc[nn] - c, Na[nn], ca, eps, inv, tab) * v;
  } else {
    if (nn > 0 && c > Nc[0])
      C += edge_exp(c - Nc[0], Na[0], ca, eps, inv, tab) * v;
    else if (c0 > 0)
      E += edge_exp(c - Nc[-1], Na[-1], ca, eps, inv, tab) * v;
  }
}

// Both directions' contributions of one next-half column.
__device__ __forceinline__ void next_contrib2(const double *Nc, const double *Na, int nn, int c0,
                                              int c1, int nNR, double c, double ca, double v,
                                              double eps, double inv, const double2 *tab,
                                              double &fC, double &fE, double &bC, double &bE) {
  next_contrib<true>(Nc, Na, nn, c0, c1, nNR, c, ca, v, eps, inv, tab, fC, fE);
  next_contrib<false>(Nc, Na, nn, c0, c1, nNR, c, ca, v, eps, inv, tab, bC, bE);
}

// Composite coefficients of the next-half map (each the product the
// reference's per-row ratios telescope to, kernel1d.py:133/:140).
//   fwd: A = ratio (c0-1 -> c1-1) [0 if structurally zero], B = (c0 -> c1-1)
//   bwd: A = ratio (c1 -> c0)     [0 if structurally zero], B = (c1-1 -> c0)
template <bool FWD>
__device__ __forceinline__ Tf next_map(const double *Nc, const double *Na, int nn, int c0, int c1,
                                       int nNR, double kfirst, double klast, double C, double E,
                                       double eps, double inv, const double2 *tab) {
  if (nn == 0) return Tf{1.0, 0.0, 0.0, 1.0, E};
  Tf t;
  t.C = C;
  t.D = 0.0;
  t.E = E;
  if (FWD) {
    t.B = ratio_exp(Nc[nn - 1] - Nc[0], Na[nn - 1] - Na[0], true, eps, inv, tab);
    t.A = (c0 > 0 && kfirst <= Nc[-1])
              ? ratio_exp(Nc[nn - 1] - Nc[-1], Na[nn - 1] - Na[-1], true, eps, inv, tab)
              : 0.0;
  } else {
    t.B = ratio_exp(Nc[nn - 1] - Nc[0], Na[nn - 1] - Na[0], false, eps, inv, tab);
    t.A = (c1 < nNR && klast > Nc[nn])
              ? ratio_exp(Nc[nn] - Nc[0], Na[nn] - Na[0], false, eps, inv, tab)
              : 0.0;
  }
  return t;
}

}  // namespace fb
