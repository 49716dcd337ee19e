// solve_group.cuh -- the whole 1D solve loop of a batch in ONE persistent
// kernel, a group of warps per problem (included by finom_1d.cu).
//
// Batches of independent problems (config 5: 8192 x 16384) need no
// communication between problems, so a problem's every iteration can run
// inside one group of g warps of one CTA (g = 1 for large batches):
//   * the carries of a half come from the tile maps the previous half's
//     epilogue wrote (tile_compute), composed by the group itself (lane
//     chunks, warp scan, the group's other warps through shared memory) into
//     per-tile incoming states -- no resolve tree, no k_resolve launch;
//   * the partials (marginal error, extremes, failure) are reduced in tile
//     order as the warp walks its tiles, then across the group's warps in
//     warp order (deterministic), and run_driver's bookkeeping
//     (solver.py:173-198) runs in registers of every warp of the group;
//   * an absorption (solver._shift + kernel1d.absorb) rebuilds the group's
//     tile records in place (absorb_core) -- no k_absorb launch;
//   * problems are taken from a queue (one atomic per problem), so a batch of
//     equal problems keeps every SM busy until the tail.
// The per-tile work (bulk-copied record, one-state walk, epilogue) is the
// k_step code; only the carry source and the bookkeeping differ.
#pragma once

namespace fb {

#ifndef FB_GW
#define FB_GW 16
#endif
constexpr int GW = FB_GW;               // warps per CTA
constexpr int GTHR = 32 * GW;
// The next half's tile maps of a warp's first STASH tiles stay in shared
// memory after the loop's working area (the carries then need no global
// round trip: the node loads took 5.4 of a half's 11 us of carries at config 5,
// their lines long evicted from L2); absorb_core's larger area overlaps the
// stash, so a rebuild invalidates it.
constexpr int STASH = 16;
constexpr int WSTASH = WST + 2 * 5 * STASH;
constexpr int WREG = WSTASH > WSM ? WSTASH : WSM;  // shared doubles per warp (step / absorb)

#ifdef FB_DBG_GRP
// (timing experiment: every group's warp 0 adds the globaltimer durations of
// its iteration phases into g_grp[k] (k = 0..6), g_grp[15] counts the
// iterations; finom_grp_read, tools/grp_time.py)
__device__ unsigned long long g_grp[16];
__device__ __forceinline__ unsigned long long grp_now() {
  unsigned long long t_;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));
  return t_;
}
#define GRP_STAMP(k)                                       \
  do {                                                     \
    if (j == 0 && lane == 0) {                             \
      const unsigned long long n_ = grp_now();             \
      if (k > 0) atomicAdd(&g_grp[k - 1], n_ - grp_t);     \
      else atomicAdd(&g_grp[15], 1ull);                    \
      grp_t = n_;                                          \
    }                                                      \
  } while (0)
#else
#define GRP_STAMP(k)
#endif
#define GRP_STAMP_IN(k)

struct GX;
struct GroupArgs {
  Dev d;
  double *S4;       // per tile: incoming (p, acc, q, accb) of the current half
  int *queue;       // [0]: next problem
  int g;            // warps per problem (1, 2, 4, 8, 16; cluster form: up to 256)
  GX *gxg;          // cluster form: exchange slots, g per cluster (global)
  long long gxstride;  // (unused by this loop form)
  double *a_out, *b_out;
  long long *info;
};

// One group's exchange slots in shared memory: per warp the chunk aggregates
// of both directions and the partials (err, max, min, fail).
struct GX {
  Tf f, b;
  double part[4];
  int prob, pad;
};

// A problem's group: g warps, this one is warp j.  CTA groups (g <= 16)
// synchronize with a named barrier and exchange through shared memory;
// cluster groups (a small problem spread over a thread-block cluster, up to
// 16 CTAs) with the cluster barrier and a global scratch (L2).
struct Grp {
  int g, j, bar;
  bool cluster;
  GX *gx;
  __device__ __forceinline__ void sync() const {
    if (cluster) {
      __threadfence();  // (gx lives in global memory)
      asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;"
                   ::: "memory");
    } else if (g == 1) {
      __syncwarp();
    } else {
      asm volatile("bar.sync %0, %1;" ::"r"(bar), "r"(32 * g) : "memory");
    }
  }
};
__device__ __forceinline__ Tf ld_tf(const Tf *p, bool global) {
  return global ? ldcg_tf(p) : *p;
}
__device__ __forceinline__ double ld_d(const double *p, bool global) {
  return global ? __ldcg(p) : *p;
}

// The states entering warp j of the group from the totals gx[0..g) of every
// warp: the composition of warps 0..j-1 (forward) / g-1..j+1 (backward)
// applied to the problem's zero boundary states, 32 warps per warp scan.
__device__ __forceinline__ void group_prefix(const Grp &G, int lane, double &p, double &acc,
                                             double &q, double &accb) {
  const int g = G.g, j = G.j;
  double sp = 0.0, sa = 0.0;
  for (int c = 0; c < g; c += 32) {
    const int k = c + lane;
    const Tf f = k < g ? ld_tf(&G.gx[k].f, G.cluster) : tf_id();
    Tf xf, xb, tf_, tb_;
    warp_scan2<true>(f, tf_id(), xf, xb, tf_, tb_);
    double pp = sp, aa = sa;
    tf_apply_g(xf, pp, aa);
    const int src = min(max(j - c, 0), 31);
    pp = __shfl_sync(0xffffffffu, pp, src);
    aa = __shfl_sync(0xffffffffu, aa, src);
    if (j >= c && j < c + 32) {
      p = pp;
      acc = aa;
    }
    tf_apply_g(tf_, sp, sa);
  }
  double sq = 0.0, sb = 0.0;
  const int nch = (g + 31) / 32;
  for (int ci = nch - 1; ci >= 0; --ci) {
    const int c = 32 * ci, k = c + lane;
    const Tf b = k < g ? ld_tf(&G.gx[k].b, G.cluster) : tf_id();
    Tf xf, xb, tf_, tb_;
    warp_scan2<true>(tf_id(), b, xf, xb, tf_, tb_);
    double qq = sq, bb = sb;
    tf_apply_g(xb, qq, bb);
    const int src = min(max(j - c, 0), 31);
    qq = __shfl_sync(0xffffffffu, qq, src);
    bb = __shfl_sync(0xffffffffu, bb, src);
    if (j >= c && j < c + 32) {
      q = qq;
      accb = bb;
    }
    tf_apply_g(tb_, sq, sb);
  }
}


// Per-tile incoming states of one half for tiles [b, e) of the warp (the
// warp's share of its problem): lane chunks composed sequentially, a warp
// scan, the group's other warps' totals (shared memory), then per-tile states
// into S4 (lane-sequential).  Maps: R.lev[0] (written by the previous half's
// epilogue or by the table build), forward composed left to right, backward
// right to left; guarded compositions (a structural zero stays zero).
__device__ __noinline__ void group_carries(const Resolve &R, double *S4, int b, int e,
                                           const Grp &G, int lane, const Tf *stash) {
  const int g = G.g, j = G.j;
  GX *gx = G.gx;
  const Node *nd = R.lev[0];
  const int n = e - b;
  const int L = (n + 31) / 32;
  const int lb = min(b + lane * L, e), le = min(lb + L, e);
  Tf f = tf_id(), bk = tf_id();
  if (stash && n <= STASH) {  // (L <= 1: this lane's tile, if any)
    if (lb < le) {
      f = stash[2 * (lb - b)];
      bk = stash[2 * (lb - b) + 1];
    }
  } else {
    for (int t = lb; t < le; ++t) f = tf_cat_g(f, ldcg_tf(&nd[t].tf));
    for (int t = le - 1; t >= lb; --t) bk = tf_cat_g(bk, ldcg_tf(&nd[t].tb));
  }
  GRP_STAMP_IN(8);
  Tf xf, xb, totf, totb;
  warp_scan2<true>(f, bk, xf, xb, totf, totb);
  GRP_STAMP_IN(9);
  double p = 0.0, acc = 0.0, q = 0.0, accb = 0.0;
  if (g > 1) {
    if (lane == 0) {
      gx[j].f = totf;
      gx[j].b = totb;
    }
    G.sync();
    GRP_STAMP_IN(10);
    // the totals of the group's earlier warps (forward) and later warps
    // (backward), applied to the problem's zero boundary states
    if (g <= 16) {
      for (int k = 0; k < j; ++k) tf_apply_g(ld_tf(&gx[k].f, G.cluster), p, acc);
      for (int k = g - 1; k > j; --k) tf_apply_g(ld_tf(&gx[k].b, G.cluster), q, accb);
    } else {
      group_prefix(G, lane, p, acc, q, accb);
    }
    GRP_STAMP_IN(11);
    // (no barrier: the partials write other fields of gx, and the next
    // writes of f / b come after the partials' barrier)
  }
  tf_apply_g(xf, p, acc);
  tf_apply_g(xb, q, accb);
  if (stash && n <= STASH) {
    if (lb < le) {
      S4[4 * (size_t)lb] = p;
      S4[4 * (size_t)lb + 1] = acc;
      S4[4 * (size_t)lb + 2] = q;
      S4[4 * (size_t)lb + 3] = accb;
    }
  } else {
    for (int t = lb; t < le; ++t) {
      S4[4 * (size_t)t] = p;
      S4[4 * (size_t)t + 1] = acc;
      tf_apply_g(ldcg_tf(&nd[t].tf), p, acc);
    }
    for (int t = le - 1; t >= lb; --t) {
      S4[4 * (size_t)t + 2] = q;
      S4[4 * (size_t)t + 3] = accb;
      tf_apply_g(ldcg_tf(&nd[t].tb), q, accb);
    }
  }
  __syncwarp();
}

// L2 prefetch of [p, p + bytes) (16-byte aligned interior).
__device__ __forceinline__ void l2_prefetch(const void *p, size_t bytes) {
  const unsigned long long a = reinterpret_cast<unsigned long long>(p);
  const unsigned long long a16 = (a + 15) & ~15ull, e16 = (a + bytes) & ~15ull;
  if (e16 > a16)
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(a16), "r"((unsigned)(e16 - a16))
                 : "memory");
}
// The next tile's record and vectors into L2 while this one computes.
template <int HALF>
__device__ __forceinline__ void group_prefetch(const Dev &d, int t, const TileStep &ts) {
  const int nr = HALF == 0 ? ts.ny : ts.nx, nc = HALF == 0 ? ts.nx : ts.ny;
  l2_prefetch(d.TR[HALF] + (size_t)t * TREC, (size_t)(((REC_KT + 3 * nr) * 8 + 15) & ~15));
  const long long rb = HALF == 0 ? ts.yb : ts.xb, cb = HALF == 0 ? ts.xb : ts.yb;
  if (HALF == 0) l2_prefetch(d.PSI + rb, 8 * (size_t)nr);
  l2_prefetch((HALF == 0 ? d.PHI : d.PSI) + cb, 8 * (size_t)nc);
}

// The scalings and records the bulk copies read were written by this
// kernel's generic stores (the previous half, a table rebuild): every lane
// orders its stores before the async-proxy reads -- once per half / rebuild.
__device__ __forceinline__ void proxy_fence() {
  asm volatile("fence.proxy.async.global;" ::: "memory");
  __syncwarp();
}

// One half step of tile t with incoming states init = S4 + 4t (the k_step
// loads without the tree and control reads); partials to part.  nts: the
// next tile's descriptor (prefetched into L2 during this tile), if any.
template <int HALF>
__device__ __forceinline__ void group_tile(const Dev &d, int t, const TileStep &ts, bool next,
                                           int tn, const TileStep &nts, double *wsm,
                                           unsigned long long *bar, int lane, unsigned &phase,
                                           const double *init, double *part, Tf *stash) {
  TileIn in;
  in.t = t;
  in.nr = HALF == 0 ? ts.ny : ts.nx;
  in.nc = HALF == 0 ? ts.nx : ts.ny;
  in.rb = HALF == 0 ? ts.yb : ts.xb;
  in.cb = HALF == 0 ? ts.xb : ts.yb;
  in.r0 = HALF == 0 ? ts.y0 : ts.x0;
  in.rec = wsm;
  in.reset = 0;
  const unsigned rbytes = (unsigned)(((REC_KT + 3 * in.nr) * 8 + 15) & ~15);
  const double *Rs = (HALF == 0 ? d.PSI : d.PHI) + in.rb;
  const double *Cs = (HALF == 0 ? d.PHI : d.PSI) + in.cb;
  in.rold = vec_place(in.rec + TREC, Rs);
  in.cv = vec_place(in.rold + (HALF == 0 ? in.nr : 0), Cs);
  if (lane == 0) {
    const VecStage vr = vec_stage(Rs, HALF == 0 ? in.nr : 0), vc = vec_stage(Cs, in.nc);
    bulk_expect(bar, rbytes + vr.bytes + vc.bytes);
    bulk_rec(in.rec, d.TR[HALF] + (size_t)t * TREC, rbytes, bar);
    vec_issue(in.rold, Rs, vr, bar);
    vec_issue(in.cv, Cs, vc, bar);
    // (measured at config 5: prefetch distance 2 1074 ms, record only
    // 1050, distance 1 with the vectors 1047 ms per solve)
    if (next) group_prefetch<HALF>(d, tn, nts);
  }
  // lanes 0 / 4: the incoming states (forward / backward), off the walk's path
  double st0 = 0.0, st1 = 0.0;
  if (lane == 0 || lane == 4) {
    st0 = __ldcg(init + (lane == 0 ? 0 : 2));
    st1 = __ldcg(init + (lane == 0 ? 1 : 3));
  }
  cp_async_wait();
  bar_wait(bar, phase & 1u);
  ++phase;
  __syncwarp();
#ifdef FB_DBG_PHASE
  long long ph_t0 = 0;
  tile_compute<HALF, true, false>(d, in, tf_id(), lane, ph_t0, nullptr, part, true, st0, st1,
                                  stash);
#else
  tile_compute<HALF, true, false>(d, in, tf_id(), lane, nullptr, part, true, st0, st1, stash);
#endif
}

// Partials of the warp's tiles (in tile order) -> the group's (in warp order).
__device__ __noinline__ void group_partials(double (&pw)[4], const Grp &G, int lane) {
  const int g = G.g, j = G.j;
  GX *gx = G.gx;
  if (g == 1) return;
  if (lane == 0)
    for (int k = 0; k < 4; ++k) gx[j].part[k] = pw[k];
  G.sync();
  double e = 0.0, mx = 0.0, mn = INFINITY, fl = -1.0;
  if (g <= 16) {  // (shared memory: warp order)
    for (int k = 0; k < g; ++k) {
      e = __dadd_rn(e, ld_d(&gx[k].part[0], G.cluster));
      mx = fmax(mx, ld_d(&gx[k].part[1], G.cluster));
      mn = fmin(mn, ld_d(&gx[k].part[2], G.cluster));
      fl = fmax(fl, ld_d(&gx[k].part[3], G.cluster));
    }
  } else {
    // large (cluster) groups: the lanes load the partials in parallel (one
    // round of loads per 32 warps instead of g dependent rounds), then fixed
    // butterfly reductions -- a fixed order for a given g.  (config 1 with
    // FB_CLUSTER=1: 68.6 -> 46.6 us per iteration)
    for (int c = 0; c < g; c += 32) {
      const int k = c + lane;
      if (k < g) {
        e = __dadd_rn(e, ld_d(&gx[k].part[0], G.cluster));
        mx = fmax(mx, ld_d(&gx[k].part[1], G.cluster));
        mn = fmin(mn, ld_d(&gx[k].part[2], G.cluster));
        fl = fmax(fl, ld_d(&gx[k].part[3], G.cluster));
      }
    }
    e = warp_sum(e);
    mx = warp_max(mx);
    mn = warp_min(mn);
    fl = warp_max(fl);
  }
  pw[0] = e;
  pw[1] = mx;
  pw[2] = mn;
  pw[3] = fl;
  // (no barrier: the next writes of the partials come after the next
  // half's barriers)
}

// The table (re)build of the warp's tiles, out of line: it runs at the start
// of a problem and on absorptions only, and keeps the hot loop's code small
// (the instruction cache holds the two half steps).
__device__ __noinline__ void group_build(const Dev &d, int build, int b, int e, double *wsm,
                                         const double2 *tab, int sb, bool had) {
  for (int t = b; t < e; ++t) {
    absorb_core(d, build, t, wsm, tab, sb, had);
    __syncwarp();
  }
}

// CLUSTER = false: groups of g <= 16 warps inside a CTA, problems from the
// queue.  CLUSTER = true: a thread-block cluster per problem (problem =
// cluster index), its warps one group (a.g = warps per CTA x cluster size),
// exchange through a.gxg (global, g entries per cluster).
template <bool CLUSTER>
__global__ void __launch_bounds__(GTHR, 1) k_solve_group(GroupArgs a) {
  extern __shared__ __align__(16) double smem[];
  __shared__ double2 tab[64];
  __shared__ GX gxs[GW];
  __shared__ int gprob[GW];
  __shared__ unsigned long long mbar[GW];  // (absorb_core uses the whole warp region)
  load_tab(tab);
  __syncthreads();
  const Dev &d = a.d;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nw = blockDim.x >> 5;
  Grp G;
  G.cluster = CLUSTER;
  int grp = 0, crank = 0, cid = 0;
  if (CLUSTER) {
    asm("mov.u32 %0, %%cluster_ctarank;" : "=r"(crank));
    asm("mov.u32 %0, %%clusterid.x;" : "=r"(cid));
    G.g = a.g;
    G.j = crank * nw + warp;
    G.bar = 0;
    G.gx = a.gxg + (size_t)cid * a.g;
  } else {
    G.g = a.g;
    G.j = warp % a.g;
    grp = warp / a.g;
    G.bar = 1 + grp;  // named barrier of the group (g > 1)
    G.gx = gxs + grp * a.g;
  }
  const int g = G.g, j = G.j;
  double *wsm = smem + (size_t)warp * WREG;
  unsigned long long *mb = mbar + warp;
  if (lane == 0) bar_init(mb);
  __syncwarp();
  unsigned phase = 0;
  for (int round = 0;; ++round) {
    int prob;
    if (CLUSTER) {
      prob = round == 0 ? cid : d.P;  // one problem per cluster
    } else {
      if (j == 0 && lane == 0) gprob[grp] = atomicAdd(a.queue, 1);
      G.sync();
      prob = gprob[grp];
      G.sync();
    }
    if (prob >= d.P) break;
    const ProbDesc &P = d.probs[prob];
    const int b = P.tile0 + (int)((long long)P.ntiles * j / g);
    const int e = P.tile0 + (int)((long long)P.ntiles * (j + 1) / g);
    // ---- solve prologue (solver.py:165-166): phi = psi = 1/n, shifts 0
    const double h0 = 1.0 / (double)P.n;
    if (e > b) {
      const TileDesc t0d = d.tiles[b], t1d = d.tiles[e - 1];
      for (int k = t0d.x0 + lane; k < t1d.x1; k += 32) {
        d.PHI[P.xoff + k] = h0;
        d.A[0][P.xoff + k] = 0.0;
      }
      for (int k = t0d.y0 + lane; k < t1d.y1; k += 32) {
        d.PSI[P.yoff + k] = h0;
        d.B[0][P.yoff + k] = 0.0;
      }
    }
    G.sync();
    // tables of the initial kernel, half A's maps for the initial phi
    group_build(d, 1, b, e, wsm, tab, 0, false);
    G.sync();
    int it = 0, status = 0, fail_it = 0, sbuf = 0, n_abs = 0, converged = 0;
#ifdef FB_DBG_GRP
    unsigned long long grp_t = 0;
#endif
    bool absorbed = false;
    bool stash_ok = false;  // (group_build wrote half A's maps to global only)
    Tf *stash = reinterpret_cast<Tf *>(wsm + WST);
    double err = 0.0;
    for (;;) {
      // ---- half A: psi <- v / K'^T phi (_kernels.py:278-314)
      GRP_STAMP(0);
      proxy_fence();
      group_carries(d.RA, a.S4, b, e, G, lane, stash_ok ? stash : nullptr);
      stash_ok = true;  // (half A's tiles write it for half B)
      GRP_STAMP(1);
      double pw[4] = {0.0, 0.0, INFINITY, -1.0};
      TileStep ts = d.steps[b < e ? b : 0];
      for (int t = b; t < e; ++t) {
        double pt[4];
        const TileStep nts = d.steps[t + 1 < e ? t + 1 : t];
        group_tile<0>(d, t, ts, t + 1 < e, t + 1, nts, wsm, mb, lane, phase,
                      a.S4 + 4 * (size_t)t, pt, t - b < STASH ? stash + 2 * (t - b) : nullptr);
        ts = nts;
        pw[0] = __dadd_rn(pw[0], pt[0]);
        pw[1] = fmax(pw[1], pt[1]);
        pw[2] = fmin(pw[2], pt[2]);
        pw[3] = fmax(pw[3], pt[3]);
      }
      pw[0] = warp_sum(pw[0]);  // (lane partials of the warp's tiles, in tile order per lane)
      GRP_STAMP(2);
      group_partials(pw, G, lane);
      GRP_STAMP(3);
      err = pw[0];
      const bool ps_oor = pw[1] > 0.0;  // (epi_rows<.., EXT = false>: out-of-range flag)
      if (j == 0 && lane == 0) d.hist[(long long)prob * d.itr_max + it] = err;
      if (pw[3] >= 0.0) {  // solver.py:177-184 (failure in half A)
        const long long fl = (long long)pw[3];
        status = (int)(fl & 3);
        fail_it = it + 1;
        it += 1;
        break;
      }
      // ---- half B: phi <- u / K' psi (_kernels.py:315-349)
      // (every psi of the problem is final: each warp passed the partials'
      // barrier after its tiles)
      GRP_STAMP(4);
      proxy_fence();
      group_carries(d.RB, a.S4, b, e, G, lane, stash_ok ? stash : nullptr);
      GRP_STAMP(5);
      double qw[4] = {0.0, 0.0, INFINITY, -1.0};
      // half B walks the warp's tiles backwards (half A forwards): its first
      // tiles read the scalings half A wrote last, still in L2 (and half A's
      // first ones half B's last); config 5: 1003.5 -> 995 ms
      TileStep ts1 = d.steps[e > b ? e - 1 : 0];
      for (int t = e - 1; t >= b; --t) {
        double pt[4];
        const TileStep nts = d.steps[t - 1 >= b ? t - 1 : t];
        group_tile<1>(d, t, ts1, t - 1 >= b, t - 1, nts, wsm, mb, lane, phase,
                      a.S4 + 4 * (size_t)t, pt, t - b < STASH ? stash + 2 * (t - b) : nullptr);
        ts1 = nts;
        qw[1] = fmax(qw[1], pt[1]);
        qw[2] = fmin(qw[2], pt[2]);
        qw[3] = fmax(qw[3], pt[3]);
      }
      GRP_STAMP(6);
      group_partials(qw, G, lane);
      GRP_STAMP(7);
      const bool ph_oor = qw[1] > 0.0;
      const int k = ++it;  // solver.py:177
      if (qw[3] >= 0.0) {
        const long long fl = (long long)qw[3];
        status = (int)(fl & 3);
        fail_it = k;
        break;
      }
      if (d.tol > 0.0 && err <= d.tol) {  // solver.py:188-192
        converged = 1;
        break;
      }
      bool reb = false;
      if (d.stabilize && (ph_oor || ps_oor)) {  // solver.py:193-198: absorb, phi = psi = 1
        reb = true;
        if (j == 0 && lane == 0 && d.absorb_its)
          d.absorb_its[(long long)prob * d.itr_max + n_abs] = k;
        n_abs += 1;
        G.sync();  // every phi of the problem is final
        group_build(d, 0, b, e, wsm, tab, sbuf, absorbed);
        stash_ok = false;  // (absorb_core's area overlaps the stash; the maps are in global)
        G.sync();  // every tile has read the old shifts and scalings
        sbuf ^= 1;
        absorbed = true;
        if (e > b) {
          const TileDesc t0d = d.tiles[b], t1d = d.tiles[e - 1];
          for (int q = t0d.x0 + lane; q < t1d.x1; q += 32) d.PHI[P.xoff + q] = 1.0;
          for (int q = t0d.y0 + lane; q < t1d.y1; q += 32) d.PSI[P.yoff + q] = 1.0;
        }
        __syncwarp();
      }
      if (k >= d.itr_max) break;
      // every phi / half-A map of the problem is final: the partials' barrier
      // covers the tiles; after a rebuild, the resets above need one more
      if (reb) G.sync();
    }
    // ---- k_final's part: shifts out, info, control block
    const double *As = d.A[sbuf], *Bs = d.B[sbuf];
    if (e > b) {
      const TileDesc t0d = d.tiles[b], t1d = d.tiles[e - 1];
      for (int q = t0d.x0 + lane; q < t1d.x1; q += 32)
        a.a_out[P.xoff + q] = absorbed ? As[P.xoff + q] : 0.0;
      for (int q = t0d.y0 + lane; q < t1d.y1; q += 32)
        a.b_out[P.yoff + q] = absorbed ? Bs[P.yoff + q] : 0.0;
    }
    if (j == 0 && lane == 0) {
      long long *inf = a.info + 5 * (long long)prob;
      inf[0] = it;
      inf[1] = converged;
      inf[2] = status;
      inf[3] = n_abs;
      inf[4] = fail_it;
      Ctl c{};
      c.it = it;
      c.done = 1;
      c.status = status;
      c.fail_it = fail_it;
      c.absorbed = absorbed;
      c.converged = converged;
      c.n_absorb = n_abs;
      c.sbuf = sbuf;
      c.err = err;
      d.ctl[prob] = c;
    }
    G.sync();
  }
}

}  // namespace fb
