// Square line sweeps: the 2D sweeps when a grid axis of the source equals
// the target's (BASELINE configs 3 and 4: source grid == target grid).
//
// On such a line every mesh point z_r is both a row and a column, so the
// merged order of kernel1d's dividing index (searchsorted "right",
// kernel1d.py:55-62: the tie column r belongs to row r's lower block) is
// fixed and the two recurrences of _dp_apply / _dp_apply_dyn
// (_kernels.py:53-203) take one step per point instead of one per slot:
//
//   P_r = rho_r * P_{r-1} + delta_r * v_r        (lower block, columns <= r)
//   Q_r = sigma_r * Q_{r+1} + mu_r * v_{r+1}     (upper block, columns > r)
//   out_r = P_r + Q_r
//
// with, for row-side shifts alpha and column-side shifts beta of the line
// (both zero before the first absorption) and g_r = z_r - z_{r-1}:
//   rho_r   = exp((-g_r + alpha_r - alpha_{r-1}) / eps)      lower ratio
//   delta_r = exp((alpha_r + beta_r) / eps)                  diagonal edge
//   sigma_r = exp((-g_{r+1} + alpha_r - alpha_{r+1}) / eps)  upper ratio
//   mu_r    = exp((-g_{r+1} + alpha_r + beta_{r+1}) / eps)   upper edge
// -- the reference's exponent expressions: "/ eps" (kernel1d.py:121-159)
// for the baked tables before the first absorption, "* inv_eps"
// (_kernels.py:128-203) for the dyn form after it; evaluated once per
// absorption epoch.
//
// Records per tile of SQT = 256 points (lane l holds points 8l .. 8l+7):
//   F: (rho, delta) then (sigma, mu), double2 at [j][k][lane]   (8 KB)
//   W: (wf, wb) double2 at [k][lane], the tile-map weights      (4 KB)
//      wf_r = delta_r prod_{s > r} rho_s, wb_r = mu_r prod_{s < r} sigma_s
//   S: (prod rho, prod sigma) of the tile
// so a tile's maps for values v are P_last = S.x P_in + sum wf v and
// Q_first = S.y Q_after + sum wb v_{+1} (k_sq_pre), resolved along the line
// (k_sq_scan) and applied (k_sq_apply).
#pragma once

namespace fb {

constexpr int SQE = 8;                 // points per lane of a square-sweep tile

// Partials of the 2D scaling update (k_epi2d, fused square sweeps).
struct EpiPart {
  double err, vmax, vmin;
  long long fail;  // min over failing flat indices of (idx << 2) | status; LLONG_MAX if none
};
// The CTA's partial in a fixed order: warp trees, then thread 0 folds the warps.
__device__ __forceinline__ void epi_block_part(double err, double vmax, double vmin,
                                               long long fail, EpiPart *out) {
  __shared__ EpiPart sp[32];
  err = warp_sum(err);
  vmax = warp_max(vmax);
  vmin = warp_min(vmin);
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    const long long o = __shfl_xor_sync(0xffffffffu, fail, off);
    fail = o < fail ? o : fail;
  }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (lane == 0) sp[warp] = EpiPart{err, vmax, vmin, fail};
  __syncthreads();
  if (threadIdx.x == 0) {
    EpiPart r{0.0, 0.0, INFINITY, LLONG_MAX};
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) {
      r.err += sp[w].err;
      r.vmax = fmax(r.vmax, sp[w].vmax);
      r.vmin = fmin(r.vmin, sp[w].vmin);
      r.fail = sp[w].fail < r.fail ? sp[w].fail : r.fail;
    }
    *out = r;
  }
}

constexpr int SQT = 32 * SQE;          // points per tile
constexpr int SQF = 2 * SQE * 32;      // double2 of F per tile
constexpr int SQW = SQE * 32;          // double2 of W per tile

struct SqArgs {
  const double *Z;        // the line mesh (z[0..n))
  const double *alpha;    // nullable: row-side shifts, line p at alpha + p * n
  const double *beta;     // nullable: column-side shifts, same layout
  double2 *F, *W, *S;     // records (shared: one line's worth)
  // split records (column-side shifts only): F, S shared (the ratios do not
  // depend on beta), W shared raw factors (prod rho, prod sigma parts), and
  // per line only D = (delta, mu), double2 at [tile][k][lane]
  double2 *D;
  int wraw;               // k_sq_build: write W as the raw factors (split mode)
  Node *nodes;            // per (line, tile): maps / exclusive maps
  const double *vin;      // input values, line p at vin + p * n
  double *out_t;          // output, transposed: out_t[r * lines + p]
  int n, lines, tl;       // points per line, lines, tiles per line
  int shared;             // records shared by every line (no shifts)
  double inv;             // 1 / eps
  double eps;
  int baked;              // k_sq_build: the baked (pre-absorption) exponents x / eps
                          // (kernel1d.py:142, :148) instead of the dyn x * inv_eps
  // fused scaling update (nullable ew: plain sweep): SC <- W / out over the
  // flat grid out_t addresses, marginal error (eerr), extremes, failures;
  // per-CTA partials into epart (k_epi_fold reduces them in a fixed order)
  const double *ew;
  double *esc;
  EpiPart *epart;
  int eerr;
  int ek0, eng;           // failure indices: row shard [ek0, ..) of eng grid rows (0, lines: whole grid)
  // row-shard window (the x sweeps of a shard): the lines are the segment
  // [k0, k0 + n) of lines of the whole mesh (Z already offset by k0)
  int k0;
  const double *carry;    // nullable: per line incoming (p, acc, q, accb) from the other shards
  double *tot;            // nullable: per line segment totals (forward Tf, backward Tf)
};

// Records of one tile (warp per (line, tile); shared records: line 0 only).
__global__ void __launch_bounds__(NTHR) k_sq_build(SqArgs a) {
  const int lane = threadIdx.x & 31;
  const long long w = (long long)blockIdx.x * WPC + (threadIdx.x >> 5);
  const int nl = a.shared ? 1 : a.lines;
  if (w >= (long long)nl * a.tl) return;
  const int p = (int)(w / a.tl), t = (int)(w % a.tl);
  const double *al = a.alpha ? a.alpha + (size_t)p * a.n : nullptr;
  const double *be = a.beta ? a.beta + (size_t)p * a.n : nullptr;
  auto A = [&](int r) { return al ? al[r] : 0.0; };
  auto B = [&](int r) { return be ? be[r] : 0.0; };
  const int r0 = t * SQT + SQE * lane;
  // exponent argument: baked tables divide by eps (kernel1d.py:142, :148;
  // q_div is the IEEE quotient), the dyn form multiplies by inv_eps
  // (_kernels.py:140-159)
  auto arg = [&](double num) { return a.baked ? q_div(num, a.eps, a.inv) : __dmul_rn(num, a.inv); };
  double rho[SQE], del[SQE], sig[SQE], mu[SQE];
#pragma unroll
  for (int k = 0; k < SQE; ++k) {
    const int r = r0 + k;
    rho[k] = 1.0; del[k] = 0.0; sig[k] = 1.0; mu[k] = 0.0;  // padding: identity steps
    if (r < a.n) {
      del[k] = exp(arg(__dadd_rn(A(r), B(r))));
      if (r > 0 || a.k0 > 0)  // (a window's first point: the mesh point before it is a.Z[-1])
        rho[k] = exp(arg(__dadd_rn(-(a.Z[r] - a.Z[r - 1]), __dsub_rn(A(r), A(r - 1)))));
      if (r + 1 < a.n) {
        const double g = a.Z[r + 1] - a.Z[r];
        sig[k] = exp(arg(__dadd_rn(-g, __dsub_rn(A(r), A(r + 1)))));
        mu[k] = exp(arg(__dadd_rn(-g, __dadd_rn(A(r), B(r + 1)))));
      }
    }
  }
  // in-lane suffix products of rho (after k) and prefix products of sigma (before k)
  double sp[SQE], pp[SQE];
  sp[SQE - 1] = 1.0;
  for (int k = SQE - 2; k >= 0; --k) sp[k] = __dmul_rn(rho[k + 1], sp[k + 1]);
  pp[0] = 1.0;
  for (int k = 1; k < SQE; ++k) pp[k] = __dmul_rn(sig[k - 1], pp[k - 1]);
  const double rt = __dmul_rn(rho[0], sp[0]), st = __dmul_rn(sig[SQE - 1], pp[SQE - 1]);
  // across lanes: products of later lanes' rho, of earlier lanes' sigma
  double sx = rt, px = st;
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    const double o1 = __shfl_down_sync(0xffffffffu, sx, off);
    const double o2 = __shfl_up_sync(0xffffffffu, px, off);
    if (lane + off < 32) sx = __dmul_rn(sx, o1);
    if (lane >= off) px = __dmul_rn(o2, px);
  }
  // inclusive -> exclusive
  double sxe = __shfl_down_sync(0xffffffffu, sx, 1), pxe = __shfl_up_sync(0xffffffffu, px, 1);
  if (lane == 31) sxe = 1.0;
  if (lane == 0) pxe = 1.0;
  const size_t tile = (size_t)p * a.tl + t;
  double2 *F = a.F + tile * SQF, *W = a.W + tile * SQW;
#pragma unroll
  for (int k = 0; k < SQE; ++k) {
    F[k * 32 + lane] = make_double2(rho[k], del[k]);
    F[(SQE + k) * 32 + lane] = make_double2(sig[k], mu[k]);
    W[k * 32 + lane] = a.wraw ? make_double2(__dmul_rn(sp[k], sxe), __dmul_rn(pp[k], pxe))
                              : make_double2(__dmul_rn(del[k], __dmul_rn(sp[k], sxe)),
                                             __dmul_rn(mu[k], __dmul_rn(pp[k], pxe)));
  }
  const double af = __shfl_sync(0xffffffffu, sx, 0), ab = __shfl_sync(0xffffffffu, px, 31);
  if (lane == 0) a.S[tile] = make_double2(af, ab);
}

// Per-line (delta, mu) of the split records: k_sq_build's expressions with
// alpha = 0 (warp per (line, tile)).
__global__ void __launch_bounds__(NTHR) k_sq_build_d(SqArgs a) {
  const int lane = threadIdx.x & 31;
  const long long w = (long long)blockIdx.x * WPC + (threadIdx.x >> 5);
  if (w >= (long long)a.lines * a.tl) return;
  const int p = (int)(w / a.tl), t = (int)(w % a.tl);
  const double *be = a.beta + (size_t)p * a.n;
  const int r0 = t * SQT + SQE * lane;
  double2 *D = a.D + (size_t)w * SQW;
#pragma unroll
  for (int k = 0; k < SQE; ++k) {
    const int r = r0 + k;
    double del = 0.0, mu = 0.0;
    if (r < a.n) {
      del = exp(__dmul_rn(__dadd_rn(0.0, be[r]), a.inv));
      if (r + 1 < a.n)
        mu = exp(__dmul_rn(__dadd_rn(-(a.Z[r + 1] - a.Z[r]), __dadd_rn(0.0, be[r + 1])), a.inv));
    }
    D[k * 32 + lane] = make_double2(del, mu);
  }
}

// This lane's v_r for r = t0 + SQE lane .. + SQE (SQE + 1 values, zero past
// the line): the warp's SQT + 1 values are loaded coalesced into xs (one pad
// double per SQE, so the lanes' SQE-strided reads hit distinct banks), then
// each lane reads its run.  (A lane reading its run straight from global
// memory touches 32 sectors per instruction.)
constexpr int SQX = SQT + SQT / SQE + 2;  // staging doubles per warp
__device__ __forceinline__ int sq_pad(int i) { return i + i / SQE; }
__device__ __forceinline__ void sq_load_v(const double *v, int t0, int n, double *xs,
                                          double (&x)[SQE + 1]) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int k = 0; k < SQE; ++k) {
    const int i = lane + 32 * k;
    xs[sq_pad(i)] = t0 + i < n ? __ldg(v + t0 + i) : 0.0;
  }
  if (lane == 0) xs[sq_pad(SQT)] = t0 + SQT < n ? __ldg(v + t0 + SQT) : 0.0;
  __syncwarp();
#pragma unroll
  for (int k = 0; k <= SQE; ++k) x[k] = xs[sq_pad(SQE * lane + k)];
  __syncwarp();
}

// The tiles' maps for the input values: tf = (prod rho, 0, sum wf v, 1, 0),
// tb = (prod sigma, 0, sum wb v_{+1}, 1, 0) in the Tf encoding
// (p' = A p + C; acc unused), written as the tile's node.
__global__ void __launch_bounds__(NTHR) k_sq_pre(SqArgs a) {
  const int lane = threadIdx.x & 31;
  const long long w = (long long)blockIdx.x * WPC + (threadIdx.x >> 5);
  if (w >= (long long)a.lines * a.tl) return;
  const int p = (int)(w / a.tl), t = (int)(w % a.tl);
  griddep_wait();  // (programmatic dependent launch: the input is the previous sweep's output)
  const size_t rec = a.shared || a.D ? (size_t)t : (size_t)w;
  const double2 *W = a.W + rec * SQW;
  const double2 *D = a.D ? a.D + (size_t)w * SQW : nullptr;
  __shared__ double xs[WPC][SQX];
  double x[SQE + 1];
  double2 sprod = make_double2(1.0, 1.0);  // (lane 0: the tile's ratio products, loaded early)
  if (lane == 0) sprod = __ldg(a.S + rec);
  sq_load_v(a.vin + (size_t)p * a.n, t * SQT, a.n, xs[threadIdx.x >> 5], x);
  double cf = 0.0, cb = 0.0;
#pragma unroll
  for (int k = 0; k < SQE; ++k) {
    double2 wk = __ldg(W + k * 32 + lane);
    if (D) {  // split records: the same products as k_sq_build's W
      const double2 dk = __ldcs(D + k * 32 + lane);
      wk = make_double2(__dmul_rn(dk.x, wk.x), __dmul_rn(dk.y, wk.y));
    }
    cf = __fma_rn(wk.x, x[k], cf);
    cb = __fma_rn(wk.y, x[k + 1], cb);
  }
  cf = warp_sum(cf);
  cb = warp_sum(cb);
  if (lane == 0) {
    Node *nd = a.nodes + w;
    nd->tf = Tf{sprod.x, 0.0, cf, 1.0, 0.0};
    nd->tb = Tf{sprod.y, 0.0, cb, 1.0, 0.0};
  }
  griddep_launch();
}

// Exclusive maps of every tile along its line (warp per line, chunks of 32
// tiles carried across chunks; guarded compositions as across 1D tiles).
__global__ void __launch_bounds__(NTHR) k_sq_scan(SqArgs a) {
  const int lane = threadIdx.x & 31;
  const int p = blockIdx.x * WPC + (threadIdx.x >> 5);
  if (p >= a.lines) return;
  griddep_wait();
  Node *lv = a.nodes + (size_t)p * a.tl;
  const int n = a.tl, nch = (n + 31) / 32;
  Tf cf = tf_id(), cb = tf_id();
  for (int c = 0; c < nch; ++c) {
    const int lt = 32 * c + lane;
    const bool have = lt < n;
    const Tf f = have ? ldcg_tf(&lv[lt].tf) : tf_id();
    const Tf b = have && nch == 1 ? ldcg_tf(&lv[lt].tb) : tf_id();
    Tf xf, xb, totf, totb;
    warp_scan2<true>(f, b, xf, xb, totf, totb);
    if (have) {
      lv[lt].xf = tf_cat_g(cf, xf);
      if (nch == 1) lv[lt].xb = xb;
    }
    cf = tf_cat_g(cf, totf);
    if (nch == 1) cb = totb;
  }
  for (int c = nch - 1; nch > 1 && c >= 0; --c) {
    const int lt = 32 * c + lane;
    const bool have = lt < n;
    const Tf b = have ? ldcg_tf(&lv[lt].tb) : tf_id();
    Tf xf, xb, totf, totb;
    warp_scan2<true>(tf_id(), b, xf, xb, totf, totb);
    if (have) lv[lt].xb = tf_cat_g(cb, xb);
    cb = tf_cat_g(cb, totb);
  }
  if (a.tot && lane == 0) {  // the line segment's totals (row shards: k_sq_seg_tot)
    double *o = a.tot + 10 * (size_t)p;
    o[0] = cf.A; o[1] = cf.B; o[2] = cf.C; o[3] = cf.D; o[4] = cf.E;
    o[5] = cb.A; o[6] = cb.B; o[7] = cb.C; o[8] = cb.D; o[9] = cb.E;
  }
  griddep_launch();
}

// A row shard's exported segment totals (k_seg_carry's input, 10 doubles per
// line): the forward total as is; the backward total extended by the step
// into the last row of the shard before (row k0 - 1 of the whole mesh):
// Q_{k0-1} = sigma_{k0-1} Q_{k0} + mu_{k0-1} v_{k0}, with k_sq_build's
// exponent expressions (alpha = 0, beta = this line's shifts).
__global__ void k_sq_seg_tot(SqArgs a, double *out) {
  for (int p = blockIdx.x * blockDim.x + threadIdx.x; p < a.lines; p += gridDim.x * blockDim.x) {
    const double *t = a.tot + 10 * (size_t)p;
    double *o = out + 10 * (size_t)p;
    for (int k = 0; k < 5; ++k) o[k] = t[k];
    double A = t[5], C = t[7];
    if (a.k0 > 0) {
      const double g = a.Z[0] - a.Z[-1];
      const double be = a.beta ? a.beta[(size_t)p * a.n] : 0.0;
      auto arg = [&](double num) {
        return a.baked ? q_div(num, a.eps, a.inv) : __dmul_rn(num, a.inv);
      };
      const double sig = exp(arg(__dadd_rn(-g, __dsub_rn(0.0, 0.0))));
      const double mu = exp(arg(__dadd_rn(-g, __dadd_rn(0.0, be))));
      const double v0 = a.vin[(size_t)p * a.n];
      A = gm(sig, A);
      C = __dadd_rn(gm(sig, C), __dmul_rn(mu, v0));
    }
    o[5] = A; o[6] = t[6]; o[7] = C; o[8] = t[8]; o[9] = t[9];
  }
}

// The sweep: CTA = tile t of LPC consecutive lines (a warp per line); lane l
// walks points 8l .. 8l+7 of its warp's tile.  Lane maps of both
// recurrences, two warp scans (the tile's incoming P / Q folded into the end
// lanes), the final recurrences in the reference's operation order
// ((r * p) + acc, p + q), then the CTA writes the rows transposed: LPC
// consecutive doubles of every output row (LPC = 16: whole 128-byte lines;
// 4: 32-byte sectors).
template <int LPC>
__global__ void __launch_bounds__(32 * LPC) k_sq_apply(SqArgs a) {
  constexpr int THR = 32 * LPC;
  __shared__ double so[LPC][SQX];  // input staging, then the tile's outputs
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int t = blockIdx.x % a.tl, p0 = (blockIdx.x / a.tl) * LPC, p = p0 + warp;
  griddep_wait();
  // the fused scaling update's operands (weights, old scalings) start into
  // shared memory with the tile's other loads (cp.async: no registers held),
  // each thread its own elements: the update finds them on chip instead of
  // paying a second DRAM round trip at the end of the CTA (config 4: 399 ->
  // 381 ms per solve; 4 lines per CTA only -- 16 KB of shared memory)
  __shared__ double sew[LPC == 4 ? 2 * LPC * SQT : 1];
  if (LPC == 4 && a.ew) {
    const int cnt0 = min(SQT, a.n - t * SQT);
#pragma unroll
    for (int q = 0; q < SQT * LPC / THR; ++q) {
      const int kk = threadIdx.x + q * THR, i = kk / LPC, w = kk % LPC;
      if (kk < cnt0 * LPC && p0 + w < a.lines) {
        const long long idx = (long long)(t * SQT + i) * a.lines + p0 + w;
        cp_async8(sew + kk, a.ew + idx);
        if (a.eerr) cp_async8(sew + LPC * SQT + kk, a.esc + idx);
      }
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  }
  if (p < a.lines) {
    const size_t tile = (size_t)p * a.tl + t;
    const size_t rec = a.shared || a.D ? (size_t)t : tile;
    const double2 *F = a.F + rec * SQF;
    double2 f0[SQE], f1[SQE];
    // lanes 0 / 31: the tile's exclusive maps and the line's incoming carry
    // (their latency hides behind the loads below)
    double nA = 1.0, nC = 0.0, ncar = 0.0;
    if (lane == 0 || lane == 31) {
      const Tf *xm = lane == 0 ? &a.nodes[tile].xf : &a.nodes[tile].xb;
      nA = __ldcg(&xm->A);
      nC = __ldcg(&xm->C);
      if (a.carry) ncar = __ldg(a.carry + 4 * (size_t)p + (lane == 0 ? 0 : 2));
    }
    // the input first (its staging is the first dependent use), then the
    // factors (config 4: 437 -> 423 ms per solve)
    double xr[SQE + 1];
    {
      const double *v = a.vin + (size_t)p * a.n;
      const int t0 = t * SQT;
#pragma unroll
      for (int kk = 0; kk < SQE; ++kk) {
        const int i = lane + 32 * kk;
        xr[kk] = t0 + i < a.n ? __ldg(v + t0 + i) : 0.0;
      }
      xr[SQE] = lane == 0 && t0 + SQT < a.n ? __ldg(v + t0 + SQT) : 0.0;
    }
    if (a.D) {  // split records: shared ratios, the line's (delta, mu)
      const double2 *D = a.D + tile * SQW;
#pragma unroll
      for (int k = 0; k < SQE; ++k) {
        const double2 dk = __ldcs(D + k * 32 + lane);
        f0[k] = make_double2(__ldg(&F[k * 32 + lane].x), dk.x);
        f1[k] = make_double2(__ldg(&F[(SQE + k) * 32 + lane].x), dk.y);
      }
    } else {
#pragma unroll
      for (int k = 0; k < SQE; ++k) {
        f0[k] = __ldcs(F + k * 32 + lane);
        f1[k] = __ldcs(F + (SQE + k) * 32 + lane);
      }
    }
    double x[SQE + 1];
    {
      double *sw = so[warp];
#pragma unroll
      for (int kk = 0; kk < SQE; ++kk) sw[sq_pad(lane + 32 * kk)] = xr[kk];
      if (lane == 0) sw[sq_pad(SQT)] = xr[SQE];
      __syncwarp();
#pragma unroll
      for (int kk = 0; kk <= SQE; ++kk) x[kk] = sw[sq_pad(SQE * lane + kk)];
      __syncwarp();
    }
    double pin = 0.0, qin = 0.0;  // the tile's incoming P (lane 0) / Q (lane 31)
    // (the tile's exclusive maps applied to the line's incoming states: zero,
    // or a row shard's carries from the other shards, as tf_apply_g)
    if (lane == 0) pin = (gm(nA, ncar) + 0.0) + nC;
    if (lane == 31) qin = (gm(nA, ncar) + 0.0) + nC;
    // lane maps: forward P_end = af P_in + cf, backward Q_first = ab Q_after + cb
    double af = 1.0, cf = 0.0, ab = 1.0, cb = 0.0;
#pragma unroll
    for (int k = 0; k < SQE; ++k) {
      f0[k].y = __dmul_rn(f0[k].y, x[k]);      // delta v
      f1[k].y = __dmul_rn(f1[k].y, x[k + 1]);  // mu v_{+1}
      af = __dmul_rn(f0[k].x, af);
      cf = __dadd_rn(__dmul_rn(f0[k].x, cf), f0[k].y);
    }
#pragma unroll
    for (int k = SQE - 1; k >= 0; --k) {
      ab = __dmul_rn(f1[k].x, ab);
      cb = __dadd_rn(__dmul_rn(f1[k].x, cb), f1[k].y);
    }
    // fold the tile's inputs into the end lanes, then inclusive scans
    if (lane == 0) { cf = __fma_rn(af, pin, cf); af = 0.0; }
    if (lane == 31) { cb = __fma_rn(ab, qin, cb); ab = 0.0; }
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      const double oa = __shfl_up_sync(0xffffffffu, af, off);
      const double oc = __shfl_up_sync(0xffffffffu, cf, off);
      const double ob = __shfl_down_sync(0xffffffffu, ab, off);
      const double od = __shfl_down_sync(0xffffffffu, cb, off);
      if (lane >= off) { cf = __fma_rn(af, oc, cf); af = __dmul_rn(af, oa); }
      if (lane + off < 32) { cb = __fma_rn(ab, od, cb); ab = __dmul_rn(ab, ob); }
    }
    double pp = __shfl_up_sync(0xffffffffu, cf, 1), qq = __shfl_down_sync(0xffffffffu, cb, 1);
    if (lane == 0) pp = pin;
    if (lane == 31) qq = qin;
    // final recurrences (_kernels.py:65-67 / :80-87 order)
#pragma unroll
    for (int k = 0; k < SQE; ++k) {
      pp = __dadd_rn(__dmul_rn(f0[k].x, pp), f0[k].y);
      f0[k].y = pp;
    }
#pragma unroll
    for (int k = SQE - 1; k >= 0; --k) {
      qq = __dadd_rn(__dmul_rn(f1[k].x, qq), f1[k].y);
      so[warp][SQE * lane + k] = __dadd_rn(f0[k].y, qq);
    }
  }
  __syncthreads();
  const int cnt = min(SQT, a.n - t * SQT);
  if (!a.ew) {
    for (int k = threadIdx.x; k < cnt * LPC; k += THR) {
      const int i = k / LPC, w = k % LPC;
      if (p0 + w < a.lines) a.out_t[(size_t)(t * SQT + i) * a.lines + p0 + w] = so[w][i];
    }
    griddep_launch();
    return;
  }
  // the grid's scaling update on the same addresses (k_epi2d's rules,
  // _kernels.py:376-397 / :408-427): no T round trip through HBM
  double err = 0.0, vmax = 0.0, vmin = INFINITY;
  long long fail = LLONG_MAX;
  // every load of the thread's elements is issued before the first use
  constexpr int EPER = SQT * LPC / THR;
  double wq[EPER], sq[EPER];
  if (LPC == 4) {
    asm volatile("cp.async.wait_group 0;" ::: "memory");
#pragma unroll
    for (int q = 0; q < EPER; ++q) {
      const int k = threadIdx.x + q * THR, w = k % LPC;
      const bool live = k < cnt * LPC && p0 + w < a.lines;
      wq[q] = live ? sew[k] : 0.0;
      sq[q] = live && a.eerr ? sew[LPC * SQT + k] : 0.0;
    }
  } else {
#pragma unroll
    for (int q = 0; q < EPER; ++q) {
      const int k = threadIdx.x + q * THR, i = k / LPC, w = k % LPC;
      const bool live = k < cnt * LPC && p0 + w < a.lines;
      const long long idx = (long long)(t * SQT + i) * a.lines + p0 + w;
      wq[q] = live ? __ldcs(a.ew + idx) : 0.0;
      sq[q] = live && a.eerr ? __ldcs(a.esc + idx) : 0.0;
    }
  }
  // fast path: t in [2^-1021, 2^1021] and weight < 4 -- no rule of
  // _kernels.py:376-397 can fire and div_fast is the IEEE quotient (a
  // subnormal quotient takes the exact path below); branch-free, the y sweep
  // being issue-bound on this update (config 4: 370 -> 364 ms per solve)
  bool slow = false;
  {
    double e2 = 0.0, mx = 0.0, mn = INFINITY;
#pragma unroll
    for (int q = 0; q < EPER; ++q) {
      const int k = threadIdx.x + q * THR, i = k / LPC, w = k % LPC;
      const bool lv = k < cnt * LPC && p0 + w < a.lines;
      const long long idx = (long long)(t * SQT + i) * a.lines + p0 + w;
      const double wv = wq[q], tt = lv ? so[w][i] : 1.0;
      if (a.eerr) e2 = __dadd_rn(e2, fabs(__dsub_rn(__dmul_rn(sq[q], tt), wv)));
      const double nv = div_fast(wv, tt);
      slow |= !(tt >= 0x1p-1021 && tt <= 0x1p1021 && wv < 4.0) || (nv < 0x1p-1000 && wv != 0.0);
      const bool ok = wv > 0.0;
      mx = ok && nv > mx ? nv : mx;
      mn = ok && nv < mn ? nv : mn;
      if (lv) a.esc[idx] = nv;
    }
    if (!slow) { err = e2; vmax = mx; vmin = mn; }
  }
  if (slow) {
#pragma unroll
  for (int q = 0; q < EPER; ++q) {
    const int k = threadIdx.x + q * THR, i = k / LPC, w = k % LPC;
    if (k >= cnt * LPC || p0 + w >= a.lines) continue;
    const long long idx = (long long)(t * SQT + i) * a.lines + p0 + w;
    // flat index of the whole grid (a row shard holds rows [ek0, ek0 + lines) of eng)
    const long long kg = a.ek0 + p0 + w + (long long)a.eng * (t * SQT + i);
    const double wv = wq[q], tt = so[w][i];
    if (a.eerr) err = __dadd_rn(err, fabs(__dsub_rn(__dmul_rn(sq[q], tt), wv)));
    double nv;
    if (tt == 0.0) {
      if (wv > 0.0) fail = min(fail, (kg << 2) | ST_ZD);
      nv = 0.0;
    } else {
      nv = __ddiv_rn(wv, tt);
      if (!isfinite(nv)) fail = min(fail, (kg << 2) | ST_NF);
      else if (wv > 0.0) {
        vmax = fmax(vmax, nv);
        vmin = fmin(vmin, nv);
      }
    }
    a.esc[idx] = nv;
  }
  }
  epi_block_part(err, vmax, vmin, fail, a.epart + blockIdx.x);
  griddep_launch();
}

// Short lines (tl <= SQ_FUSE = 4 tiles, config 3): one CTA per LPC lines runs a
// whole sweep -- k_sq_pre's tile maps, k_sq_scan's single-chunk warp scan and
// k_sq_apply, with the same operations in the same order (bitwise equal to
// the three-kernel path), the maps exchanged through shared memory.  Warp w
// takes tile w / LPC of line p0 + w % LPC; the input tile is read once (the
// pre phase's registers feed the apply phase) and the records of both phases
// are issued before the first dependent read.  The transposed output and the
// fused scaling update run per tile over the tile's LPC warps (named barrier
// 1 + tile), so the partials are k_sq_apply's, per (line group, tile).
constexpr int SQ_FUSE = 4;
template <int LPC>
__global__ void __launch_bounds__(32 * LPC * SQ_FUSE) k_sq_fused(SqArgs a) {
  extern __shared__ __align__(16) double fsm[];
  constexpr int GT = 32 * LPC;  // threads per tile group
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int t = warp / LPC, l = warp % LPC, tl = a.tl;
  const int p0 = blockIdx.x * LPC, p = p0 + l;
  double *so = fsm + (size_t)warp * SQX;
  Tf *maps = reinterpret_cast<Tf *>(fsm + (size_t)LPC * tl * SQX);  // [LPC][tl][2]
  const bool live = p < a.lines;
  const size_t tile = (size_t)p * tl + t;
  const size_t rec = a.shared || a.D ? (size_t)t : tile;
  double2 f0[SQE], f1[SQE];
  double x[SQE + 1];
  griddep_wait();
  if (live) {
    const double2 *W = a.W + rec * SQW;
    sq_load_v(a.vin + (size_t)p * a.n, t * SQT, a.n, so, x);
    // ---- k_sq_pre: the tile's maps
    double cf = 0.0, cb = 0.0;
    if (a.D) {  // split records: shared ratios and raw W, the line's (delta, mu)
      const double2 *D = a.D + tile * SQW;
#pragma unroll
      for (int k = 0; k < SQE; ++k) {
        const double2 dk = __ldcs(D + k * 32 + lane);
        const double2 w = __ldg(W + k * 32 + lane);
        f0[k].y = dk.x;
        f1[k].y = dk.y;
        cf = __fma_rn(__dmul_rn(dk.x, w.x), x[k], cf);
        cb = __fma_rn(__dmul_rn(dk.y, w.y), x[k + 1], cb);
      }
    } else {
#pragma unroll
      for (int k = 0; k < SQE; ++k) {
        const double2 w = __ldg(W + k * 32 + lane);
        cf = __fma_rn(w.x, x[k], cf);
        cb = __fma_rn(w.y, x[k + 1], cb);
      }
    }
    cf = warp_sum(cf);
    cb = warp_sum(cb);
    if (lane == 0) {
      const double2 s = __ldg(a.S + rec);
      maps[2 * (l * tl + t)] = Tf{s.x, 0.0, cf, 1.0, 0.0};
      maps[2 * (l * tl + t) + 1] = Tf{s.y, 0.0, cb, 1.0, 0.0};
    }
  }
  __syncthreads();
  if (live) {
    // ---- k_sq_scan (one chunk), then lane t's exclusive maps applied to zero
    const bool have = lane < tl;
    const Tf f = have ? maps[2 * (l * tl + lane)] : tf_id();
    const Tf b = have ? maps[2 * (l * tl + lane) + 1] : tf_id();
    Tf xf, xb, totf, totb;
    warp_scan2<true>(f, b, xf, xb, totf, totb);
    const Tf X = tf_cat_g(tf_id(), xf);
    const double pv = (gm(X.A, 0.0) + 0.0) + X.C, qv = (gm(xb.A, 0.0) + 0.0) + xb.C;
    double pin = __shfl_sync(0xffffffffu, pv, t), qin = __shfl_sync(0xffffffffu, qv, t);
    // ---- k_sq_apply (its records)
    const double2 *F = a.F + rec * SQF;
    if (a.D) {
#pragma unroll
      for (int k = 0; k < SQE; ++k) {
        f0[k].x = __ldg(&F[k * 32 + lane].x);
        f1[k].x = __ldg(&F[(SQE + k) * 32 + lane].x);
      }
    } else {
#pragma unroll
      for (int k = 0; k < SQE; ++k) {
        f0[k] = __ldcs(F + k * 32 + lane);
        f1[k] = __ldcs(F + (SQE + k) * 32 + lane);
      }
    }
    double af = 1.0, cf = 0.0, ab = 1.0, cb = 0.0;
#pragma unroll
    for (int k = 0; k < SQE; ++k) {
      f0[k].y = __dmul_rn(f0[k].y, x[k]);
      f1[k].y = __dmul_rn(f1[k].y, x[k + 1]);
      af = __dmul_rn(f0[k].x, af);
      cf = __dadd_rn(__dmul_rn(f0[k].x, cf), f0[k].y);
    }
#pragma unroll
    for (int k = SQE - 1; k >= 0; --k) {
      ab = __dmul_rn(f1[k].x, ab);
      cb = __dadd_rn(__dmul_rn(f1[k].x, cb), f1[k].y);
    }
    if (lane == 0) { cf = __fma_rn(af, pin, cf); af = 0.0; }
    if (lane == 31) { cb = __fma_rn(ab, qin, cb); ab = 0.0; }
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      const double oa = __shfl_up_sync(0xffffffffu, af, off);
      const double oc = __shfl_up_sync(0xffffffffu, cf, off);
      const double ob = __shfl_down_sync(0xffffffffu, ab, off);
      const double od = __shfl_down_sync(0xffffffffu, cb, off);
      if (lane >= off) { cf = __fma_rn(af, oc, cf); af = __dmul_rn(af, oa); }
      if (lane + off < 32) { cb = __fma_rn(ab, od, cb); ab = __dmul_rn(ab, ob); }
    }
    double pp = __shfl_up_sync(0xffffffffu, cf, 1), qq = __shfl_down_sync(0xffffffffu, cb, 1);
    if (lane == 0) pp = pin;
    if (lane == 31) qq = qin;
#pragma unroll
    for (int k = 0; k < SQE; ++k) {
      pp = __dadd_rn(__dmul_rn(f0[k].x, pp), f0[k].y);
      f0[k].y = pp;
    }
#pragma unroll
    for (int k = SQE - 1; k >= 0; --k) {
      qq = __dadd_rn(__dmul_rn(f1[k].x, qq), f1[k].y);
      so[SQE * lane + k] = __dadd_rn(f0[k].y, qq);
    }
  }
  // ---- per tile: transposed write or the fused scaling update (k_sq_apply's)
  const int tid = threadIdx.x - GT * t;  // thread within the tile's group
  asm volatile("bar.sync %0, %1;" ::"r"(1 + t), "r"(GT) : "memory");
  const int cnt = min(SQT, a.n - t * SQT);
  double *sg = fsm + (size_t)t * LPC * SQX;  // the group's LPC output rows
  if (!a.ew) {
    for (int k = tid; k < cnt * LPC; k += GT) {
      const int i = k / LPC, w = k % LPC;
      if (p0 + w < a.lines) a.out_t[(size_t)(t * SQT + i) * a.lines + p0 + w] = sg[w * SQX + i];
    }
    griddep_launch();
    return;
  }
  double err = 0.0, vmax = 0.0, vmin = INFINITY;
  long long fail = LLONG_MAX;
  constexpr int EPER = SQT * LPC / GT;
  double wq[EPER], sq[EPER];
#pragma unroll
  for (int q = 0; q < EPER; ++q) {
    const int k = tid + q * GT, i = k / LPC, w = k % LPC;
    const bool lv = k < cnt * LPC && p0 + w < a.lines;
    const long long idx = (long long)(t * SQT + i) * a.lines + p0 + w;
    wq[q] = lv ? __ldcs(a.ew + idx) : 0.0;
    sq[q] = lv && a.eerr ? __ldcs(a.esc + idx) : 0.0;
  }
#pragma unroll
  for (int q = 0; q < EPER; ++q) {
    const int k = tid + q * GT, i = k / LPC, w = k % LPC;
    if (k >= cnt * LPC || p0 + w >= a.lines) continue;
    const long long idx = (long long)(t * SQT + i) * a.lines + p0 + w;
    const long long kg = a.ek0 + p0 + w + (long long)a.eng * (t * SQT + i);
    const double wv = wq[q], tt = sg[w * SQX + i];
    if (a.eerr) err = __dadd_rn(err, fabs(__dsub_rn(__dmul_rn(sq[q], tt), wv)));
    double nv;
    if (tt == 0.0) {
      if (wv > 0.0) fail = min(fail, (kg << 2) | ST_ZD);
      nv = 0.0;
    } else {
      nv = __ddiv_rn(wv, tt);
      if (!isfinite(nv)) fail = min(fail, (kg << 2) | ST_NF);
      else if (wv > 0.0) {
        vmax = fmax(vmax, nv);
        vmin = fmin(vmin, nv);
      }
    }
    a.esc[idx] = nv;
  }
  // epi_block_part over the group's LPC warps (same fold order as a LPC-warp CTA)
  __shared__ EpiPart sp[SQ_FUSE][LPC];
  err = warp_sum(err);
  vmax = warp_max(vmax);
  vmin = warp_min(vmin);
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    const long long o = __shfl_xor_sync(0xffffffffu, fail, off);
    fail = o < fail ? o : fail;
  }
  if (lane == 0) sp[t][l] = EpiPart{err, vmax, vmin, fail};
  asm volatile("bar.sync %0, %1;" ::"r"(1 + t), "r"(GT) : "memory");
  if (tid == 0) {
    EpiPart r{0.0, 0.0, INFINITY, LLONG_MAX};
    for (int w = 0; w < LPC; ++w) {
      r.err += sp[t][w].err;
      r.vmax = fmax(r.vmax, sp[t][w].vmax);
      r.vmin = fmin(r.vmin, sp[t][w].vmin);
      r.fail = sp[t][w].fail < r.fail ? sp[t][w].fail : r.fail;
    }
    a.epart[(size_t)blockIdx.x * tl + t] = r;
  }
  griddep_launch();
}

// The same short-line sweep with ONE scan per tile (the default): the lane
// maps of both recurrences come from the factors the warp holds in registers,
// their inclusive warp scans give the tile's maps (lane 31 / lane 0) -- no W
// records, no separate tile-map pass --, the maps of a line's <= SQ_FUSE tiles
// meet in shared memory, a guarded two-component scan gives the tile's
// incoming P / Q, and every lane starts its recurrences from
// (lanes before) o (tiles before) applied to zero.  The reference's per-point
// operations ((r * p) + acc, p + q; _kernels.py:65-67 / :80-87) are
// unchanged; the cross-lane compositions are reassociated differently from
// k_sq_fused / the three kernels (1e-14 apart).  Fewer instructions and one
// dependent phase less per tile: config 3 26.0 -> 23.6 ms per solve even
// through a cluster launch (the experiment this came from), see DESIGN.md.
template <int LPC>
__global__ void __launch_bounds__(32 * LPC * SQ_FUSE) k_sq_fuse1(SqArgs a) {
  extern __shared__ __align__(16) double fsm[];
  constexpr int GT = 32 * LPC;  // threads per tile group
  __shared__ EpiPart sp[SQ_FUSE][LPC];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int t = warp / LPC, l = warp % LPC, tl = a.tl;
  const int p0 = blockIdx.x * LPC, p = p0 + l;
  double *so = fsm + (size_t)warp * SQX;
  // (fwd A, fwd C, bwd A, bwd C) per (line, tile)
  double4 *maps = reinterpret_cast<double4 *>(fsm + (size_t)LPC * tl * SQX);
  const bool live = p < a.lines;
  const size_t tile = (size_t)p * tl + t;
  double2 f0[SQE], f1[SQE];
  double exa = 1.0, exc = 0.0, exb = 1.0, exd = 0.0;  // the lanes before / after this one
  griddep_wait();
  if (live) {
    const size_t rec = a.shared || a.D ? (size_t)t : tile;
    const double2 *F = a.F + rec * SQF;
    // the input first (its staging is the first dependent use), then the factors
    double xr[SQE + 1];
    {
      const double *v = a.vin + (size_t)p * a.n;
      const int t0 = t * SQT;
#pragma unroll
      for (int kk = 0; kk < SQE; ++kk) {
        const int i = lane + 32 * kk;
        xr[kk] = t0 + i < a.n ? __ldg(v + t0 + i) : 0.0;
      }
      xr[SQE] = lane == 0 && t0 + SQT < a.n ? __ldg(v + t0 + SQT) : 0.0;
    }
    if (a.D) {  // split records: shared ratios, the line's (delta, mu)
      const double2 *D = a.D + tile * SQW;
#pragma unroll
      for (int k = 0; k < SQE; ++k) {
        const double2 dk = __ldcs(D + k * 32 + lane);
        f0[k] = make_double2(__ldg(&F[k * 32 + lane].x), dk.x);
        f1[k] = make_double2(__ldg(&F[(SQE + k) * 32 + lane].x), dk.y);
      }
    } else if (a.shared) {
#pragma unroll
      for (int k = 0; k < SQE; ++k) {
        f0[k] = __ldg(F + k * 32 + lane);
        f1[k] = __ldg(F + (SQE + k) * 32 + lane);
      }
    } else {
#pragma unroll
      for (int k = 0; k < SQE; ++k) {
        f0[k] = __ldcs(F + k * 32 + lane);
        f1[k] = __ldcs(F + (SQE + k) * 32 + lane);
      }
    }
    double x[SQE + 1];
#pragma unroll
    for (int kk = 0; kk < SQE; ++kk) so[sq_pad(lane + 32 * kk)] = xr[kk];
    if (lane == 0) so[sq_pad(SQT)] = xr[SQE];
    __syncwarp();
#pragma unroll
    for (int kk = 0; kk <= SQE; ++kk) x[kk] = so[sq_pad(SQE * lane + kk)];
    __syncwarp();
    // lane maps: forward P_end = af P_in + cf, backward Q_first = ab Q_after + cb
    double af = 1.0, cf = 0.0, ab = 1.0, cb = 0.0;
#pragma unroll
    for (int k = 0; k < SQE; ++k) {
      f0[k].y = __dmul_rn(f0[k].y, x[k]);      // delta v
      f1[k].y = __dmul_rn(f1[k].y, x[k + 1]);  // mu v_{+1}
      af = __dmul_rn(f0[k].x, af);
      cf = __dadd_rn(__dmul_rn(f0[k].x, cf), f0[k].y);
    }
#pragma unroll
    for (int k = SQE - 1; k >= 0; --k) {
      ab = __dmul_rn(f1[k].x, ab);
      cb = __dadd_rn(__dmul_rn(f1[k].x, cb), f1[k].y);
    }
    // inclusive scans of the lane maps (in-tile products stay in range: no guards)
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      const double oa = __shfl_up_sync(0xffffffffu, af, off);
      const double oc = __shfl_up_sync(0xffffffffu, cf, off);
      const double ob = __shfl_down_sync(0xffffffffu, ab, off);
      const double od = __shfl_down_sync(0xffffffffu, cb, off);
      if (lane >= off) { cf = __fma_rn(af, oc, cf); af = __dmul_rn(af, oa); }
      if (lane + off < 32) { cb = __fma_rn(ab, od, cb); ab = __dmul_rn(ab, ob); }
    }
    // the tile's maps: lane 31 holds the forward one, lane 0 the backward one
    double *mp = reinterpret_cast<double *>(&maps[l * tl + t]);
    if (lane == 31) { mp[0] = af; mp[1] = cf; }
    if (lane == 0) { mp[2] = ab; mp[3] = cb; }
    exa = __shfl_up_sync(0xffffffffu, af, 1);
    exc = __shfl_up_sync(0xffffffffu, cf, 1);
    exb = __shfl_down_sync(0xffffffffu, ab, 1);
    exd = __shfl_down_sync(0xffffffffu, cb, 1);
    if (lane == 0) { exa = 1.0; exc = 0.0; }
    if (lane == 31) { exb = 1.0; exd = 0.0; }
  }
  __syncthreads();  // every tile map of the CTA's lines is written
  if (live) {
    // lane j: tile j's maps of this line; guarded inclusive scans along the
    // line (cross-tile products may overflow or underflow: a structurally
    // zero state stays zero, as tf_cat_g); SQ_FUSE <= 4 tiles: two levels
    double fa = 1.0, fc = 0.0, ba = 1.0, bc = 0.0;
    if (lane < tl) {
      const double4 m = maps[l * tl + lane];
      fa = m.x; fc = m.y; ba = m.z; bc = m.w;
    }
#pragma unroll
    for (int off = 1; off < SQ_FUSE; off <<= 1) {
      const double oa = __shfl_up_sync(0xffffffffu, fa, off);
      const double oc = __shfl_up_sync(0xffffffffu, fc, off);
      const double ob = __shfl_down_sync(0xffffffffu, ba, off);
      const double od = __shfl_down_sync(0xffffffffu, bc, off);
      if (lane >= off) { fc = __dadd_rn(gm(fa, oc), fc); fa = gm(fa, oa); }
      if (lane + off < 32) { bc = __dadd_rn(gm(ba, od), bc); ba = gm(ba, ob); }
    }
    // the tile's incoming states: P after tile t - 1, Q before tile t + 1 (zero at the line's ends)
    double pin = __shfl_sync(0xffffffffu, fc, t > 0 ? t - 1 : 0);
    double qin = __shfl_sync(0xffffffffu, bc, t + 1);
    if (t == 0) pin = 0.0;
    if (t + 1 >= tl) qin = 0.0;
    // this lane's incoming states, then the final recurrences
    double pp = __dadd_rn(gm(exa, pin), exc), qq = __dadd_rn(gm(exb, qin), exd);
#pragma unroll
    for (int k = 0; k < SQE; ++k) {
      pp = __dadd_rn(__dmul_rn(f0[k].x, pp), f0[k].y);
      f0[k].y = pp;
    }
#pragma unroll
    for (int k = SQE - 1; k >= 0; --k) {
      qq = __dadd_rn(__dmul_rn(f1[k].x, qq), f1[k].y);
      so[SQE * lane + k] = __dadd_rn(f0[k].y, qq);
    }
  }
  // ---- per tile: transposed write or the fused scaling update (k_sq_apply's)
  const int tid = threadIdx.x - GT * t;  // thread within the tile's group
  asm volatile("bar.sync %0, %1;" ::"r"(1 + t), "r"(GT) : "memory");
  const int cnt = min(SQT, a.n - t * SQT);
  double *sg = fsm + (size_t)t * LPC * SQX;  // the group's LPC output rows
  if (!a.ew) {
    for (int k = tid; k < cnt * LPC; k += GT) {
      const int i = k / LPC, w = k % LPC;
      if (p0 + w < a.lines) a.out_t[(size_t)(t * SQT + i) * a.lines + p0 + w] = sg[w * SQX + i];
    }
    griddep_launch();
    return;
  }
  double err = 0.0, vmax = 0.0, vmin = INFINITY;
  long long fail = LLONG_MAX;
  constexpr int EPER = SQT * LPC / GT;
  double wq[EPER], sq[EPER];
#pragma unroll
  for (int q = 0; q < EPER; ++q) {
    const int k = tid + q * GT, i = k / LPC, w = k % LPC;
    const bool lv = k < cnt * LPC && p0 + w < a.lines;
    const long long idx = (long long)(t * SQT + i) * a.lines + p0 + w;
    wq[q] = lv ? __ldcs(a.ew + idx) : 0.0;
    sq[q] = lv && a.eerr ? __ldcs(a.esc + idx) : 0.0;
  }
#pragma unroll
  for (int q = 0; q < EPER; ++q) {
    const int k = tid + q * GT, i = k / LPC, w = k % LPC;
    if (k >= cnt * LPC || p0 + w >= a.lines) continue;
    const long long idx = (long long)(t * SQT + i) * a.lines + p0 + w;
    const long long kg = a.ek0 + p0 + w + (long long)a.eng * (t * SQT + i);
    const double wv = wq[q], tt = sg[w * SQX + i];
    if (a.eerr) err = __dadd_rn(err, fabs(__dsub_rn(__dmul_rn(sq[q], tt), wv)));
    double nv;
    if (tt == 0.0) {
      if (wv > 0.0) fail = min(fail, (kg << 2) | ST_ZD);
      nv = 0.0;
    } else {
      nv = __ddiv_rn(wv, tt);
      if (!isfinite(nv)) fail = min(fail, (kg << 2) | ST_NF);
      else if (wv > 0.0) {
        vmax = fmax(vmax, nv);
        vmin = fmin(vmin, nv);
      }
    }
    a.esc[idx] = nv;
  }
  // epi_block_part over the group's LPC warps (same fold order as a LPC-warp CTA)
  err = warp_sum(err);
  vmax = warp_max(vmax);
  vmin = warp_min(vmin);
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    const long long o = __shfl_xor_sync(0xffffffffu, fail, off);
    fail = o < fail ? o : fail;
  }
  if (lane == 0) sp[t][l] = EpiPart{err, vmax, vmin, fail};
  asm volatile("bar.sync %0, %1;" ::"r"(1 + t), "r"(GT) : "memory");
  if (tid == 0) {
    EpiPart r{0.0, 0.0, INFINITY, LLONG_MAX};
    for (int w = 0; w < LPC; ++w) {
      r.err += sp[t][w].err;
      r.vmax = fmax(r.vmax, sp[t][w].vmax);
      r.vmin = fmin(r.vmin, sp[t][w].vmin);
      r.fail = sp[t][w].fail < r.fail ? sp[t][w].fail : r.fail;
    }
    a.epart[(size_t)blockIdx.x * tl + t] = r;
  }
  griddep_launch();
}

}  // namespace fb
