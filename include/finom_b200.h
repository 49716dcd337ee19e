/*
 * finom_b200.h -- C ABI of the B200-native FINOM hot path.
 *
 * The reference (pure Python + numba, /root/reference/pkg/src/finom) has no
 * native FFI; its hot path is the numba kernel table routed by
 * _kernels._route (_kernels.py:540-596).  Each entry point below replaces
 * one of those kernels or the Python loop that drives them; the reference
 * interface it stands in for is cited per function.  INTEGRATION.md shows
 * the ctypes binding a maintainer would add to finom._kernels.
 *
 * Conventions
 *   - plain pointers and sizes only; `stream` is a cudaStream_t (NULL = the
 *     legacy default stream);
 *   - *_dev pointers are device memory, *_host pointers host memory;
 *   - every function returns a status: 0 OK, 1 ZERO_DENOM, 2 NONFINITE
 *     (_kernels.py:47-50), >= 100 argument / CUDA errors
 *     (finom_last_error() has the message);
 *   - 1D problems are batched: P problems, problem p owns
 *     x[xoff[p] .. xoff[p+1]) and y[yoff[p] .. yoff[p+1]) of the
 *     concatenated meshes (P = 1 is the reference's single problem);
 *   - no global mutable state: a plan owns its buffers; distinct plans may
 *     be used from different host threads on different streams.
 */
#ifndef FINOM_B200_H
#define FINOM_B200_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define FINOM_OK 0
#define FINOM_ZERO_DENOM 1
#define FINOM_NONFINITE 2
#define FINOM_EARG 100
#define FINOM_ECUDA 101

typedef struct finom_plan1d finom_plan1d;

/* Message of the last error on this thread. */
const char *finom_last_error(void);

/* Library / kernel build identification (sm_100a). */
const char *finom_build_info(void);

/* Builds the device plan for P 1D problems: uploads the meshes, computes the
 * dividing-index tile partition (kernel1d.dividing_index,
 * kernel1d.py:55-62, and the merge-path split of x U y) and allocates the
 * work buffers.  Replaces kernel1d.build_operator (kernel1d.py:234-255).
 * The solve loop keeps per-tile kernel tables for the current absorption
 * epoch (built on the device at solve start and rebuilt at every
 * absorption, like the reference's assembled reps, kernel1d.py:121-159);
 * apply / cost evaluate their factors on the fly. */
int finom_plan1d_create(int64_t P, const int64_t *xoff_host, const double *x_host,
                        const int64_t *yoff_host, const double *y_host,
                        const double *eps_host, void *stream, finom_plan1d **plan_out);
int finom_plan1d_destroy(finom_plan1d *plan);

/* The same plan from P separate host meshes (x_ptrs[p] of n[p] doubles,
 * y_ptrs[p] of m[p]): staged straight from the problems' arrays, no host
 * concatenation (the batched API). */
int finom_plan1d_create_v(int64_t P, const int64_t *n_host, const double *const *x_ptrs,
                          const int64_t *m_host, const double *const *y_ptrs,
                          const double *eps_host, void *stream, finom_plan1d **plan_out);

/* Plans and grids allocate from a library-owned memory pool that keeps up to
 * FINOM_POOL_KEEP_GB (env, default 64) GiB of freed memory for the next
 * plan; this returns all of it to the driver. */
int finom_release_memory(void);

/* Host-only: the merge-path tile partition of one mesh pair and the
 * merged-order masks the kernels walk (no CUDA call; for tests).  Returns the
 * tile count; fills up to max_tiles entries of tiles4 (x0, x1, y0, y1) and
 * masks16 (8 words half A order | 8 words half B order, bit = column). */
int64_t finom_tile_partition(int64_t n, const double *x, int64_t m, const double *y,
                             int64_t max_tiles, int32_t *tiles4, uint32_t *masks16);
/* Number of tiles, points etc. (for tests and bench accounting). */
int finom_plan1d_info(const finom_plan1d *plan, int64_t *info8);

/* The scaling loop for every problem of the plan, entirely on device:
 * solver.run_driver (solver.py:156-199) with adapter.iterate ==
 * _kernels.iter_1d (_kernels.py:260-350) and adapter.absorb ==
 * kernel1d.absorb + solver._shift (kernel1d.py:313-325, solver.py:135-153).
 *   u_dev, v_dev        weights (concatenated like x, y)
 *   phi_dev, psi_dev    out: scaling vectors (initialised to 1/n inside)
 *   a_dev, b_dev        out: accumulated log-domain shifts
 *   hist_dev            out: P x itr_max, err of every iteration
 *                       (history cadence is applied by the caller)
 *   info_dev            out: P x 5 int64: iterations_run, converged,
 *                       status, n_absorb, failed iteration
 *   absorb_its_dev      out (nullable): P x itr_max absorb iterations
 * Returns the worst per-problem status (0 if all problems ran clean). */
int finom_solve1d(finom_plan1d *plan, const double *u_dev, const double *v_dev,
                  double *phi_dev, double *psi_dev, double *a_dev, double *b_dev,
                  int64_t itr_max, double tol, int stabilize, double absorb_threshold,
                  double *hist_dev, int64_t *info_dev, int64_t *absorb_its_dev, void *stream);

/* finom_solve1d without waiting for the device: returns 0 once the loop is
 * queued on `stream` (or an error >= 100); each problem's status is
 * info_dev[5 p + 2] when the stream has run.  The batched API's pipeline
 * queues chunk k's solve and stages chunk k + 1 while it runs. */
int finom_solve1d_async(finom_plan1d *plan, const double *u_dev, const double *v_dev,
                        double *phi_dev, double *psi_dev, double *a_dev, double *b_dev,
                        int64_t itr_max, double tol, int stabilize, double absorb_threshold,
                        double *hist_dev, int64_t *info_dev, int64_t *absorb_its_dev,
                        void *stream);

/* transport_cost_fast (solver.py:252-271) per problem, with the shifts
 * a_dev/b_dev (nullable = zero) folded into the kernel. cost_dev: P doubles,
 * final once `stream` has run (no host wait inside). */
int finom_cost1d(finom_plan1d *plan, const double *a_dev, const double *b_dev,
                 const double *phi_dev, const double *psi_dev, double *cost_dev, void *stream);

/* kernel1d.apply / apply_transpose / apply_blocks (kernel1d.py:284-310),
 * i.e. _kernels.dp_apply / dp_blocks (_kernels.py:53-125) on the operator
 * with shifts a_dev/b_dev (nullable = zero).
 *   mode 0: out = K' in   (in: len m per problem, out: len n)
 *   mode 1: out = K'^T in (in: len n, out: len m)
 *   mode 2: out = K'_L in, out2 = K'_U in (blocks of mode 0) */
int finom_apply1d(finom_plan1d *plan, const double *a_dev, const double *b_dev,
                  const double *in_dev, int mode, double *out_dev, double *out2_dev,
                  void *stream);

/* One scaling iteration from an arbitrary state, in place: the adapter
 * protocol's iterate(u, v, phi, psi) (solver.py:1-16, :126-128) for a
 * kernel carrying shifts a_dev/b_dev (nullable).  res_dev receives, per
 * problem, 6 doubles: err, status, psmax, psmin, phmax, phmin. */
int finom_iterate1d(finom_plan1d *plan, const double *u_dev, const double *v_dev,
                    double *phi_dev, double *psi_dev, const double *a_dev, const double *b_dev,
                    double *res_dev, void *stream);

/* Per-kernel timing of `iters` solve-loop iterations launched without a
 * graph, CUDA events on `stream` around every launch (bench.py roofline).
 * ms_out[6]: mean ms of the half-A tile kernel, the half-B tile kernel, one
 * carry scan, the absorb kernel, one whole iteration; launches/iteration. */
int finom_profile1d(finom_plan1d *plan, const double *u_dev, const double *v_dev,
                    double *phi_dev, double *psi_dev, double *a_dev, double *b_dev,
                    int64_t iters, int stabilize, double absorb_threshold, double *hist_dev,
                    double *ms_out, void *stream);

/* Host <-> device copy of one contiguous buffer through the library's pinned
 * staging ring (host threads per 8 MB piece, pipelined DMA): dir 0 host ->
 * device, dir 1 device -> host.  Synchronous.  (The batched API's
 * transfers; pageable copies run at a fraction of the link rate.) */
int finom_stage_copy(int dir, void *host, void *dev, int64_t bytes);

/* count host pieces (host_ptrs[k], bytes[k]) <-> one contiguous device
 * buffer dev (dir 0: gather into dev, dir 1: scatter out of dev) through the
 * pinned staging ring; abutting pieces share slots.  Synchronous. */
int finom_stage_pieces(int dir, void *const *host_ptrs, const int64_t *bytes, int64_t count,
                       void *dev);

/* Number of kernel launches one finom_solve1d call issues. */
int64_t finom_solve1d_launches(const finom_plan1d *plan, int64_t itr_max, int stabilize);

/* Loop form finom_solve1d uses for this plan: 0 = the tile-parallel loop
 * (k_step / k_resolve per half, device-looped graph), g > 0 = the group
 * solve (one persistent k_solve_group launch, g warps per problem; batches
 * that fill the GPU).  FB_GROUP=0/1 in the environment forces. */
int finom_solve1d_group(const finom_plan1d *plan);

/* End-to-end call with HOST buffers (one problem): sinkhorn_1d
 * (solver.py:202-230) including transport_cost_fast.  hist_host: itr_max
 * doubles; info_host: 5 int64 (as finom_solve1d); cost_host: 1 double.
 * timing_host (nullable): 3 doubles = setup s, loop s, cost s. */
int finom_sinkhorn1d_host(int64_t n, const double *x, int64_t m, const double *y,
                          const double *u, const double *v, double eps, int64_t itr_max,
                          double tol, int stabilize, double absorb_threshold, double *phi,
                          double *psi, double *a, double *b, double *hist, int64_t *info,
                          int64_t *absorb_its, double *cost, double *timing_host);

/* 2D grids (kernel2d.py:363-391 sinkhorn_2d with transport_cost_fast_2d).
 * Source grid x1[n1] x y1[m1], target x2[n2] x y2[m2]; U (n1 x m1) and V
 * (n2 x m2) column-major (x fastest, mesh.py:85-107), or row-major when
 * w_rowmajor != 0 (a C-ordered numpy grid; transposed on the device).
 * Outputs phi, A (n1*m1), psi, B (n2*m2) flat column-major; hist / info /
 * absorb_its / cost / timing as finom_sinkhorn1d_host.  Replaces
 * _kernels.iter_2d_baked / iter_2d_dyn (_kernels.py:353-521) driven by
 * run_driver. */
int finom_sinkhorn2d_host(int64_t n1, const double *x1, int64_t m1, const double *y1, int64_t n2,
                          const double *x2, int64_t m2, const double *y2, const double *U,
                          const double *V, double eps, int64_t itr_max, double tol, int stabilize,
                          double absorb_threshold, double *phi, double *psi, double *A_out,
                          double *B_out, double *hist, int64_t *info, int64_t *absorb_its,
                          double *cost, double *timing, int w_rowmajor);

/* KernelOperator2D.apply (transpose = 0: out n1*m1 = K' in, in n2*m2) and
 * apply_transpose (transpose = 1) with optional shift grids A, B
 * (kernel2d.py:70-90, apply_2d / apply_2d_stabilized :139-258). */
int finom_apply2d_host(int64_t n1, const double *x1, int64_t m1, const double *y1, int64_t n2,
                       const double *x2, int64_t m2, const double *y2, double eps, const double *A,
                       const double *B, const double *in, int transpose, double *out);

/* transport_cost_fast_2d (kernel2d.py:394-465) for a given state. */
int finom_cost2d_host(int64_t n1, const double *x1, int64_t m1, const double *y1, int64_t n2,
                      const double *x2, int64_t m2, const double *y2, double eps, const double *A,
                      const double *B, const double *phi, const double *psi, double *cost);

/* ---- 2D grids on device buffers (the plan / solve split of sinkhorn_2d) ----
 * A grid plan holds the sweep plans, scratch grids and solve state of one
 * (source x1[n1] x y1[m1], target x2[n2] x y2[m2], eps) -- build it once,
 * then solve / iterate / cost on caller-owned device buffers with no
 * allocation.  Grids are flat column-major (x fastest, mesh.py:85-107).
 * Replaces kernel2d.build_operator_2d + _GridAdapter (kernel2d.py:293-360)
 * and the _kernels.iter_2d_baked / iter_2d_dyn loop (_kernels.py:353-521). */
typedef struct finom_grid finom_grid;
int finom_grid_create(int64_t n1, const double *x1_host, int64_t m1, const double *y1_host,
                      int64_t n2, const double *x2_host, int64_t m2, const double *y2_host,
                      double eps, void *stream, finom_grid **grid_out);
int finom_grid_destroy(finom_grid *grid);
/* info8: n1, m1, n2, m2, table-driven sweeps, square x sweeps, square y
 * sweeps, kernel launches of the last finom_solve2d (graph nodes counted) */
int finom_grid_info(const finom_grid *grid, int64_t *info8);
/* sinkhorn_2d's loop (run_driver, solver.py:156-199): U_dev (n1 m1), V_dev
 * (n2 m2) weights; phi_dev / psi_dev out; a_dev / b_dev out: the shift grids
 * (the loop's work buffers); hist_dev itr_max doubles; info_dev 5 int64 (as
 * finom_solve1d); absorb_its_dev itr_max int64 (nullable).  The host only
 * wakes at absorptions (tables rebuilt) and at the end. */
int finom_solve2d(finom_grid *grid, const double *U_dev, const double *V_dev, double *phi_dev,
                  double *psi_dev, double *a_dev, double *b_dev, int64_t itr_max, double tol,
                  int stabilize, double absorb_threshold, double *hist_dev, int64_t *info_dev,
                  int64_t *absorb_its_dev, void *stream);
/* transport_cost_fast_2d (kernel2d.py:394-465) of (phi, psi, a, b) into one
 * device double (a_dev, b_dev both NULL: the plain kernel). */
int finom_cost2d(finom_grid *grid, const double *phi_dev, const double *psi_dev,
                 const double *a_dev, const double *b_dev, double *cost_dev, void *stream);
/* KernelOperator2D.apply / apply_transpose (kernel2d.py:70-90) on device
 * buffers with shift grids a_dev, b_dev (both NULL: the plain kernel). */
int finom_apply2d(finom_grid *grid, const double *in_dev, double *out_dev, int transpose,
                  const double *a_dev, const double *b_dev, void *stream);
/* The adapter protocol (solver.py:1-16) on a grid: set_shifts = the state
 * after _GridAdapter.absorb (kernel2d.py:355-360; both NULL: the plain
 * kernel), iterate2d = _GridAdapter.iterate (kernel2d.py:343-353) in place
 * with res_dev = (err, status, psmax, psmin, phmax, phmin). */
int finom_grid_set_shifts(finom_grid *grid, const double *a_dev, const double *b_dev,
                          void *stream);
int finom_iterate2d(finom_grid *grid, const double *U_dev, const double *V_dev, double *phi_dev,
                    double *psi_dev, double *res_dev, void *stream);

/* ---- Dense realizations / plans on the device (small sizes) ----
 * finom_dense1d: out (n x m, row-major) = kernel1d.dense_realization
 * (kernel1d.py:328-338), exp(((-|x_i - y_j| + a_i) + b_j) / eps) with
 * a_dev / b_dev nullable (zero); with phi_dev / psi_dev (both or neither) the
 * transport plan of solver.plan_dense (solver.py:240-249),
 * (phi_i * K'_ij) * psi_j.  finom_dense2d: the same for grids
 * (kernel2d.dense_realization_2d, kernel2d.py:278-290), (n1 m1) x (n2 m2)
 * over the flat column-major grid vectors. */
int finom_dense1d(int64_t n, int64_t m, const double *x_dev, const double *y_dev,
                  const double *a_dev, const double *b_dev, double eps, const double *phi_dev,
                  const double *psi_dev, double *out_dev, void *stream);
int finom_dense2d(int64_t n1, int64_t m1, int64_t n2, int64_t m2, const double *x1_dev,
                  const double *y1_dev, const double *x2_dev, const double *y2_dev,
                  const double *a_dev, const double *b_dev, double eps, const double *phi_dev,
                  const double *psi_dev, double *out_dev, void *stream);

/* ---- Distributed 1D scan (BASELINE north star; no reference equivalent) ----
 * One 1D problem split into R segments of the merged order x U y (merge-path
 * splits at diagonals r (n+m) / R, ties never split), one per rank.  The
 * caller drives run_driver and the collectives
 * (paper_2605_26659_b200.sharding.sinkhorn_1d_segmented): per half,
 * finom_seg1d_pre writes the segment's totals of both recurrences
 * (_kernels.py:53-88; 10 doubles), the caller all-gathers them ([R][10]),
 * finom_seg1d_finish composes the other segments' totals into the segment's
 * incoming states, computes its rows and their scaling update, and writes
 * its partials (err, max, min, status or -1) for a rank-order combine.
 * Data arrays (weights, scalings, shifts) are whole-length on every rank.
 * half 0 = psi <- v / K'^T phi, half 1 = phi <- u / K' psi. */
typedef struct finom_seg1d finom_seg1d;
/* bounds: 2 (R + 1) int64, the split points (i_k, j_k), k = 0..R (host only) */
int finom_seg1d_split(int64_t n, const double *x, int64_t m, const double *y, int64_t R,
                      int64_t *bounds);
int finom_seg1d_create(int64_t n, const double *x_host, int64_t m, const double *y_host,
                       double eps, int64_t R, int64_t r, void *stream, finom_seg1d **out);
int finom_seg1d_destroy(finom_seg1d *seg);
/* w4: the segment's windows x [w0, w1), y [w2, w3) */
int finom_seg1d_window(const finom_seg1d *seg, int64_t *w4);
int finom_seg1d_pre(finom_seg1d *seg, int half, const double *in_dev, const double *a_dev,
                    const double *b_dev, double *tot_out_dev, void *stream);
int finom_seg1d_finish(finom_seg1d *seg, int half, const double *in_dev, const double *a_dev,
                       const double *b_dev, const double *tot_all_dev, const double *W_dev,
                       double *SC_dev, double *part_out_dev, void *stream);
/* shift += _shift(W, SC) (solver.py:135-153) over the whole vector; SC all
 * scalings, prv / nxt the previous / next positive-mass index of W */
int finom_seg1d_absorb(finom_seg1d *seg, int side, double *shift_dev, const double *W_dev,
                       const double *SC_dev, const int32_t *prv_dev, const int32_t *nxt_dev,
                       void *stream);
/* run_driver's decisions (solver.py:173-198) of a distributed-scan iteration
 * on the device, as finom_grid2d_decide (ctl, hist, absorb_its the same),
 * with the segments' partials (err, max, min, status or -1) combined in rank
 * order and the LAST failing segment's status reported (the reference's
 * loops run downward). */
int finom_seg1d_decide(const double *parts_a, const double *parts_b, int R, int64_t *ctl,
                       double *hist, int64_t *absorb_its, int64_t itr_max, double tol,
                       int stabilize, double absorb_threshold, void *stream);

/* ---- Row-sharded 2D grids (no reference equivalent) ----
 * One handle per rank for source == target grids x[n] x (y1[m1] | y2[m2]),
 * rank holding grid rows [k0, k1).  The caller drives run_driver's loop
 * and the collectives (paper_2605_26659_b200.sharding.sinkhorn_2d_row_sharded):
 * per half, finom_grid2d_xpre writes this shard's segment totals of the x
 * sweep (10 doubles per line), the caller all-gathers them ([R][line][10]),
 * finom_grid2d_finish completes the half and writes the shard's partials
 * (err, max, min, failure code) for an all-reduce.  Local grids are
 * column-major (k1 - k0) x m. */
typedef struct finom_grid2d finom_grid2d;
int finom_grid2d_create(int64_t n, const double *x, int64_t m1, const double *y1, int64_t m2,
                        const double *y2, double eps, int64_t k0, int64_t k1, finom_grid2d **out);
int finom_grid2d_destroy(finom_grid2d *g);
int finom_grid2d_set_shifts(finom_grid2d *g, const double *A, const double *B, void *stream);
int finom_grid2d_xpre(finom_grid2d *g, int half, const double *in, const double *shift, int dyn,
                      double *seg_out, void *stream);
int finom_grid2d_finish(finom_grid2d *g, int half, const double *in, const double *A,
                        const double *B, int dyn, const double *seg_all, int R, int r,
                        const double *W, double *SC, double *part_out, void *stream);
int finom_grid2d_absorb(finom_grid2d *g, int side, double *shift, const double *W,
                        const double *SC_all, const int32_t *prv, const int32_t *nxt, int R, int r,
                        void *stream);
/* Neighbour-only absorption exchange (replaces the all-gather of the whole
 * scaling grids for finom_grid2d_absorb): solver._shift's np.interp fill
 * (solver.py:135-153) reaches into another shard only at the last / first
 * positive-mass point of that shard's segment of a column.
 * finom_grid2d_edges writes this shard's m x 2 scalings at those points
 * (lastpos / firstpos: local indices, -1 if the segment has no mass); the
 * caller all-gathers them ([R][m][2]); finom_grid2d_absorb_nb updates the
 * shift grid: prv_src / nxt_src per local point (>= 0 local index, <= -2
 * segment -2 - src of the gathered edges, -1 none), prv_g / nxt_g the
 * neighbours' flat indices in the whole grid. */
int finom_grid2d_edges(finom_grid2d *g, const double *SC, const int32_t *lastpos,
                       const int32_t *firstpos, int m, double *edges_out, void *stream);
int finom_grid2d_absorb_nb(finom_grid2d *g, int side, double *shift, const double *W,
                           const double *SC, const int32_t *prv_src, const int32_t *nxt_src,
                           const int32_t *prv_g, const int32_t *nxt_g, const double *edges_all,
                           void *stream);
/* run_driver's decisions (solver.py:173-198) of a row-sharded iteration on
 * the device: the all-gathered partials of both halves ([R][4] each, as
 * finom_grid2d_finish writes them) combined in rank order; ctl (8 int64,
 * zeroed before the loop): it, status, converged, absorb this iteration,
 * done, n_absorb, failure code. */
int finom_grid2d_decide(const double *parts_a, const double *parts_b, int R, int64_t *ctl,
                        double *hist, int64_t *absorb_its, int64_t itr_max, double tol,
                        int stabilize, double threshold, void *stream);

#ifdef __cplusplus
}
#endif
#endif
