/*
 * pdot.h — C ABI of the B200-native PDOT restarted-PDHG solver (libpdot.so).
 *
 * This is the drop-in boundary for the reference's iteration path
 * (otsolve.solve, /root/reference/pkg/src/otsolve/pdhg.py:254-399) and for the
 * unit entry points the reference tests call directly.  Plain pointers and
 * sizes only: every matrix is row-major fp64 with an explicit, EVEN leading
 * dimension and a 16-byte aligned base; "dev" pointers are CUDA device
 * pointers, "any" pointers may be host or device (copied with UVA).
 *
 * Every function returns 0 on success or a negative PDOT_E* status; the
 * message of the last failure on the calling thread is pdot_last_error().
 * The Python host (paper_2407_19689_b200) maps statuses to the reference's
 * exception types:
 *   PDOT_EINVAL      -> ValueError   (pdhg.py:61-75, kkt.py:66-67)
 *   PDOT_ENONFINITE  -> RuntimeError("numerical failure: non-finite iterate")      pdhg.py:321
 *   PDOT_ELINESEARCH -> RuntimeError("step-size line search failed to find an admissible eta")  pdhg.py:251
 *   PDOT_ECUDA / PDOT_ENCCL -> RuntimeError
 */
#ifndef PDOT_H_
#define PDOT_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PDOT_OK 0
#define PDOT_EINVAL (-1)
#define PDOT_ECUDA (-2)
#define PDOT_ENONFINITE (-3)
#define PDOT_ELINESEARCH (-4)
#define PDOT_ENCCL (-5)
#define PDOT_ESTATE (-6)

/* termination reasons (SolveReport.termination_reason, reports.py:78) */
#define PDOT_REASON_NONE 0
#define PDOT_REASON_TOLERANCE 1
#define PDOT_REASON_ITERATION_LIMIT 2
#define PDOT_REASON_TIME_LIMIT 3

/* trace event types (SolveTrace, pdhg.py:106-118) */
#define PDOT_EV_START 1   /* x = initial metric, y = initial relative KKT */
#define PDOT_EV_ACCEPT 2  /* x = eta, y = step bound  (trace.etas / trace.step_bounds) */
#define PDOT_EV_CAND 3    /* x = candidate KKT (trace.candidate_kkts), y = current, z = average; ia = 1 if current won */
#define PDOT_EV_RESTART 4 /* ia = inner length, x = candidate KKT, y = omega after update */
#define PDOT_EV_REJECT 5  /* x = rejected eta, y = bound */

typedef struct pdot_solver pdot_solver; /* opaque handle: one problem shape on one GPU */

/* SolverConfig, pdhg.py:43-75 (restart_mode -> adaptive, kkt_mode -> relative). */
typedef struct {
  double tol;
  double time_limit_s;
  double beta;
  double beta_sufficient;
  double beta_necessary;
  double beta_artificial;
  double theta;
  double eps_zero;
  int64_t max_iters;
  int64_t kkt_stride;
  int32_t adaptive;    /* 1: "adaptive", 0: "fixed" */
  int32_t relative;    /* 1: "relative", 0: "absolute" */
  double eta0;         /* <= 0: default 1/(2 sqrt(m+n)), pdhg.py:225-227 */
  double omega0;
  int32_t trace_level; /* 0: restarts only, 1: + etas/bounds/candidates, 2: + rejections */
  int32_t poll_passes; /* passes per CUDA-graph batch (0: automatic) */
  int32_t host_omega;  /* 1: the primal weight of an adaptive restart is evaluated on the host
                          with libm exp/log, the functions math.exp / math.log call
                          (pdhg.py:185): the device pauses at the restart, the host
                          evaluates omega and the device resumes.  0: device exp/log. */
  int32_t reserved;
} pdot_config;

typedef struct {
  int32_t reason;         /* PDOT_REASON_* */
  int32_t final_slot;
  int64_t iterations;     /* accepted steps, SolveReport.iterations */
  int64_t restarts;       /* SolveReport.restarts */
  int64_t passes;         /* streaming passes (accepted + rejected + restart + start) */
  int64_t rejected;       /* line-search rejections */
  double final_relative_kkt;
  double eta, omega, scale_R;
  double elapsed_s;       /* wall time of the loop, same scope as pdhg.py:268-380 */
  double device_s;        /* CUDA-event time of the graph replays on the solver stream */
} pdot_result;

typedef struct {
  int32_t type;
  int32_t ia;
  double x, y, z;
} pdot_event;

const char* pdot_last_error(void);
int pdot_version(void);

/* ---- handle lifecycle (replaces the Python state of pdhg.py:269-297) ---- */
int pdot_create(int64_t m, int64_t n, int device, pdot_solver** out);
int pdot_destroy(pdot_solver* h);
int pdot_geometry(const pdot_solver* h, int64_t* ldx, int64_t* row_tile, int64_t* n_row_tiles,
                  int64_t* n_col_tiles);
/* Bind the problem (OTProblem accessors C, f, g, cost_fro_norm, marginal_norm,
 * instance.py:122-150).  C/f/g are borrowed device buffers that must outlive
 * the handle; ldc must be even. */
int pdot_set_problem(pdot_solver* h, const double* C_dev, int64_t ldc, const double* f_dev,
                     const double* g_dev, double cost_fro_norm, double marginal_norm);
/* Matrix-free variant: C_ij is generated in registers from
 * grid coordinates (kind/a as in pdot_gen_cost) instead of being streamed from
 * HBM -- 32 instead of 40 bytes per plan entry per pass, and no m x n cost
 * buffer at all.  The generated values are exact integers, so results are
 * bit-identical to binding the explicit matrix. */
int pdot_set_problem_implicit(pdot_solver* h, int kind, const int64_t* a, const double* f_dev,
                              const double* g_dev, double cost_fro_norm, double marginal_norm);
/* Load (X, p, q) into slot `slot` (0..5).  X_any may be NULL for zeros. */
int pdot_set_slot(pdot_solver* h, int slot, const double* X_any, int64_t ldX, const double* p_any,
                  const double* q_any);
/* Copy slot `slot` out (any of the pointers may be NULL). */
int pdot_get_slot(pdot_solver* h, int slot, double* X_any, int64_t ldX, double* p_any,
                  double* q_any);
/* Copy slot `slot` out moving only its occupied 8 x 16 cells (screened handles,
 * where every other cell is exactly +0.0 on the device): X_host must be
 * zero-filled by the caller (e.g. calloc / np.zeros).  *cells_out = cells moved.
 * PDOT_ESTATE when screening is off. */
int pdot_get_slot_sparse(pdot_solver* h, int slot, double* X_host, int64_t ldX, double* p_any, double* q_any,
                         int64_t* cells_out);
/* Device pointers of a slot's buffers (X has leading dimension ldx). */
int pdot_slot_ptrs(pdot_solver* h, int slot, double** X, double** p, double** q);

/* ---- the solve loop: otsolve.solve (pdhg.py:254-399), starting from slot 0 ---- */
/* pdot_solve = pdot_begin + pdot_advance(-1) + pdot_finish. */
int pdot_solve(pdot_solver* h, const pdot_config* cfg, double elapsed_before_s, pdot_result* res);

typedef struct {
  int32_t done;
  int32_t roles[4];  /* slots holding: current iterate, running average, restart anchor, best */
  int32_t op;        /* next pass: 0 step, 1 restart distance, 2 start KKT */
  int64_t iterations, restarts, passes;
  int32_t avg_written; /* the pass just run wrote the running-average matrix of the last */
  int32_t avg_slot;    /* accepted iterate into slot avg_slot (it is computed one pass late) */
} pdot_progress;

/* Validate cfg (pdhg.py:61-75), load the control block; slot 0 holds the start point. */
int pdot_begin(pdot_solver* h, const pdot_config* cfg, double elapsed_before_s);
/* Run `max_passes` passes one by one (synchronously), or, with max_passes < 0,
 * replay the CUDA-graph batches until the device controller reports done. */
int pdot_advance(pdot_solver* h, int64_t max_passes, pdot_progress* prog);
/* Collect the result of a finished run (maps device errors to PDOT_E* codes). */
int pdot_finish(pdot_solver* h, pdot_result* res);
/* Resume a finished/limited run with a new iteration limit (benchmarking). */
int pdot_resume(pdot_solver* h, int64_t max_iters, pdot_result* res);
/* Drain recorded trace events (returns the count copied, <= cap). */
int64_t pdot_get_events(pdot_solver* h, pdot_event* out, int64_t cap);

/* ---- rounding: round_to_feasible (rounding.py:18-40) + <C, X_feas> ---- */
/* Rounds slot `slot`; writes X_feas to Xf_any (ld ldX) unless NULL.
 * out3 = {rounded objective <C,X_feas>, f.p + g.q of the slot, l1 marginal violation of X_feas}. */
int pdot_round(pdot_solver* h, int slot, double* Xf_any, int64_t ldX, double* out3);

/* ---- unit entry points on slot 0 (input) / slot 1 (second input or output) ---- */
/* pdhg_step (pdhg.py:121-129): slot0 -> slot1.  With k > 0 the running-average
 * update of pdhg.py:314-317 is applied too: slot2 (average) -> slot3 with
 * A' = A + (X+ - A)/k (and the same for p, q). */
int pdot_unit_step(pdot_solver* h, double tau, double sigma, double k);
/* stepsize_bound (pdhg.py:132-149) for (slot0 -> slot1); out5 = {bound, |dX|^2, |dp|^2, |dq|^2, coupling} */
int pdot_unit_bound(pdot_solver* h, double omega, double eps_zero, double* out5);
/* kkt_error (kkt.py:56-94) of slot0; viol_any (ld ldV) receives the dual-violation matrix unless NULL;
 * out10 = {gap, composite, relative, pobj, dobj, primal_sq, dual_sq, |X|^2, |p|^2, |q|^2};
 * rows/cols (any, may be NULL) receive X 1 and X^T 1. */
int pdot_unit_kkt(pdot_solver* h, double scale_R, double* viol_any, int64_t ldV, double* rows_any,
                  double* cols_any, double* out10);
/* apply_A (operator.py:36-38) of slot0's X */
int pdot_unit_apply_A(pdot_solver* h, double* rows_any, double* cols_any);
/* apply_At (operator.py:41-43): out[i*ldo + j] = p[i] + q[j] (device pointers) */
int pdot_apply_At(const double* p_dev, const double* q_dev, int64_t m, int64_t n, double* out_dev,
                  int64_t ldo);

/* ---- row sharding over GPUs ----
 * Rows are split in whole groups of the 8-group reduction tree (1, 2, 4 or 8
 * shards; the number of 128-row tiles must be a multiple of 8), so every GPU
 * count reproduces the single-GPU reduction order bit for bit.  Per pass each
 * shard reduces its groups' column partials and scalars, one all-gather
 * (NCCL over NVLink) exchanges them, and every shard runs the identical
 * combine + controller.  Shard handles bind their row slices of C and f (and
 * the full g); everything else (p, the averages, ...) is local to the rows. */
int pdot_shard_rows(int64_t m_total, int64_t n, int nranks, int rank, int64_t* row0, int64_t* row1);
int pdot_create_shard(int64_t m_total, int64_t n, int nranks, int rank, int device, pdot_solver** out);
int pdot_shard_info(const pdot_solver* h, int64_t* m_total, int64_t* row0, int32_t* nranks, int32_t* rank);
/* NCCL communicator: rank 0 creates the 128-byte id, the host broadcasts it. */
int pdot_nccl_unique_id(void* out128);
int pdot_comm_init(pdot_solver* h, const void* id128);
/* Single-GPU emulation of a sharded run (tests): the host steps every shard
 * through phase 0 (stream + group partials), pdot_exchange_local, phase 1
 * (combine + controller). */
int pdot_set_virtual(pdot_solver* h, int on);
/* Peer-memory exchange instead of NCCL: the finalize kernel stores its group
 * partials straight into every rank's exchange buffer over NVLink and publishes
 * a sequence flag; the combine kernel acquires every rank's flag (bounded spin,
 * PDOT_ENCCL after 20 s).  Ranks share their buffers through CUDA IPC handles
 * (64 bytes each, exchanged by the host); single-GPU emulation links handles. */
int pdot_ipc_handle(pdot_solver* h, void* out64);
int pdot_p2p_open(pdot_solver* h, const void* handles64, int count);
int pdot_p2p_link_local(pdot_solver** hs, int count);
/* device time (ms) of the last pdot_shard_pass call of phase 0 (K0/K1/K1b/K2a) and 1 (K2b) */
int pdot_shard_pass_ms(const pdot_solver* h, double* ms2);
/* Test hook: the peer-exchange protocol (group stores into every rank's buffer,
 * st.release of the sequence flags, ld.acquire spin, parity double buffering)
 * with `count` linked ranks emulated as the blocks of ONE cooperative launch,
 * so the ranks run concurrently and the spins really wait.  out3r[3r + 0..2] =
 * rank r's value mismatches, longest wait in ns, exchange-timeout flag. */
int pdot_p2p_selftest(pdot_solver** hs, int count, int rounds, double delay_us, unsigned long long* out3r);
int pdot_shard_pass(pdot_solver* h, int phase, pdot_progress* prog);
int pdot_exchange_local(pdot_solver** hs, int count);

/* ---- log-domain Sinkhorn baseline (sinkhorn.py:58-130) ----
 * Runs on the bound explicit cost; leaves the plan exp((phi+psi-C)/eps) in
 * slot 0's X and the potentials (phi, psi) in slot 0's (p, q).  res->reason
 * and res->iterations follow the reference's loop. */
typedef struct {
  double penalty;
  double tol;
  int64_t max_iters;
  double time_limit_s;
  int32_t poll_iters;  /* iterations per host poll (0: 16) */
} pdot_sinkhorn_config;
int pdot_sinkhorn_solve(pdot_solver* h, const pdot_sinkhorn_config* cfg, double elapsed_before_s,
                        pdot_result* res);

/* ---- instance generation on the device ---- */
#define PDOT_COST_SQEUCLID_GRID 0 /* a = (r, r): (di^2 + dj^2) on an r x r grid   */
#define PDOT_COST_L1_GRID 1       /* a = (r, r): |di| + |dj|                      */
#define PDOT_COST_L1_RECT 2       /* a = (sr, sc, tr, tc): |2 a_i - c_j| + |2 b_i - d_j| */
int pdot_gen_cost(double* C_dev, int64_t m, int64_t n, int64_t ldc, int kind, const int64_t* a);
/* rows [row0, row0 + rows) of the same matrix (a row shard) */
int pdot_gen_cost_rows(double* C_dev, int64_t row0, int64_t rows, int64_t n, int64_t ldc, int kind,
                       const int64_t* a);
/* ||C||_F on the device (deterministic): used for OTProblem.cost_fro_norm of device-built C */
/* Host -> device copy of an m x n row-major matrix (cost upload of
 * solve(host problem), pdhg.py:254-259 takes plain arrays): one DMA from
 * page-locked memory; pageable memory is staged through two pinned 64 MB
 * buffers, host threads filling one while the other is DMA'd. */
int pdot_h2d_matrix(double* dst_dev, int64_t ldd, const double* src_host, int64_t lds, int64_t m, int64_t n,
                    int device);
int pdot_fro_norm(const double* C_dev, int64_t m, int64_t n, int64_t ldc, double* out);

/* ---- measurement helpers (bench.py) ---- */
/* Launch the streaming STEP kernel `iters` times on the current state (no
 * controller) and time it with CUDA events on the kernel's stream. */
int pdot_time_stream_kernel(pdot_solver* h, int iters, double* ms_per_launch);
/* Time the finalize kernel alone (OP_STEP reductions + vector updates, no controller decisions). */
int pdot_time_finalize(pdot_solver* h, int iters, double* ms_per_launch);
/* Number of kernels launched so far by this handle (graph nodes count individually). */
int64_t pdot_kernel_launches(const pdot_solver* h);

/* ---- block screening of the STEP pass (csrc/screen.cu) ----
 * Same results bit for bit (pdhg.py:121-129 / kkt.py:56-94 arithmetic is
 * unchanged); the pass only skips 8 x 16 cells whose every output and every
 * reduction term is exactly +0.  On by default from 2^22 plan entries
 * (PDOT_SCREEN=0/1 forces it for new handles); toggling rebuilds the min-C
 * table and rescans the slots. */
int pdot_set_screening(pdot_solver* h, int on);
/* Counters since the last reset: out12 = {screened STEP passes, active cells,
 * cells visited, bytes moved by K1, K0 metadata bytes, summed K1 ns
 * (%globaltimer), screening on, cells per plan, summed K2 ns up to the last
 * block, summed K2 controller-tail ns, controller reduce / decide / publish ns}. */
int pdot_screen_stats(pdot_solver* h, int reset, unsigned long long* out20);

#ifdef __cplusplus
}
#endif
#endif /* PDOT_H_ */
