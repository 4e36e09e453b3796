/* docp_cuda.h — C ABI of the B200-native DiffMPC hot path (libdocp_cuda.so).
 *
 * The drop-in boundary for the reference's solver/operator API
 * (/root/reference/proj/include/docp, namespace docp). The reference is a
 * header-only C++ library whose "FFI" is its free functions on value types;
 * every entry point below replaces one of them for a whole BATCH of
 * independent problems that live on one GPU:
 *
 *   docp_linearize        <- docp::linearize        problem.hpp:202-257
 *   docp_assemble_schur   <- docp::assemble_schur   schur.hpp:114-180
 *   docp_assemble_gamma   <- docp::assemble_gamma   schur.hpp:187-211
 *   docp_pcg_solve        <- docp::pcg_solve        pcg.hpp:52-109
 *   docp_recover_primal   <- docp::recover_primal   sqp.hpp:62-89
 *   docp_line_search      <- docp::line_search      sqp.hpp:151-206
 *   docp_kkt_residual     <- docp::kkt_residual     problem.hpp:263-300 (inf-norm)
 *   docp_sqp_solve        <- docp::sqp_solve        sqp.hpp:213-261
 *                            (and docp::batch_solve batch.hpp:83-108 when the
 *                             Z/LAMBDA fields hold the warm-start cache)
 *   docp_backward_vjp     <- docp::backward_vjp     backward.hpp:27-50
 *   docp_il_epoch         <- the train_il epoch body train.hpp:82-131
 *   docp_rollout          <- docp::rollout          batch.hpp:172-212 (affine env, train.hpp:195-213)
 *   docp_rollout_backward <- docp::rollout_backward batch.hpp:221-258
 *   docp_pcg_invocations  <- docp::stats::pcg_invocations common.hpp:112-115
 *
 * Callbacks (OcpDefinition's std::functions, problem.hpp:43-54) cannot cross
 * to the device, so a problem is described by a family tag plus its packed
 * theta (docp_problem). Errors never cross the ABI as exceptions: host-side
 * failures return a docp_code, per-problem solver failures are status words
 * (docp_status) that the host wrapper re-raises as the matching docp::Error
 * with the reference's message (docp_format_status).
 *
 * Layouts (fp64, per problem, problems contiguous):
 *   THETA   family layout (affine_quadratic.hpp:27-37, cartpole.hpp:82-89,
 *           attitude.hpp:44-53 + the instance inertia, see DOCP_ATTITUDE)
 *   Z       flat interleaved (x_0,u_0,...,x_{T-1},u_{T-1},x_T)  trajectory.hpp:7-39
 *   LAMBDA  n_x*(T+1)
 * Schur blocks move through docp_batch_{upload,download}_schur in the
 * reference's dense column-major layout; on the device they live in the
 * swizzled block layout described in DESIGN.md.
 *
 * Threading: a docp_batch is used from one host thread at a time; calls on
 * different batches are independent. All compute calls are asynchronous on
 * the batch's stream except where noted (sqp_solve reads the active-problem
 * count once per SQP iteration).
 */
#ifndef DOCP_CUDA_H
#define DOCP_CUDA_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define DOCP_ABI_VERSION 1

/* DOCP_ATTITUDE (attitude.hpp): n_x = n_u = 3, cost scale 0.5, dt from
 * docp_problem.dt. Its per-instance AttitudeParams::inertia rides in THETA's
 * tail: THETA = [w_x 3 | w_u 3 | omega_0 3 | inertia 3] (the reference's 9
 * entries, make_attitude_theta, then the inertia); GRAD_THETA's inertia tail is 0. */
/* DOCP_DRIFT (include/docp_drift_model.h; no reference implementation exists,
 * SURVEY.md §8(f)5): dynamic bicycle with Fiala tires, n_x = 8, n_u = 2, cost
 * scale 0.5, Heun steps over docp_problem.dt; THETA = [w_x 8 | w_u 2 |
 * xbar_0 8 | X_ref 8 | vehicle parameters 10] (36); GRAD_THETA covers the first
 * 18 entries (make_quadratic_cost_theta_vjp), the tail is 0. */
enum docp_family { DOCP_AFFINE_QUADRATIC = 1, DOCP_CARTPOLE = 2, DOCP_ATTITUDE = 3, DOCP_DRIFT = 4 };

/* docp::Error hierarchy (common.hpp:18-54) plus ABI-level failures. */
enum docp_code {
  DOCP_OK = 0,
  DOCP_DIMENSION = 1,  /* DimensionError  */
  DOCP_EVALUATION = 2, /* EvaluationError */
  DOCP_NUMERICAL = 3,  /* NumericalError  */
  DOCP_BREAKDOWN = 4,  /* BreakdownError  */
  DOCP_DIVERGENCE = 5, /* DivergenceError */
  DOCP_UNSUPPORTED = 6,
  DOCP_CUDA_ERROR = 7,
  DOCP_INVALID = 8
};

/* Where a per-problem failure happened (selects the reference message). */
enum docp_where {
  DOCP_AT_NONE = 0,
  DOCP_AT_STATE_COST = 1,    /* problem.hpp:223-225 */
  DOCP_AT_CONTROL_COST = 2,  /* problem.hpp:233-235 */
  DOCP_AT_DYNAMICS = 3,      /* problem.hpp:243-246 */
  DOCP_AT_INITIAL_STATE = 4, /* problem.hpp:254 */
  DOCP_AT_CHOL_Q = 5,        /* schur.hpp:99-107 */
  DOCP_AT_CHOL_R = 6,
  DOCP_AT_CHOL_CHI = 7,
  DOCP_AT_PCG_CURVATURE = 8, /* pcg.hpp:88-93 */
  DOCP_AT_PCG_PRECOND = 9,   /* pcg.hpp:72-79 */
  DOCP_AT_MERIT_STATE = 10,  /* sqp.hpp:104-106 */
  DOCP_AT_MERIT_CONTROL = 11,
  DOCP_AT_SQP_ITERATE = 12,  /* sqp.hpp:240-243 */
  DOCP_AT_INITIAL_GUESS = 13, /* sqp.hpp:220-221 */
  DOCP_AT_ROLLOUT_ENV = 14    /* batch.hpp:195-199: environment produced a non-finite state at step index */
};

typedef struct docp_status {
  int32_t code;  /* docp_code */
  int32_t where; /* docp_where */
  int32_t index; /* stage, PCG iteration (BreakdownError::iteration) or SQP iteration */
  int32_t step;  /* rollout statuses: 1 + the episode step a solve failed at (RolloutTruncation,
                    batch.hpp:186-191; formatted as "rollout: solve failed at step k: ..."), else 0 */
} docp_status;

typedef struct docp_problem {
  int32_t family; /* docp_family */
  int32_t n_x, n_u, horizon;
  double cost_scale;                             /* affine-quadratic (affine_quadratic.hpp:25) */
  double cart_mass, pole_mass, length, gravity;  /* cart-pole (cartpole.hpp:17-26) */
  double dt;                                     /* cart-pole, attitude and drift time step */
} docp_problem;

/* PCG arithmetic: PARITY reproduces the reference's operation order
 * (sequential folds, no FMA) bit for bit; FAST uses FMA and tree reductions. */
/* FAST: fp64, FMA and tree reductions inside K2 (<= 1e-9 of the reference).
 * PARITY: fp64, the reference's operation order bit for bit.
 * FP32: K2 on fp32 blocks and iterates (dots and scalars fp64), n_x = 8;
 *       K1/K3/K4 stay fp64. epsilon is RELATIVE in this mode: the solve stops
 *       at eta <= epsilon^2 * gamma' Phi^-1 gamma (an absolute 1e-12 is below
 *       fp32 resolution). Stated bound: z, lambda, lambda~ and the theta-
 *       gradient within 1e-4 relative of the fp64 reference at epsilon = 1e-6. */
enum docp_pcg_mode { DOCP_PCG_FAST = 0, DOCP_PCG_PARITY = 1, DOCP_PCG_FP32 = 2 };

typedef struct docp_pcg_config { /* PcgConfig, pcg.hpp:7-23 */
  double epsilon;                /* exit when eta = r'r~ <= epsilon^2 */
  int32_t max_iters;             /* 0 -> 2 * n_x * (T+1) */
  int32_t mode;                  /* docp_pcg_mode */
} docp_pcg_config;

#define DOCP_MAX_STEP_CANDIDATES 8
typedef struct docp_sqp_config { /* SqpConfig, sqp.hpp:7-34 */
  int32_t max_sqp_iters;
  int32_t n_step_candidates;
  double step_candidates[DOCP_MAX_STEP_CANDIDATES];
  double eta_armijo;
  double rho_penalty;
  docp_pcg_config pcg;
  double convergence_tol;
  double mu_floor_denominator;
  double eps_pd;
} docp_sqp_config;

/* Per-problem device-resident fields of a batch. */
enum docp_field {
  DOCP_F_THETA = 0,        /* [B][n_theta]  in */
  DOCP_F_Z = 1,            /* [B][n_z]      initial guess in, solution out */
  DOCP_F_LAMBDA = 2,       /* [B][n_lambda] warm start in, multiplier out */
  DOCP_F_LAMBDA_TILDE = 3, /* [B][n_lambda] adjoint warm start in / out */
  DOCP_F_LOSS_GRAD_Z = 4,  /* [B][n_z]      backward cotangent in */
  DOCP_F_GRAD_THETA = 5,   /* [B][n_theta]  backward out */
  DOCP_F_GAMMA = 6,        /* [B][n_lambda] stored right-hand side (-gamma) */
  DOCP_F_Z_QP = 7,         /* [B][n_z]      recovered QP primal / adjoint z~ */
  DOCP_F_STATUS = 8,       /* [B] docp_status */
  DOCP_F_SQP_ITERS = 9,    /* [B] int32 */
  DOCP_F_CONVERGED = 10,   /* [B] int32 (sqp converged) */
  DOCP_F_KKT = 11,         /* [B] double, ||kkt_residual||_inf at the returned point */
  DOCP_F_PCG_ITERS = 12,   /* [B] int32, iterations of the last pcg solve */
  DOCP_F_PCG_CONVERGED = 13, /* [B] int32 */
  DOCP_F_FINAL_ETA = 14,   /* [B] double */
  DOCP_F_PCG_HISTORY = 15, /* [B][max_sqp_iters] int32, per-SQP-iteration pcg iterations */
  DOCP_F_STEP_SIZES = 16,  /* [B][max_sqp_iters] double, accepted alpha */
  DOCP_F_PD_PROJECTED = 17,/* [B] int32 */
  DOCP_F_MU = 18,          /* [B] double, merit penalty threaded through SQP */
  DOCP_F_ALPHA = 19,       /* [B] double, last line-search alpha */
  DOCP_F_ACCEPTED = 20,    /* [B] int32, last line-search accepted flag */
  DOCP_F_LOSS = 21,        /* [B] double, per-instance IL loss */
  DOCP_F_ROLLOUT_STATUS = 22, /* [B] docp_status of the last rollout (+ its backward) */
  DOCP_F_REWARD = 23,      /* [B] double, total reward of the last rollout */
  DOCP_F_COUNT = 24
};

typedef struct docp_batch docp_batch;

/* ---- lifecycle ---------------------------------------------------------- */
int docp_abi_version(void);
int docp_theta_size(const docp_problem* problem);
int docp_batch_create(const docp_problem* problem, int32_t batch_size, int32_t device, docp_batch** out);
void docp_batch_destroy(docp_batch* batch);
/* stream: a cudaStream_t (NULL = the legacy default stream). */
int docp_batch_set_stream(docp_batch* batch, void* stream);
int docp_batch_sync(docp_batch* batch);
int32_t docp_batch_size(const docp_batch* batch);

/* ---- data movement (host <-> device are synchronous on the batch stream) -- */
int docp_batch_field_ptr(docp_batch* batch, int32_t field, void** device_ptr, size_t* bytes);
int docp_batch_upload(docp_batch* batch, int32_t field, const void* src, int32_t src_on_device);
int docp_batch_download(docp_batch* batch, int32_t field, void* dst, int32_t dst_on_device);
/* Blocks in the reference layout: column-major n_x*n_x, per problem
 * s_diag[T+1], s_sub[T] (block (i+1,i)), p_diag[T+1], p_super[T] (block (i,i+1)). */
int docp_batch_upload_schur(docp_batch* batch, const double* s_diag, const double* s_sub, const double* p_diag,
                            const double* p_super);
int docp_batch_download_schur(docp_batch* batch, double* s_diag, double* s_sub, double* p_diag, double* p_super);
/* QpData of the last linearize (problem.hpp:103-151), dense column-major
 * blocks: Q[T+1][nx*nx], q[T+1][nx], R[T][nu*nu], r[T][nu], A[T][nx*nx],
 * B[T][nx*nu], C[T][nx], x_s[nx]. A_plus is the identity for every family. */
int docp_batch_download_qp(docp_batch* batch, double* Q, double* q, double* R, double* r, double* A, double* B,
                           double* C, double* x_s);

/* ---- the hot path (asynchronous unless noted) ---------------------------- */
int docp_linearize(docp_batch* batch, double eps_pd);             /* Z, THETA -> QpData */
int docp_assemble_schur(docp_batch* batch);                        /* QpData -> -S, Phi^-1, factors */
enum docp_rhs { DOCP_RHS_FORWARD = 0, DOCP_RHS_ADJOINT = 1 };
/* FORWARD: b = flat_b, d = flat_d; ADJOINT: b = -LOSS_GRAD_Z, d = 0 (backward.hpp:38-40). */
int docp_assemble_gamma(docp_batch* batch, int32_t rhs);
/* (-S) x = GAMMA warm-started from `solution_field` (DOCP_F_LAMBDA or
 * DOCP_F_LAMBDA_TILDE), which receives the solution. */
int docp_pcg_solve(docp_batch* batch, const docp_pcg_config* cfg, int32_t solution_field);
/* Z_QP = recover_primal(lambda_field, rhs b of docp_rhs). */
int docp_recover_primal(docp_batch* batch, int32_t lambda_field, int32_t rhs);
/* Z <- line_search(Z, Z_QP) with MU in/out, ALPHA, ACCEPTED out. */
int docp_line_search(docp_batch* batch, const docp_sqp_config* cfg);
int docp_kkt_residual(docp_batch* batch); /* KKT <- ||F(Z, LAMBDA)||_inf */
/* Full forward pass; Z and LAMBDA hold the initial guess and receive the
 * solution; the final QpData/Schur system stay resident for backward.
 * The loop is enqueued without waiting on the device: every kernel reads the
 * active-problem count from device memory, and the host reads it back only
 * after SQP iterations 4, 8, 16, ... to stop early (one synchronization for
 * max_sqp_iters = 5). For the affine-quadratic family the -S / Phi^-1 blocks
 * depend on theta only, so they are assembled at the first iteration and kept
 * (bitwise the reference's re-assembly; DOCP_REASSEMBLE=1 forces it). */
int docp_sqp_solve(docp_batch* batch, const docp_sqp_config* cfg);
/* backward_vjp on the resident forward result: LOSS_GRAD_Z and the warm
 * LAMBDA_TILDE in; GRAD_THETA, LAMBDA_TILDE, PCG_ITERS out. */
int docp_backward_vjp(docp_batch* batch, const docp_pcg_config* cfg);

/* One imitation-learning epoch over the batch (train.hpp:82-131 for any
 * family): THETA's [learn_start, +learn_size) segment is overwritten with
 * `weights` (shared learnable parameters, device pointer) for every instance;
 * each solve starts from z0 = demos[j] (device, [B][n_z]) with LAMBDA as the
 * warm cache; loss_j = |u_j - u^_j|^2 / loss_denominator; backward
 * warm-started from LAMBDA_TILDE; then the fixed-order (instance order)
 * sums into loss_sum[1] and grad_sum[learn_size] (device pointers).
 * LAMBDA and LAMBDA_TILDE are left holding the updated caches. */
int docp_il_epoch(docp_batch* batch, const docp_sqp_config* cfg, const double* weights, int32_t learn_start,
                  int32_t learn_size, const double* demos, double loss_denominator, double* loss_sum,
                  double* grad_sum);
/* The reference fails an epoch on the first demonstration whose solve or
 * backward threw (train.hpp:111-119). docp_il_epoch never synchronizes, so
 * instead a failed demonstration contributes zero to both sums, and is
 * counted on the device. This call waits for the batch's stream, returns the
 * number of failed demonstrations in the epochs since the last call and the
 * smallest failed index (-1 if none), and resets both. STATUS holds the
 * failures of the last epoch (docp_format_status renders them). */
int docp_il_failures(docp_batch* batch, int32_t* n_failed, int32_t* first_failed);

/* Closed-loop MPC rollouts (batch.hpp:172-212) with the benchmark tasks'
 * environments: affine-quadratic instances step their own dynamics with
 * reward -(|x'|^2 + |u|^2) (make_affine_env, train.hpp:195-213); attitude
 * instances step attitude_step with reward -(0.1 |x'|^2 + |u|^2)
 * (make_attitude_rl_task, train.hpp:239-263). For each instance: the initial-state
 * segment of THETA is set to the current state, the problem is solved warm-
 * started from the previous step (Z, LAMBDA; zero at step 0), the first
 * control is applied, the reward accumulated. x_init: [B][n_x], on the device
 * when x_init_on_device != 0, else host memory (copied synchronously).
 * Per-instance truncations go to ROLLOUT_STATUS; REWARD receives the totals.
 * Every step's solution is recorded on the device for docp_rollout_backward. */
int docp_rollout(docp_batch* batch, const docp_sqp_config* cfg, const double* x_init, int32_t x_init_on_device,
                 int32_t episode_length);
/* rollout_backward (batch.hpp:221-258) of the last rollout: GRAD_THETA <-
 * dJ/dtheta of the total reward, its initial-state segment = dJ/dx_init.
 * The adjoint multiplier is chained across steps; instances whose rollout
 * was truncated are skipped (their ROLLOUT_STATUS is not OK). */
int docp_rollout_backward(docp_batch* batch, const docp_pcg_config* cfg);

/* ---- synthetic inputs (the reference generators' recipe, generators.hpp) -- */
/* count sequential random_convex_instance (convex != 0) / random_linear_instance
 * draws from mt19937_64(seed), as thetas ([count][n_theta], host memory). */
int docp_generate_affine_quadratic(int32_t n_x, int32_t n_u, uint64_t seed, int32_t count, int32_t convex,
                                   double* thetas);
int docp_generate_uniform(uint64_t seed, int32_t n, double lo, double hi, double* out);
/* pcg_study's drifting sequence (study.hpp:37-48, 74-124): random_convex_instance
 * from mt19937_64(seed), coefficients of A, B, b, x_s scaled by 1 + U(-m, m)
 * after every step; thetas [steps][n_theta]. */
int docp_generate_drift_sequence(int32_t n_x, int32_t n_u, uint64_t seed, int32_t steps, double magnitude,
                                 double* thetas);
/* gen_cartpole initial states (generators.hpp:142-152), [n][4]. */
int docp_generate_cartpole_x0(uint64_t seed, int32_t n, double* x0);

/* ---- profiling: CUDA events around every launch on the batch stream ------ */
enum docp_prof_kind {
  DOCP_PROF_ASSEMBLE = 0, DOCP_PROF_GAMMA = 1, DOCP_PROF_PCG = 2, DOCP_PROF_RECOVER = 3,
  DOCP_PROF_STEP = 4, DOCP_PROF_KKT = 5, DOCP_PROF_VJP = 6, DOCP_PROF_KINDS = 7
};
typedef struct docp_profile {
  int32_t launches[DOCP_PROF_KINDS];
  double ms[DOCP_PROF_KINDS];            /* summed launch durations */
  uint64_t pcg_iterations;               /* PCG iterations performed */
  uint64_t pcg_solves;                   /* PCG solves performed */
  double pcg_bytes_per_iteration;        /* B_it = 16 n_x^2 (2T+1) */
  double pcg_algorithmic_bytes;          /* (iterations + solves) B_it + solves 24 n_lambda */
  double span_ms;                        /* first profiled launch start -> last profiled launch end */
  double gap_ms;                         /* span minus the profiled launches (other ops, launch gaps) */
  double max_gap_ms;                     /* largest single gap between consecutive profiled launches */
  int32_t max_gap_after, max_gap_before; /* docp_prof_kind on either side of that gap */
} docp_profile;
int docp_profile_begin(docp_batch* batch);
int docp_profile_end(docp_batch* batch, docp_profile* out);

/* ---- diagnostics --------------------------------------------------------- */
uint64_t docp_pcg_invocations(void);      /* PCG system solves performed (one per problem per solve; counted on the device, synchronizes) */
uint64_t docp_kernel_launches(void);      /* kernels this library has launched */
const char* docp_last_error(void);        /* thread-local message of the last failing call */
/* Reference-style message for a per-problem status (e.g. "pcg: p'Sp <= 0 ...
 * at iteration 3"); returns the number of characters written. */
int docp_format_status(const docp_status* status, char* buffer, int32_t capacity);
/* Name of the device-block layout and PCG kernel variant chosen for a problem. */
int docp_describe(const docp_problem* problem, char* buffer, int32_t capacity);

#ifdef __cplusplus
}
#endif
#endif /* DOCP_CUDA_H */
