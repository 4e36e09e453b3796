/* docp_port — plain-C restatement of the reference hot path (TEST
 * INFRASTRUCTURE / ORACLE). Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline leg of bench.py may load this library, and only as the checker.
 *
 * Every routine follows a reference function (file:line under
 * /root/reference/proj/include/docp) and the eigen_lite arithmetic convention
 * (oracle/eigen_lite/Eigen/Dense header), so its results are bit-identical to
 * the reference headers compiled against eigen_lite (checked by
 * tests/test_oracle_port.py).
 *
 * Layouts (shared with the product C ABI, include/docp_cuda.h):
 *   z      flat interleaved (x_0,u_0,...,x_{T-1},u_{T-1},x_T)   trajectory.hpp:7-39
 *   lambda n_x*(T+1)
 *   theta  family layout (affine_quadratic.hpp:27-37, cartpole.hpp:82-89)
 *   matrices column-major, n x n, one block after another.
 */
#ifndef DOCP_PORT_H
#define DOCP_PORT_H

#ifdef __cplusplus
extern "C" {
#endif

enum { PORT_AFFINE_QUADRATIC = 1, PORT_CARTPOLE = 2, PORT_ATTITUDE = 3 /* ref build only */,
       PORT_DRIFT = 4 /* ref build only: the reference solver on include/docp_drift_model.h */ };
enum {
  PORT_OK = 0,
  PORT_DIMENSION = 1,
  PORT_EVALUATION = 2,
  PORT_NUMERICAL = 3,
  PORT_BREAKDOWN = 4,
  PORT_DIVERGENCE = 5
};

typedef struct {
  int family;
  int nx, nu, horizon;
  double cost_scale;                                   /* affine-quadratic */
  double cart_mass, pole_mass, length, gravity, dt;    /* cart-pole (dt: attitude too) */
  double inertia[3];                                   /* attitude (AttitudeParams, attitude.hpp:10-14) */
} port_problem;

typedef struct {
  int code;      /* PORT_* */
  int iteration; /* BreakdownError::iteration */
  char message[192];
} port_status;

typedef struct {
  int max_sqp_iters;
  int n_alphas;
  double alphas[8];
  double eta_armijo;
  double rho_penalty;
  double pcg_epsilon;
  int pcg_max_iters;
  double convergence_tol;
  double mu_floor_denominator;
  double eps_pd;
} port_sqp_config;

typedef struct port_solver port_solver;

port_solver* port_create(const port_problem* prob);
void port_destroy(port_solver* s);
int port_theta_size(const port_problem* prob);

/* problem.hpp:202-257 — QpData into the solver's slot. */
int port_linearize(port_solver* s, const double* theta, const double* z, double eps_pd, port_status* st);
/* schur.hpp:114-180 */
int port_assemble(port_solver* s, port_status* st);
/* schur.hpp:187-211 — returns -gamma into out (n_lambda). */
int port_gamma(port_solver* s, const double* b, const double* d, double* out, port_status* st);
/* pcg.hpp:52-109 on the solver's assembled system. eta_hist may be NULL. */
int port_pcg(port_solver* s, const double* gamma, const double* lambda0, double epsilon, int max_iters,
             double* lambda_out, int* iters, double* final_eta, int* converged, double* eta_hist,
             int eta_hist_cap, port_status* st);
/* sqp.hpp:62-89 */
int port_recover(port_solver* s, const double* lambda, const double* b, double* z_out, port_status* st);
/* problem.hpp:131-150: flat_b / flat_d of the current QP */
void port_flat_b(port_solver* s, double* b);
void port_flat_d(port_solver* s, double* d);
/* sqp.hpp:129-133 */
int port_merit(port_solver* s, const double* theta, const double* z, double mu, double* out, port_status* st);
/* sqp.hpp:151-206 */
int port_line_search(port_solver* s, const double* theta, const double* z_old, const double* z_qp,
                     const port_sqp_config* cfg, double mu_prev, double* z_new, double* alpha,
                     int* accepted, double* mu_out, port_status* st);
/* problem.hpp:263-300, reduced to its infinity norm */
int port_kkt_inf_norm(port_solver* s, const double* theta, const double* z, const double* lambda,
                      double* out, port_status* st);
/* sqp.hpp:213-261. pcg_iters/step_sizes hold max_sqp_iters entries. The final
 * QP and Schur system stay in the solver for port_backward. */
int port_sqp_solve(port_solver* s, const double* theta, const double* z0, const double* lambda0,
                   const port_sqp_config* cfg, double* z_out, double* lambda_out, int* sqp_iters,
                   int* converged, double* kkt_inf_norm, int* pcg_iters, double* step_sizes,
                   port_status* st);
/* backward.hpp:27-50 (uses the last port_sqp_solve's z, lambda, QP, Schur). */
int port_backward(port_solver* s, const double* theta, const double* loss_grad_z,
                  const double* lambda_tilde0, double pcg_epsilon, int pcg_max_iters, double* grad_theta,
                  double* lambda_tilde_out, int* pcg_iters, port_status* st);

/* Accessors for parity tests (dense column-major blocks). */
void port_get_qp(port_solver* s, double* Q, double* q, double* R, double* r, double* Ap, double* A,
                 double* B, double* C, double* x_s, int* pd_projected);
/* Block-tridiagonal system: diag (T+1) blocks, sub (T) blocks (block (i+1,i)),
 * precond diag (T+1), precond super (T) (block (i,i+1)). */
void port_get_schur(port_solver* s, double* s_diag, double* s_sub, double* p_diag, double* p_super);
/* Runs pcg on externally supplied blocks (for KATs on hand-built systems). */
int port_pcg_blocks(int nx, int n_blocks, const double* s_diag, const double* s_sub, const double* s_super,
                    const double* p_diag, const double* p_sub, const double* p_super, const double* gamma,
                    const double* lambda0, double epsilon, int max_iters, double* lambda_out, int* iters,
                    double* final_eta, int* converged, port_status* st);

/* One imitation-learning epoch body (train.hpp:82-131): per instance j a
 * solve from z0 = demo_j warm-started with lambda_cache_j, the control MSE
 * loss, a backward pass warm-started with lambda_tilde_cache_j, and the
 * fixed-order sums. thetas[j] already carry the shared learnable weights.
 * Caches are updated in place (WarmStartCache::store / store_backward).
 * grad_sum has learn_size entries (theta segment [learn_start, +learn_size)). */
int port_il_epoch(const port_problem* prob, int batch, const double* thetas, const double* demos,
                  double* lambda_cache, double* lambda_tilde_cache, const port_sqp_config* cfg,
                  int learn_start, int learn_size, double* loss_sum, double* grad_sum, double* losses,
                  double* grads, int* sqp_iters, long* pcg_iters, port_status* st);

#ifdef __cplusplus
}
#endif
#endif
