// ref_driver.cpp — C ABI over the UNMODIFIED reference headers
// (/root/reference/proj/include, compiled against oracle/eigen_lite).
//
// TEST INFRASTRUCTURE / ORACLE. Built by oracle/Makefile into
// oracle/_ref/libdocp_ref.so (git-ignored; travels to the GPU box as a
// prebuilt file). It mirrors oracle/port/docp_port.h function for function
// (prefix ref_ instead of port_) so tests can check the C restatement against
// the reference itself, and it exposes the reference's own generators and
// training loop for golden-vector generation. Nothing here re-implements the
// algorithm: every numeric result comes from a reference function.
#include "docp/bench/study.hpp"
#include "docp/bench/train.hpp"
#include "docp/oracle.hpp"

#include <cstring>
#include <memory>

#include "port/docp_port.h"
// The drifting family has no reference implementation: its
// single model definition is shared with the GPU path, so this harness runs
// the REFERENCE solver (sqp_solve / backward_vjp / train_il body) on it.
#include "docp_drift_model.h"

using namespace docp;

namespace {

int to_code(const std::exception& e) {
  if (dynamic_cast<const DimensionError*>(&e)) return PORT_DIMENSION;
  if (dynamic_cast<const EvaluationError*>(&e)) return PORT_EVALUATION;
  if (dynamic_cast<const NumericalError*>(&e)) return PORT_NUMERICAL;
  if (dynamic_cast<const BreakdownError*>(&e)) return PORT_BREAKDOWN;
  if (dynamic_cast<const DivergenceError*>(&e)) return PORT_DIVERGENCE;
  return 99;
}

int set_status(port_status* st, const std::exception& e) {
  int code = to_code(e);
  if (st) {
    st->code = code;
    st->iteration = 0;
    if (auto* b = dynamic_cast<const BreakdownError*>(&e)) st->iteration = b->iteration;
    std::snprintf(st->message, sizeof st->message, "%s", e.what());
  }
  return code;
}

void clear(port_status* st) {
  if (st) {
    st->code = PORT_OK;
    st->iteration = 0;
    st->message[0] = 0;
  }
}

Vector vec(const double* p, Eigen::Index n) { return Eigen::Map<const Vector>(p, n); }
void put(const Vector& v, double* out) {
  if (out) std::memcpy(out, v.data(), sizeof(double) * static_cast<std::size_t>(v.size()));
}
void put(const Matrix& m, double* out) {
  if (out) std::memcpy(out, m.data(), sizeof(double) * static_cast<std::size_t>(m.size()));
}

/// Family -> OcpDefinition. AffineQuadratic reads every coefficient from
/// theta (affine_quadratic.hpp:39-81), so the struct only carries sizes.
OcpDefinition make_ocp(const port_problem& p) {
  if (p.family == PORT_DRIFT) {  // the cart-pole pattern (cartpole.hpp:91-107) on the shared drift model
    OcpDefinition ocp;
    ocp.n_x = docp_drift::NX;
    ocp.n_u = docp_drift::NU;
    ocp.horizon = p.horizon;
    ocp.state_cost = make_diag_quadratic_cost(segment::state_cost, 0.5);
    ocp.control_cost = make_diag_quadratic_cost(segment::control_cost, 0.5);
    const double dt = p.dt;
    ocp.dynamics_residual = make_explicit_dynamics(
        [dt](int, const Vector& x, const Vector& u, const ParameterVector& theta) {
          const Vector th = theta.values();
          ExplicitStep s;
          s.x_next = Vector::Zero(docp_drift::NX);
          s.jac_x = Matrix::Zero(docp_drift::NX, docp_drift::NX);
          s.jac_u = Matrix::Zero(docp_drift::NX, docp_drift::NU);
          docp_drift::step(th.data(), dt, x.data(), u.data(), s.x_next.data(), s.jac_x.data(), s.jac_u.data());
          return s;
        });
    ocp.initial_state = [](const ParameterVector& theta) { return Vector(theta.segment(segment::initial_state)); };
    ocp.theta_vjp = make_quadratic_cost_theta_vjp(0.5);
    return ocp;
  }
  if (p.family == PORT_ATTITUDE) {
    AttitudeParams ap;
    ap.inertia = vec(p.inertia, 3);
    ap.dt = p.dt;
    ap.horizon = p.horizon;
    return make_attitude_ocp(ap);
  }
  if (p.family == PORT_CARTPOLE) {
    CartpoleParams cp;
    cp.cart_mass = p.cart_mass;
    cp.pole_mass = p.pole_mass;
    cp.length = p.length;
    cp.gravity = p.gravity;
    cp.dt = p.dt;
    cp.horizon = p.horizon;
    return make_cartpole_ocp(cp);
  }
  AffineQuadratic aq;
  aq.n_x = p.nx;
  aq.n_u = p.nu;
  aq.horizon = p.horizon;
  aq.cost_scale = p.cost_scale;
  return aq.make_ocp();
}

/// theta values -> ParameterVector with the family's segment layout.
ParameterVector make_theta(const port_problem& p, const double* th) {
  ParameterVector theta;
  int k = 0;
  auto seg = [&](const char* name, int n) {
    theta.add_segment(name, vec(th + k, n));
    k += n;
  };
  if (p.family == PORT_CARTPOLE || p.family == PORT_ATTITUDE) {
    seg(segment::state_cost, p.nx);
    seg(segment::control_cost, p.nu);
    seg(segment::initial_state, p.nx);
  } else if (p.family == PORT_DRIFT) {
    seg(segment::state_cost, p.nx);
    seg(segment::control_cost, p.nu);
    seg(segment::initial_state, p.nx);
    seg("drift_model", docp_drift::NTH - docp_drift::TH_XREF);  // X_ref + vehicle parameters
  } else {
    seg(segment::state_cost, p.nx);
    seg(segment::control_cost, p.nu);
    seg(segment::dynamics, p.nx * p.nx + p.nx * p.nu + p.nx);
    seg(segment::initial_state, p.nx);
  }
  return theta;
}

SqpConfig make_cfg(const port_sqp_config& c) {
  SqpConfig cfg;
  cfg.max_sqp_iters = c.max_sqp_iters;
  cfg.step_candidates.assign(c.alphas, c.alphas + c.n_alphas);
  cfg.eta_armijo = c.eta_armijo;
  cfg.rho_penalty = c.rho_penalty;
  cfg.pcg.epsilon = c.pcg_epsilon;
  cfg.pcg.max_iters = c.pcg_max_iters;
  cfg.convergence_tol = c.convergence_tol;
  cfg.mu_floor_denominator = c.mu_floor_denominator;
  cfg.eps_pd = c.eps_pd;
  return cfg;
}

}  // namespace

struct ref_solver {
  port_problem p;
  OcpDefinition ocp;
  SolveResult res;
};

extern "C" {

ref_solver* ref_create(const port_problem* p) {
  auto* s = new ref_solver;
  s->p = *p;
  s->ocp = make_ocp(*p);
  return s;
}
void ref_destroy(ref_solver* s) { delete s; }

int ref_linearize(ref_solver* s, const double* th, const double* z, double eps_pd, port_status* st) {
  clear(st);
  try {
    const OcpDefinition& o = s->ocp;
    Trajectory traj = Trajectory::unflatten(vec(z, o.primal_size()), o.n_x, o.n_u, o.horizon);
    s->res.qp = linearize(o, traj, make_theta(s->p, th), eps_pd);
    s->res.z = traj;
  } catch (const Error& e) {
    return set_status(st, e);
  }
  return 0;
}

int ref_assemble(ref_solver* s, port_status* st) {
  clear(st);
  try {
    s->res.schur = assemble_schur(s->res.qp);
  } catch (const Error& e) {
    return set_status(st, e);
  }
  return 0;
}

void ref_flat_b(ref_solver* s, double* b) { put(s->res.qp.flat_b(), b); }
void ref_flat_d(ref_solver* s, double* d) { put(s->res.qp.flat_d(), d); }

int ref_gamma(ref_solver* s, const double* b, const double* d, double* out, port_status* st) {
  clear(st);
  try {
    const auto& qp = s->res.qp;
    put(assemble_gamma(qp, s->res.schur, vec(b, qp.primal_size()), vec(d, qp.dual_size())), out);
  } catch (const Error& e) {
    return set_status(st, e);
  }
  return 0;
}

int ref_pcg(ref_solver* s, const double* gamma, const double* lambda0, double eps, int max_iters, double* lam,
            int* iters, double* final_eta, int* converged, double* eta_hist, int eta_hist_cap, port_status* st) {
  clear(st);
  try {
    PcgConfig cfg;
    cfg.epsilon = eps;
    cfg.max_iters = max_iters;
    cfg.record_eta_history = eta_hist != nullptr;
    Eigen::Index n = s->res.schur.dim();
    PcgOutcome out = pcg_solve(s->res.schur, vec(gamma, n), vec(lambda0, n), cfg);
    put(out.lambda, lam);
    *iters = out.iters;
    *final_eta = out.final_eta;
    *converged = out.converged;
    if (eta_hist)
      for (int k = 0; k < eta_hist_cap && k < static_cast<int>(out.eta_history.size()); ++k)
        eta_hist[k] = out.eta_history[static_cast<std::size_t>(k)];
  } catch (const Error& e) {
    return set_status(st, e);
  }
  return 0;
}

int ref_recover(ref_solver* s, const double* lam, const double* b, double* z, port_status* st) {
  clear(st);
  try {
    const auto& qp = s->res.qp;
    put(recover_primal(qp, s->res.schur, vec(lam, qp.dual_size()), vec(b, qp.primal_size())).flatten(), z);
  } catch (const Error& e) {
    return set_status(st, e);
  }
  return 0;
}

int ref_merit(ref_solver* s, const double* th, const double* z, double mu, double* out, port_status* st) {
  clear(st);
  try {
    const OcpDefinition& o = s->ocp;
    *out = merit(o, Trajectory::unflatten(vec(z, o.primal_size()), o.n_x, o.n_u, o.horizon), mu,
                 make_theta(s->p, th));
  } catch (const Error& e) {
    return set_status(st, e);
  }
  return 0;
}

int ref_line_search(ref_solver* s, const double* th, const double* z_old, const double* z_qp,
                    const port_sqp_config* cfg, double mu_prev, double* z_new, double* alpha, int* accepted,
                    double* mu_out, port_status* st) {
  clear(st);
  try {
    const OcpDefinition& o = s->ocp;
    auto tr = [&](const double* z) { return Trajectory::unflatten(vec(z, o.primal_size()), o.n_x, o.n_u, o.horizon); };
    LineSearchResult ls =
        line_search(o, s->res.qp, tr(z_old), tr(z_qp), make_theta(s->p, th), make_cfg(*cfg), mu_prev);
    put(ls.z.flatten(), z_new);
    *alpha = ls.alpha;
    *accepted = ls.accepted;
    *mu_out = ls.mu;
  } catch (const Error& e) {
    return set_status(st, e);
  }
  return 0;
}

int ref_kkt_inf_norm(ref_solver* s, const double* th, const double* z, const double* lam, double* out,
                     port_status* st) {
  clear(st);
  try {
    const OcpDefinition& o = s->ocp;
    Trajectory traj = Trajectory::unflatten(vec(z, o.primal_size()), o.n_x, o.n_u, o.horizon);
    *out = kkt_residual(o, traj, vec(lam, o.dual_size()), make_theta(s->p, th)).cwiseAbs().maxCoeff();
  } catch (const Error& e) {
    return set_status(st, e);
  }
  return 0;
}

int ref_sqp_solve(ref_solver* s, const double* th, const double* z0, const double* lambda0,
                  const port_sqp_config* cfg, double* z_out, double* lambda_out, int* sqp_iters, int* converged,
                  double* kkt, int* pcg_iters, double* step_sizes, port_status* st) {
  clear(st);
  try {
    const OcpDefinition& o = s->ocp;
    Trajectory traj = Trajectory::unflatten(vec(z0, o.primal_size()), o.n_x, o.n_u, o.horizon);
    s->res = sqp_solve(o, make_theta(s->p, th), traj, vec(lambda0, o.dual_size()), make_cfg(*cfg));
    put(s->res.z.flatten(), z_out);
    put(s->res.lambda, lambda_out);
    *sqp_iters = s->res.sqp_iters;
    *converged = s->res.converged;
    *kkt = s->res.kkt_inf_norm;
    for (std::size_t k = 0; k < s->res.pcg_iters.size(); ++k) {
      if (pcg_iters) pcg_iters[k] = s->res.pcg_iters[k];
      if (step_sizes) step_sizes[k] = s->res.step_sizes[k];
    }
  } catch (const Error& e) {
    return set_status(st, e);
  }
  return 0;
}

int ref_backward(ref_solver* s, const double* th, const double* loss_grad_z, const double* lt0, double eps,
                 int max_iters, double* grad, double* lt_out, int* pcg_iters, port_status* st) {
  clear(st);
  try {
    const OcpDefinition& o = s->ocp;
    PcgConfig cfg;
    cfg.epsilon = eps;
    cfg.max_iters = max_iters;
    BackwardResult b = backward_vjp(s->res, vec(loss_grad_z, o.primal_size()), vec(lt0, o.dual_size()), o,
                                    make_theta(s->p, th), cfg);
    put(b.grad_theta, grad);
    put(b.lambda_tilde, lt_out);
    *pcg_iters = b.pcg_iters;
  } catch (const Error& e) {
    return set_status(st, e);
  }
  return 0;
}

void ref_get_qp(ref_solver* s, double* Q, double* q, double* R, double* r, double* Ap, double* A, double* B,
                double* C, double* x_s, int* pd) {
  const QpData& qp = s->res.qp;
  const std::size_t nx = static_cast<std::size_t>(qp.n_x), nu = static_cast<std::size_t>(qp.n_u);
  for (std::size_t t = 0; t <= static_cast<std::size_t>(qp.horizon); ++t) {
    if (Q) put(qp.Q[t], Q + t * nx * nx);
    if (q) put(qp.q[t], q + t * nx);
    if (t == static_cast<std::size_t>(qp.horizon)) break;
    if (R) put(qp.R[t], R + t * nu * nu);
    if (r) put(qp.r[t], r + t * nu);
    if (Ap) put(qp.A_plus[t], Ap + t * nx * nx);
    if (A) put(qp.A[t], A + t * nx * nx);
    if (B) put(qp.B[t], B + t * nx * nu);
    if (C) put(qp.C[t], C + t * nx);
  }
  put(qp.x_s, x_s);
  if (pd) *pd = qp.pd_projected;
}

void ref_get_schur(ref_solver* s, double* Sd, double* Ssub, double* Pd, double* Psup) {
  const SchurSystem& sys = s->res.schur;
  const std::size_t b2 = static_cast<std::size_t>(sys.n_x) * static_cast<std::size_t>(sys.n_x);
  for (std::size_t i = 0; i < sys.neg_s.diag.size(); ++i) {
    if (Sd) put(sys.neg_s.diag[i], Sd + i * b2);
    if (Pd) put(sys.precond.diag[i], Pd + i * b2);
  }
  for (std::size_t i = 0; i < sys.neg_s.sub.size(); ++i) {
    if (Ssub) put(sys.neg_s.sub[i], Ssub + i * b2);
    if (Psup) put(sys.precond.super[i], Psup + i * b2);
  }
}

int ref_pcg_blocks(int nx, int nb, const double* Sd, const double* Ssub, const double* Ssup, const double* Pd,
                   const double* Psub, const double* Psup, const double* gamma, const double* lambda0, double eps,
                   int max_iters, double* lam, int* iters, double* final_eta, int* converged, port_status* st) {
  clear(st);
  try {
    SchurSystem sys;
    sys.n_x = nx;
    const std::size_t b2 = static_cast<std::size_t>(nx) * static_cast<std::size_t>(nx);
    auto blk = [&](const double* p, std::size_t i) { return Matrix(Eigen::Map<const Matrix>(p + i * b2, nx, nx)); };
    for (int i = 0; i < nb; ++i) {
      sys.neg_s.diag.push_back(blk(Sd, static_cast<std::size_t>(i)));
      sys.precond.diag.push_back(blk(Pd, static_cast<std::size_t>(i)));
    }
    for (int i = 0; i + 1 < nb; ++i) {
      sys.neg_s.sub.push_back(blk(Ssub, static_cast<std::size_t>(i)));
      sys.neg_s.super.push_back(blk(Ssup, static_cast<std::size_t>(i)));
      sys.precond.sub.push_back(blk(Psub, static_cast<std::size_t>(i)));
      sys.precond.super.push_back(blk(Psup, static_cast<std::size_t>(i)));
    }
    PcgConfig cfg;
    cfg.epsilon = eps;
    cfg.max_iters = max_iters;
    Eigen::Index n = static_cast<Eigen::Index>(nx) * nb;
    PcgOutcome out = pcg_solve(sys, vec(gamma, n), vec(lambda0, n), cfg);
    put(out.lambda, lam);
    *iters = out.iters;
    *final_eta = out.final_eta;
    *converged = out.converged;
  } catch (const Error& e) {
    return set_status(st, e);
  }
  return 0;
}

/// Epoch body of train_il (train.hpp:82-131) for either family, built only
/// from reference calls: sqp_solve, backward_vjp, WarmStartCache.
int ref_il_epoch(const port_problem* p, int batch, const double* thetas, const double* demos, double* lam_cache,
                 double* lt_cache, const port_sqp_config* c, int learn_start, int learn_size, double* loss_sum,
                 double* grad_sum, double* losses, double* grads, int* sqp_iters, long* pcg_iters,
                 port_status* st) {
  clear(st);
  OcpDefinition ocp = make_ocp(*p);
  SqpConfig cfg = make_cfg(*c);
  const int nth = p->family == PORT_DRIFT ? docp_drift::NTH
                  : (p->family == PORT_CARTPOLE || p->family == PORT_ATTITUDE)
                      ? 2 * p->nx + p->nu
                      : p->nx + p->nu + p->nx * p->nx + p->nx * p->nu + 2 * p->nx;
  const Eigen::Index nz = ocp.primal_size(), nl = ocp.dual_size();
  std::vector<std::string> errors(static_cast<std::size_t>(batch));
  std::vector<Vector> g(static_cast<std::size_t>(batch));
  std::vector<double> loss(static_cast<std::size_t>(batch), 0.0);
  parallel_for(static_cast<std::size_t>(batch), 0, [&](std::size_t j) {
    try {
      ParameterVector theta = make_theta(*p, thetas + j * static_cast<std::size_t>(nth));
      Trajectory demo = Trajectory::unflatten(vec(demos + j * static_cast<std::size_t>(nz), nz), ocp.n_x, ocp.n_u,
                                              ocp.horizon);
      SolveResult res = sqp_solve(ocp, theta, demo, vec(lam_cache + j * static_cast<std::size_t>(nl), nl), cfg);
      Matrix du = res.z.u - demo.u;
      loss[j] = du.squaredNorm() / batch;
      Vector loss_grad = Vector::Zero(nz);
      for (int t = 0; t < ocp.horizon; ++t)
        loss_grad.segment(flat_offset(ocp.n_x, ocp.n_u, t, false), ocp.n_u) = 2.0 / batch * du.col(t);
      BackwardResult back = backward_vjp(res, loss_grad, vec(lt_cache + j * static_cast<std::size_t>(nl), nl), ocp,
                                         theta, cfg.pcg);
      g[j] = back.grad_theta.segment(learn_start, learn_size);
      sqp_iters[j] = res.sqp_iters;
      long pc = 0;
      for (int it : res.pcg_iters) pc += it;
      pcg_iters[j] = pc + back.pcg_iters;
      put(res.lambda, lam_cache + j * static_cast<std::size_t>(nl));
      put(back.lambda_tilde, lt_cache + j * static_cast<std::size_t>(nl));
      losses[j] = loss[j];
      put(g[j], grads + j * static_cast<std::size_t>(learn_size));
    } catch (const Error& e) {
      errors[j] = e.what();
    }
  });
  for (int j = 0; j < batch; ++j)
    if (!errors[static_cast<std::size_t>(j)].empty()) {
      if (st) {
        st->code = 99;
        std::snprintf(st->message, sizeof st->message, "demonstration %d: %s", j,
                      errors[static_cast<std::size_t>(j)].c_str());
      }
      return 99;
    }
  double obj = 0.0;
  Vector grad = Vector::Zero(learn_size);
  for (int j = 0; j < batch; ++j) {
    obj += loss[static_cast<std::size_t>(j)];
    grad += g[static_cast<std::size_t>(j)];
  }
  *loss_sum = obj;
  put(grad, grad_sum);
  return 0;
}

/// The reference's own cart-pole trainer for one or more epochs
/// (train.hpp:53-145), used to pin ref_il_epoch's restated body.
int ref_train_il_cartpole(std::uint64_t seed, int horizon, int n_demos, const double* initial_weights, int epochs,
                          double lr, double* objectives, long* sqp_iters, long* pcg_iters, double* final_weights,
                          port_status* st) {
  clear(st);
  try {
    CartpoleParams cp;
    cp.horizon = horizon;
    auto bundle = bench::gen_cartpole(seed, cp, n_demos);
    bench::IlTrainOptions opts;
    opts.epochs = epochs;
    opts.learning_rate = lr;
    if (initial_weights) opts.initial_weights = vec(initial_weights, 4);
    auto rep = bench::train_il(bundle, opts);
    if (rep.failed) throw Error(rep.failure);
    for (std::size_t k = 0; k < rep.records.size(); ++k) {
      objectives[k] = rep.records[k].objective;
      sqp_iters[k] = rep.records[k].sqp_iters;
      pcg_iters[k] = rep.records[k].pcg_iters;
    }
    put(rep.final_learnable, final_weights);
  } catch (const std::exception& e) {
    return set_status(st, e);
  }
  return 0;
}

/// rollout + rollout_backward (batch.hpp:172-258) of affine-quadratic
/// instances with their own dynamics as the environment (make_affine_env,
/// train.hpp:195-213): the train_rl inner body (train.hpp:287-297), one
/// instance per theta row, x_init per row. ok[j] = 0 with the exception text
/// in messages[j * 256] when the reference throws for that instance.
int ref_rollout_affine(int nx, int nu, int horizon, int batch, const double* thetas, const double* x_inits,
                       int episode_length, const port_sqp_config* c, double* rewards, double* grads, int* ok,
                       char* messages) {
  const std::size_t nth = static_cast<std::size_t>(nx + nu + nx * nx + nx * nu + nx + nx);
  SqpConfig cfg = make_cfg(*c);
  parallel_for(static_cast<std::size_t>(batch), 0, [&](std::size_t j) {
    const double* th = thetas + j * nth;
    AffineQuadratic p;
    p.n_x = nx;
    p.n_u = nu;
    p.horizon = horizon;
    p.w_x = vec(th, nx);
    p.w_u = vec(th + nx, nu);
    p.A = Eigen::Map<const Matrix>(th + nx + nu, nx, nx);
    p.B = Eigen::Map<const Matrix>(th + nx + nu + nx * nx, nx, nu);
    p.b_affine = vec(th + nx + nu + nx * nx + nx * nu, nx);
    p.x_s = vec(th + nx + nu + nx * nx + nx * nu + nx, nx);
    OcpDefinition ocp = p.make_ocp();
    ParameterVector theta = p.make_theta();
    DiffEnv env = bench::make_affine_env(p);
    try {
      RolloutOutput roll = rollout(env, ocp, theta, vec(x_inits + j * static_cast<std::size_t>(nx), nx),
                                   episode_length, cfg);
      Vector g = rollout_backward(roll.record, env, ocp, theta, cfg.pcg);
      rewards[j] = roll.total_reward;
      put(g, grads + j * nth);
      ok[j] = 1;
    } catch (const Error& e) {
      ok[j] = 0;
      std::snprintf(messages + j * 256, 256, "%s", e.what());
    }
  });
  return 0;
}

/// rollout + rollout_backward of attitude instances with the attitude RL
/// task's environment (make_attitude_rl_task, train.hpp:239-263): step =
/// attitude_step, reward -(0.1 |x|^2 + |u|^2). thetas: [batch][9] (reference
/// layout), inertias: [batch][3].
int ref_rollout_attitude(int horizon, double dt, int batch, const double* thetas, const double* inertias,
                         const double* x_inits, int episode_length, const port_sqp_config* c, double* rewards,
                         double* grads, int* ok, char* messages) {
  SqpConfig cfg = make_cfg(*c);
  parallel_for(static_cast<std::size_t>(batch), 0, [&](std::size_t j) {
    AttitudeParams p;
    p.inertia = vec(inertias + 3 * j, 3);
    p.dt = dt;
    p.horizon = horizon;
    OcpDefinition ocp = make_attitude_ocp(p);
    ParameterVector theta = make_attitude_theta(vec(thetas + 9 * j, 3), vec(thetas + 9 * j + 3, 3),
                                                vec(thetas + 9 * j + 6, 3));
    DiffEnv env = make_diff_env(
        [p](const Vector& x, const Vector& u) { return attitude_step(p, x, u); },
        [](const Vector& x, const Vector& u) { return -(0.1 * x.squaredNorm() + u.squaredNorm()); },
        [](const Vector& x, const Vector& u) { return std::make_pair(Vector(-0.2 * x), Vector(-2.0 * u)); });
    try {
      RolloutOutput roll = rollout(env, ocp, theta, vec(x_inits + 3 * j, 3), episode_length, cfg);
      Vector g = rollout_backward(roll.record, env, ocp, theta, cfg.pcg);
      rewards[j] = roll.total_reward;
      put(g, grads + 9 * j);
      ok[j] = 1;
    } catch (const Error& e) {
      ok[j] = 0;
      std::snprintf(messages + j * 256, 256, "%s", e.what());
    }
  });
  return 0;
}

/// The reference's own pcg_study (study.hpp:56-145): per (tol, step, pass)
/// cold and warm PCG iteration counts, rows in the report's order
/// (tol-major, then step, forward before backward). Returns the row count.
int ref_pcg_study(const double* tols, int n_tols, int steps, std::uint64_t seed, int nx, int nu, int horizon,
                  int* cold_iters, int* warm_iters) {
  auto rep = bench::pcg_study(std::vector<double>(tols, tols + n_tols), steps, seed, nx, nu, horizon);
  for (std::size_t k = 0; k < rep.rows.size(); ++k) {
    cold_iters[k] = rep.rows[k].cold_iters;
    warm_iters[k] = rep.rows[k].warm_iters;
  }
  return static_cast<int>(rep.rows.size());
}

/// bench::gen_cartpole (generators.hpp:134-168): initial states (n x 4) and
/// expert demonstrations (n x n_z, flat layout).
int ref_gen_cartpole(std::uint64_t seed, int horizon, int n_demos, double* x0s, double* demos, port_status* st) {
  clear(st);
  try {
    CartpoleParams cp;
    cp.horizon = horizon;
    auto b = bench::gen_cartpole(seed, cp, n_demos);
    const std::size_t nz = static_cast<std::size_t>(b.demonstrations[0].flat_size());
    for (int i = 0; i < n_demos; ++i) {
      put(b.initial_states[static_cast<std::size_t>(i)], x0s + 4 * i);
      put(b.demonstrations[static_cast<std::size_t>(i)].flatten(), demos + nz * static_cast<std::size_t>(i));
    }
  } catch (const std::exception& e) {
    return set_status(st, e);
  }
  return 0;
}

/// Sequential draws of random_convex_instance (convex != 0) or
/// random_linear_instance from one mt19937_64(seed) (generators.hpp:52-111);
/// writes each instance's make_theta() values.
void ref_gen_aq(int nx, int nu, int horizon, std::uint64_t seed, int count, int convex, double* thetas) {
  std::mt19937_64 rng(seed);
  const std::size_t nth = static_cast<std::size_t>(nx + nu + nx * nx + nx * nu + nx + nx);
  for (int i = 0; i < count; ++i) {
    AffineQuadratic p = convex ? bench::random_convex_instance(nx, nu, horizon, rng)
                               : bench::random_linear_instance(nx, nu, horizon, rng);
    put(p.make_theta().values(), thetas + nth * static_cast<std::size_t>(i));
  }
}

/// The learnable-weight draw of train_il (train.hpp:61-64): n values of
/// uniform_real_distribution(lo, hi) from mt19937_64(seed), in order.
void ref_gen_uniform(std::uint64_t seed, int n, double lo, double hi, double* out) {
  std::mt19937_64 rng(seed);
  std::uniform_real_distribution<double> unit(lo, hi);
  for (int i = 0; i < n; ++i) out[i] = unit(rng);
}

/// The drifting model's explicit step and Jacobians (include/docp_drift_model.h), host build.
void ref_drift_step(const double* th, double dt, const double* xbar, const double* u, double* xn, double* jx,
                    double* ju) {
  docp_drift::step(th, dt, xbar, u, xn, jx, ju);
}

/// Reference spectral radius (generators.hpp:41-46) of an n x n col-major matrix.
double ref_spectral_radius(const double* a, int n) {
  return bench::spectral_radius(Matrix(Eigen::Map<const Matrix>(a, n, n)));
}

unsigned long long ref_pcg_invocations() { return stats::pcg_invocations().load(); }

}  // extern "C"
