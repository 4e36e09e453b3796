// docp_gpu.hpp — C++ drop-in for the reference solver API on the B200 path.
//
// This header lives beside the reference's own headers (proj/include/docp,
// namespace docp). It keeps their value types and function signatures and
// runs the work on the GPU through the C ABI of libdocp_cuda.so
// (include/docp_cuda.h). Only one thing is added to each signature: a
// `Family` descriptor. The reference's OcpDefinition is a bundle of
// std::function callbacks, which cannot cross to the device, so the family
// tag and its constants take their place.
//
//   reference (namespace docp)                   here (namespace docp::gpu)
//   sqp_solve(ocp, theta, z0, lambda0, cfg)      sqp_solve(family, ocp, theta, z0, lambda0, cfg)   sqp.hpp:213-261
//   backward_vjp(res, gz, lt0, ocp, theta, pcg)  backward_vjp(res, gz, lt0, family, ocp, theta, pcg) backward.hpp:27-50
//   pcg_solve(sys, gamma, lambda0, cfg)          pcg_solve(sys, gamma, lambda0, cfg)                pcg.hpp:52-109
//   batch_solve(instances, cache, cfg, workers)  batch_solve(family, instances, cache, cfg)          batch.hpp:83-108
//   (train_il inner loop, train.hpp:82-109)      BatchSolver::solve + BatchSolver::backward
//   rollout / rollout_backward (batch.hpp:172-258, affine env train.hpp:195-213)
//                                                BatchSolver::rollout + BatchSolver::rollout_backward
//
// Behaviour kept from the reference:
//   * argument checks with the reference's DimensionError messages;
//   * per-problem failures are re-raised as the same docp::Error subclass
//     and message (BreakdownError carries the iteration), or reported in
//     BatchItem{ok=false, error} by batch_solve;
//   * stats::pcg_invocations() grows by one per solved system.
//
// The returned SolveResult carries qp and schur downloaded from the device
// (Options::materialize, on by default for the single-instance calls). The
// Cholesky factors are rebuilt from the downloaded Q, R blocks. A
// reference-side backward_vjp can therefore consume a GPU SolveResult.
// Numerics: Options::mode = DOCP_PCG_PARITY reproduces the reference bits
// (eigen_lite conventions); DOCP_PCG_FAST uses FMA and tree
// reductions inside PCG, with equal iteration counts and <= 1e-9 relative error.
// PcgConfig::record_eta_history is test instrumentation and is not recorded.
#pragma once

#include <cstdint>
#include <memory>
#include <string>
#include <vector>

#include "docp/backward.hpp"
#include "docp/batch.hpp"
#include "docp/problems/affine_quadratic.hpp"
#include "docp/problems/attitude.hpp"
#include "docp/problems/cartpole.hpp"
#include "docp/sqp.hpp"
#include "docp_cuda.h"

namespace docp::gpu {

/// What the device needs instead of OcpDefinition's callbacks.
struct Family {
  docp_problem desc{};
  /// Per-problem constants the device keeps after theta's reference layout
  /// (attitude: AttitudeParams::inertia); appended to thetas that omit them.
  std::vector<double> theta_tail;
};

/// AffineQuadratic::make_ocp (affine_quadratic.hpp:39-81).
inline Family family_of(const AffineQuadratic& p) {
  Family f;
  f.desc.family = DOCP_AFFINE_QUADRATIC;
  f.desc.n_x = p.n_x;
  f.desc.n_u = p.n_u;
  f.desc.horizon = p.horizon;
  f.desc.cost_scale = p.cost_scale;
  return f;
}

/// make_attitude_ocp (attitude.hpp:55-72); the inertia rides in theta's tail.
inline Family family_of(const AttitudeParams& p) {
  Family f;
  f.desc.family = DOCP_ATTITUDE;
  f.desc.n_x = 3;
  f.desc.n_u = 3;
  f.desc.horizon = p.horizon;
  f.desc.cost_scale = 0.5;
  f.desc.dt = p.dt;
  for (Eigen::Index i = 0; i < p.inertia.size(); ++i) f.theta_tail.push_back(p.inertia[i]);
  return f;
}

/// make_cartpole_ocp (cartpole.hpp:91-127).
inline Family family_of(const CartpoleParams& p) {
  Family f;
  f.desc.family = DOCP_CARTPOLE;
  f.desc.n_x = 4;
  f.desc.n_u = 1;
  f.desc.horizon = p.horizon;
  f.desc.cost_scale = 0.5;
  f.desc.cart_mass = p.cart_mass;
  f.desc.pole_mass = p.pole_mass;
  f.desc.length = p.length;
  f.desc.gravity = p.gravity;
  f.desc.dt = p.dt;
  return f;
}

/// The drifting family (include/docp_drift_model.h; the reference has no
/// model class for it): theta is the full 36-entry device layout [w_x 8 |
/// w_u 2 | xbar_0 8 | X_ref 8 | vehicle parameters 10], built by the caller
/// (e.g. the ParameterVector the reference-solver harness oracle/ref_driver.cpp
/// uses: segments state_cost, control_cost, initial_state, "drift_model").
inline Family family_drift(int horizon, double dt) {
  Family f;
  f.desc.family = DOCP_DRIFT;
  f.desc.n_x = 8;
  f.desc.n_u = 2;
  f.desc.horizon = horizon;
  f.desc.cost_scale = 0.5;
  f.desc.dt = dt;
  return f;
}

struct Options {
  int device = 0;
  void* stream = nullptr;  // cudaStream_t; nullptr = legacy default stream
  int mode = DOCP_PCG_PARITY;
  bool materialize = true;  // fill SolveResult::qp / ::schur from the device
  /// backward_vjp(SolveResult, ...) re-linearizes at res.z: this must be the
  /// eps_pd of the forward solve's SqpConfig (a SolveResult does not record it).
  double eps_pd = kDefaultEpsPd;
};

namespace detail {

/// ABI-level failure (bad arguments, CUDA errors): DOCP_DIMENSION maps to
/// DimensionError, everything else to Error.
inline void check(int rc) {
  if (rc == DOCP_OK) return;
  const std::string msg = std::string("docp_cuda: ") + docp_last_error();
  if (rc == DOCP_DIMENSION) throw DimensionError(msg);
  throw Error(msg);
}

inline std::string status_message(const docp_status& st) {
  char buf[256];
  docp_format_status(&st, buf, sizeof(buf));
  return buf;
}

/// Re-raise a per-problem status as the reference's exception type.
[[noreturn]] inline void throw_status(const docp_status& st) {
  const std::string msg = status_message(st);
  switch (st.code) {
    case DOCP_DIMENSION: throw DimensionError(msg);
    case DOCP_EVALUATION: throw EvaluationError(msg);
    case DOCP_NUMERICAL: throw NumericalError(msg);
    case DOCP_BREAKDOWN: throw BreakdownError(msg, st.index);
    case DOCP_DIVERGENCE: throw DivergenceError(msg);
    default: throw Error(msg);
  }
}

inline docp_pcg_config to_c(const PcgConfig& c, int mode) {
  docp_pcg_config o{};
  o.epsilon = c.epsilon;
  o.max_iters = c.max_iters;
  o.mode = mode;
  return o;
}

inline docp_sqp_config to_c(const SqpConfig& c, int mode) {
  require(c.step_candidates.size() <= DOCP_MAX_STEP_CANDIDATES, "sqp: too many step candidates for the GPU path");
  docp_sqp_config o{};
  o.max_sqp_iters = c.max_sqp_iters;
  o.n_step_candidates = static_cast<int32_t>(c.step_candidates.size());
  for (std::size_t i = 0; i < c.step_candidates.size(); ++i) o.step_candidates[i] = c.step_candidates[i];
  o.eta_armijo = c.eta_armijo;
  o.rho_penalty = c.rho_penalty;
  o.pcg = to_c(c.pcg, mode);
  o.convergence_tol = c.convergence_tol;
  o.mu_floor_denominator = c.mu_floor_denominator;
  o.eps_pd = c.eps_pd;
  return o;
}

/// Adds the library's solve count delta to the reference counter on scope exit.
struct CountPcg {
  std::uint64_t start = docp_pcg_invocations();
  ~CountPcg() { stats::pcg_invocations().fetch_add(docp_pcg_invocations() - start, std::memory_order_relaxed); }
};

/// Owning handle of one device batch.
class Batch {
 public:
  Batch(const docp_problem& prob, int size, const Options& opt) : prob_(prob), size_(size) {
    check(docp_batch_create(&prob_, size, opt.device, &b_));
    if (opt.stream) check(docp_batch_set_stream(b_, opt.stream));
    nth_ = docp_theta_size(&prob_);
  }
  ~Batch() { docp_batch_destroy(b_); }
  Batch(const Batch&) = delete;
  Batch& operator=(const Batch&) = delete;

  docp_batch* get() const { return b_; }
  int size() const { return size_; }
  int n_theta() const { return nth_; }
  const docp_problem& problem() const { return prob_; }
  int n_z() const { return prob_.n_x * (prob_.horizon + 1) + prob_.n_u * prob_.horizon; }
  int n_lambda() const { return prob_.n_x * (prob_.horizon + 1); }

  void upload(int field, const std::vector<double>& host) { check(docp_batch_upload(b_, field, host.data(), 0)); }
  /// The whole field, sized from the library (per-problem stride = size() / batch size).
  template <class T>
  std::vector<T> download(int field) {
    void* ptr = nullptr;
    std::size_t bytes = 0;
    check(docp_batch_field_ptr(b_, field, &ptr, &bytes));
    std::vector<T> out(bytes / sizeof(T));
    check(docp_batch_download(b_, field, out.data(), 0));
    return out;
  }

 private:
  docp_problem prob_;
  int size_;
  int nth_ = 0;
  docp_batch* b_ = nullptr;
};

inline Vector to_vec(const double* p, Eigen::Index n) {
  Vector v(n);
  for (Eigen::Index i = 0; i < n; ++i) v[i] = p[i];
  return v;
}

inline Matrix to_mat(const double* p, Eigen::Index rows, Eigen::Index cols) {
  Matrix m(rows, cols);
  for (Eigen::Index c = 0; c < cols; ++c)
    for (Eigen::Index r = 0; r < rows; ++r) m(r, c) = p[c * rows + r];
  return m;
}

inline void put(std::vector<double>& dst, std::size_t off, const Vector& v) {
  for (Eigen::Index i = 0; i < v.size(); ++i) dst[off + static_cast<std::size_t>(i)] = v[i];
}

/// theta in the device layout: the reference values, then the family's tail
/// when the caller passed the reference layout alone.
inline void put_theta(std::vector<double>& dst, std::size_t off, const ParameterVector& theta, int nth,
                      const std::vector<double>& tail) {
  const Eigen::Index n = theta.size();
  require(n == nth || n + static_cast<Eigen::Index>(tail.size()) == nth,
          "docp_gpu: theta length does not match the family layout");
  put(dst, off, theta.values());
  if (n < nth)
    for (std::size_t k = 0; k < tail.size(); ++k) dst[off + static_cast<std::size_t>(n) + k] = tail[k];
}

/// QpData and SchurSystem of every problem, from the device (the matrices
/// the forward pass left resident for the backward pass).
inline void materialize(Batch& b, std::vector<SolveResult*>& out) {
  const docp_problem& pr = b.problem();
  const int nx = pr.n_x, nu = pr.n_u, T = pr.horizon, B = b.size();
  const std::size_t X = nx * nx, U = nu * nu, XU = nx * nu;
  std::vector<double> Q(B * (T + 1) * X), q(B * (T + 1) * nx), R(B * T * U), r(B * T * nu), A(B * T * X),
      Bm(B * T * XU), C(B * T * nx), xs(B * nx);
  check(docp_batch_download_qp(b.get(), Q.data(), q.data(), R.data(), r.data(), A.data(), Bm.data(), C.data(),
                               xs.data()));
  std::vector<double> sd(B * (T + 1) * X), ss(B * T * X), pd(B * (T + 1) * X), ps(B * T * X);
  check(docp_batch_download_schur(b.get(), sd.data(), ss.data(), pd.data(), ps.data()));
  auto proj = b.download<int32_t>(DOCP_F_PD_PROJECTED);
  for (int j = 0; j < B; ++j) {
    SolveResult* res = out[j];
    if (!res) continue;
    QpData& qp = res->qp;
    qp = QpData{};
    qp.n_x = nx;
    qp.n_u = nu;
    qp.horizon = T;
    for (int t = 0; t <= T; ++t) {
      qp.Q.push_back(to_mat(&Q[(j * (T + 1) + t) * X], nx, nx));
      qp.q.push_back(to_vec(&q[(j * (T + 1) + t) * nx], nx));
    }
    for (int t = 0; t < T; ++t) {
      qp.R.push_back(to_mat(&R[(j * T + t) * U], nu, nu));
      qp.r.push_back(to_vec(&r[(j * T + t) * nu], nu));
      qp.A_plus.push_back(Matrix::Identity(nx, nx));  // every family: f = x+ - phi(x, u)
      qp.A.push_back(to_mat(&A[(j * T + t) * X], nx, nx));
      qp.B.push_back(to_mat(&Bm[(j * T + t) * XU], nx, nu));
      qp.C.push_back(to_vec(&C[(j * T + t) * nx], nx));
    }
    qp.x_s = to_vec(&xs[j * nx], nx);
    qp.pd_projected = proj[j] != 0;

    SchurSystem& s = res->schur;
    s = SchurSystem{};
    s.n_x = nx;
    s.n_u = nu;
    s.horizon = T;
    for (int t = 0; t <= T; ++t) {
      s.neg_s.diag.push_back(to_mat(&sd[(j * (T + 1) + t) * X], nx, nx));
      s.precond.diag.push_back(to_mat(&pd[(j * (T + 1) + t) * X], nx, nx));
    }
    for (int t = 0; t < T; ++t) {
      Matrix sub = to_mat(&ss[(j * T + t) * X], nx, nx);
      Matrix sup = to_mat(&ps[(j * T + t) * X], nx, nx);
      s.neg_s.super.push_back(sub.transpose());  // schur.hpp:176
      s.neg_s.sub.push_back(std::move(sub));
      s.precond.sub.push_back(sup.transpose());  // schur.hpp:177
      s.precond.super.push_back(std::move(sup));
    }
    for (int t = 0; t <= T; ++t) s.chol_Q.emplace_back(qp.Q[t]);
    for (int t = 0; t < T; ++t) s.chol_R.emplace_back(qp.R[t]);
  }
}

}  // namespace detail

/// A device batch of instances of one family, reused across calls (the
/// train_il / batch_solve working set). Z, LAMBDA and LAMBDA_TILDE of the
/// batch double as the device-resident warm-start cache.
class BatchSolver {
 public:
  BatchSolver(const Family& family, int batch_size, Options opt = {})
      : opt_(opt), tail_(family.theta_tail), b_(std::make_shared<detail::Batch>(family.desc, batch_size, opt)) {}

  int size() const { return b_->size(); }
  detail::Batch& batch() { return *b_; }

  /// sqp_solve for every instance, z0[j], lambda0[j] as initial guesses.
  /// Returns one BatchItem per instance (ok = false with the reference's
  /// message on a per-instance failure, as batch.hpp:98-101).
  std::vector<BatchItem> solve(const std::vector<const ParameterVector*>& thetas, const std::vector<Trajectory>& z0,
                               const std::vector<Vector>& lambda0, const SqpConfig& cfg) {
    cfg.validate();
    const int B = size();
    require(static_cast<int>(thetas.size()) == B && static_cast<int>(z0.size()) == B &&
                static_cast<int>(lambda0.size()) == B,
            "batch: instance count does not match the batch size");
    const docp_problem& pr = b_->problem();
    const int nz = b_->n_z(), nl = b_->n_lambda(), nth = b_->n_theta();
    std::vector<double> th(static_cast<std::size_t>(B) * nth), z(static_cast<std::size_t>(B) * nz),
        l(static_cast<std::size_t>(B) * nl);
    std::vector<BatchItem> items(B);
    std::vector<char> pre_fail(B, 0);
    for (int j = 0; j < B; ++j) {
      try {
        require(z0[j].n_x() == pr.n_x && z0[j].n_u() == pr.n_u && z0[j].horizon() == pr.horizon,
                "trajectory dimensions do not match the problem");  // problem.hpp:62-65
        require(lambda0[j].size() == nl, "sqp: dual guess length mismatch");
        require(z0[j].all_finite() && lambda0[j].allFinite(), "sqp: initial guess must be finite");
        detail::put_theta(th, static_cast<std::size_t>(j) * nth, *thetas[j], nth, tail_);
        detail::put(z, static_cast<std::size_t>(j) * nz, z0[j].flatten());
        detail::put(l, static_cast<std::size_t>(j) * nl, lambda0[j]);
      } catch (const Error& e) {
        pre_fail[j] = 1;
        items[j].error = e.what();
      }
    }
    b_->upload(DOCP_F_THETA, th);
    b_->upload(DOCP_F_Z, z);
    b_->upload(DOCP_F_LAMBDA, l);
    const docp_sqp_config c = detail::to_c(cfg, opt_.mode);
    {
      detail::CountPcg count;
      detail::check(docp_sqp_solve(b_->get(), &c));
    }
    auto zs = b_->download<double>(DOCP_F_Z);
    auto ls = b_->download<double>(DOCP_F_LAMBDA);
    auto st = b_->download<docp_status>(DOCP_F_STATUS);
    auto it = b_->download<int32_t>(DOCP_F_SQP_ITERS);
    auto cv = b_->download<int32_t>(DOCP_F_CONVERGED);
    auto kkt = b_->download<double>(DOCP_F_KKT);
    auto ph = b_->download<int32_t>(DOCP_F_PCG_HISTORY);
    auto ss = b_->download<double>(DOCP_F_STEP_SIZES);
    const std::size_t H = ph.size() / static_cast<std::size_t>(B);  // the library's history stride
    std::vector<SolveResult*> mat(B, nullptr);
    for (int j = 0; j < B; ++j) {
      if (pre_fail[j]) continue;
      if (st[j].code != DOCP_OK) {
        items[j].error = detail::status_message(st[j]);
        continue;
      }
      SolveResult& r = items[j].result;
      items[j].ok = true;
      r.z = Trajectory::unflatten(detail::to_vec(&zs[static_cast<std::size_t>(j) * nz], nz), pr.n_x, pr.n_u,
                                  pr.horizon);
      r.lambda = detail::to_vec(&ls[static_cast<std::size_t>(j) * nl], nl);
      r.sqp_iters = it[j];
      r.converged = cv[j] != 0;
      r.kkt_inf_norm = kkt[j];
      for (int k = 0; k < it[j]; ++k) {
        r.pcg_iters.push_back(ph[static_cast<std::size_t>(j) * H + k]);
        r.step_sizes.push_back(ss[static_cast<std::size_t>(j) * H + k]);
      }
      mat[j] = &r;
    }
    last_status_ = st;
    if (opt_.materialize) detail::materialize(*b_, mat);
    return items;
  }

  /// backward_vjp for every instance of the last solve(), on the matrices
  /// that solve left resident (no re-linearization). Instances whose solve
  /// failed get an empty BackwardResult and `errors[j]` set.
  std::vector<BackwardResult> backward(const std::vector<Vector>& loss_grad_z, const std::vector<Vector>& lambda_tilde0,
                                       const PcgConfig& cfg, std::vector<std::string>* errors = nullptr) {
    const int B = size();
    const int nz = b_->n_z(), nl = b_->n_lambda(), nth = b_->n_theta();
    require(static_cast<int>(loss_grad_z.size()) == B && static_cast<int>(lambda_tilde0.size()) == B,
            "batch: instance count does not match the batch size");
    std::vector<double> g(static_cast<std::size_t>(B) * nz), lt(static_cast<std::size_t>(B) * nl);
    for (int j = 0; j < B; ++j) {
      require(loss_grad_z[j].size() == nz, "backward_vjp: cotangent length mismatch");
      require(lambda_tilde0[j].size() == nl, "backward_vjp: warm start length mismatch");
      detail::put(g, static_cast<std::size_t>(j) * nz, loss_grad_z[j]);
      detail::put(lt, static_cast<std::size_t>(j) * nl, lambda_tilde0[j]);
    }
    b_->upload(DOCP_F_LOSS_GRAD_Z, g);
    b_->upload(DOCP_F_LAMBDA_TILDE, lt);
    const docp_pcg_config c = detail::to_c(cfg, opt_.mode);
    {
      detail::CountPcg count;
      detail::check(docp_backward_vjp(b_->get(), &c));
    }
    auto gt = b_->download<double>(DOCP_F_GRAD_THETA);
    auto lts = b_->download<double>(DOCP_F_LAMBDA_TILDE);
    auto its = b_->download<int32_t>(DOCP_F_PCG_ITERS);
    auto st = b_->download<docp_status>(DOCP_F_STATUS);
    std::vector<BackwardResult> out(B);
    if (errors) errors->assign(B, std::string());
    for (int j = 0; j < B; ++j) {
      if (st[j].code != DOCP_OK) {
        if (errors) (*errors)[j] = detail::status_message(st[j]);
        continue;
      }
      out[j].grad_theta =
          detail::to_vec(&gt[static_cast<std::size_t>(j) * nth], nth - static_cast<Eigen::Index>(tail_.size()));
      out[j].lambda_tilde = detail::to_vec(&lts[static_cast<std::size_t>(j) * nl], nl);
      out[j].pcg_iters = its[j];
    }
    last_status_ = st;
    return out;
  }

  /// docp::rollout (batch.hpp:172-212) of every instance with its own affine
  /// dynamics as the environment and reward -(|x'|^2 + |u|^2) (make_affine_env,
  /// train.hpp:195-213). Returns the total rewards; errors[j] receives the
  /// reference's RolloutTruncation text for a truncated instance.
  std::vector<double> rollout(const std::vector<const ParameterVector*>& thetas, const std::vector<Vector>& x_init,
                              int episode_length, const SqpConfig& cfg, std::vector<std::string>* errors = nullptr) {
    cfg.validate();
    const int B = size(), nth = b_->n_theta(), nx = b_->problem().n_x;
    require(static_cast<int>(thetas.size()) == B && static_cast<int>(x_init.size()) == B,
            "batch: instance count does not match the batch size");
    require(episode_length >= 1, "rollout: episode length must be >= 1");
    std::vector<double> th(static_cast<std::size_t>(B) * nth), x0(static_cast<std::size_t>(B) * nx);
    for (int j = 0; j < B; ++j) {
      require(x_init[j].size() == nx, "rollout: initial state length mismatch");
      detail::put_theta(th, static_cast<std::size_t>(j) * nth, *thetas[j], nth, tail_);
      detail::put(x0, static_cast<std::size_t>(j) * nx, x_init[j]);
    }
    b_->upload(DOCP_F_THETA, th);
    const docp_sqp_config c = detail::to_c(cfg, opt_.mode);
    {
      detail::CountPcg count;
      detail::check(docp_rollout(b_->get(), &c, x0.data(), 0, episode_length));
    }
    auto reward = b_->download<double>(DOCP_F_REWARD);
    roll_status(errors);
    return reward;
  }

  /// docp::rollout_backward (batch.hpp:221-258) of the last rollout:
  /// d(total reward)/d theta per instance, the initial-state segment holding
  /// d/dx_init. Truncated instances get an empty vector.
  std::vector<Vector> rollout_backward(const PcgConfig& cfg, std::vector<std::string>* errors = nullptr) {
    const docp_pcg_config c = detail::to_c(cfg, opt_.mode);
    {
      detail::CountPcg count;
      detail::check(docp_rollout_backward(b_->get(), &c));
    }
    const int nth = b_->n_theta();
    auto g = b_->download<double>(DOCP_F_GRAD_THETA);
    auto st = roll_status(errors);
    std::vector<Vector> out(size());
    for (int j = 0; j < size(); ++j)
      if (st[j].code == DOCP_OK)
        out[j] = detail::to_vec(&g[static_cast<std::size_t>(j) * nth], nth - static_cast<Eigen::Index>(tail_.size()));
    return out;
  }

  const std::vector<docp_status>& last_status() const { return last_status_; }

 private:
  std::vector<docp_status> roll_status(std::vector<std::string>* errors) {
    auto st = b_->download<docp_status>(DOCP_F_ROLLOUT_STATUS);
    if (errors) {
      errors->assign(size(), std::string());
      for (int j = 0; j < size(); ++j)
        if (st[j].code != DOCP_OK) (*errors)[j] = detail::status_message(st[j]);
    }
    last_status_ = st;
    return st;
  }

  Options opt_;
  std::vector<double> tail_;
  std::shared_ptr<detail::Batch> b_;
  std::vector<docp_status> last_status_;
};

/// docp::sqp_solve (sqp.hpp:213-261) on the GPU; throws what the reference throws.
inline SolveResult sqp_solve(const Family& family, const OcpDefinition& ocp, const ParameterVector& theta,
                             const Trajectory& z0, const Vector& lambda0, const SqpConfig& cfg, Options opt = {}) {
  cfg.validate();
  ocp.check_dims(z0);
  require(lambda0.size() == ocp.dual_size(), "sqp: dual guess length mismatch");
  require(z0.all_finite() && lambda0.allFinite(), "sqp: initial guess must be finite");
  require(family.desc.n_x == ocp.n_x && family.desc.n_u == ocp.n_u && family.desc.horizon == ocp.horizon,
          "trajectory dimensions do not match the problem");
  BatchSolver s(family, 1, opt);
  auto items = s.solve({&theta}, {z0}, {lambda0}, cfg);
  if (!items[0].ok) detail::throw_status(s.last_status()[0]);
  return std::move(items[0].result);
}

/// docp::backward_vjp (backward.hpp:27-50) on the GPU, for a forward result
/// from either path. The device re-linearizes and re-assembles at res.z
/// (the same arithmetic the forward pass ends with, sqp.hpp:256-258), then
/// solves the adjoint system warm-started at lambda_tilde0.
inline BackwardResult backward_vjp(const SolveResult& result, const Vector& loss_grad_z, const Vector& lambda_tilde0,
                                   const Family& family, const OcpDefinition& ocp, const ParameterVector& theta,
                                   const PcgConfig& cfg, Options opt = {}) {
  require(loss_grad_z.size() == result.qp.primal_size(), "backward_vjp: cotangent length mismatch");
  require(lambda_tilde0.size() == result.qp.dual_size(), "backward_vjp: warm start length mismatch");
  ocp.check_dims(result.z);
  detail::Batch b(family.desc, 1, opt);
  std::vector<double> th(b.n_theta()), z(b.n_z()), l(b.n_lambda()), g(b.n_z()), lt(b.n_lambda());
  detail::put_theta(th, 0, theta, b.n_theta(), family.theta_tail);
  detail::put(z, 0, result.z.flatten());
  detail::put(l, 0, result.lambda);
  detail::put(g, 0, loss_grad_z);
  detail::put(lt, 0, lambda_tilde0);
  b.upload(DOCP_F_THETA, th);
  b.upload(DOCP_F_Z, z);
  b.upload(DOCP_F_LAMBDA, l);
  b.upload(DOCP_F_LOSS_GRAD_Z, g);
  b.upload(DOCP_F_LAMBDA_TILDE, lt);
  detail::check(docp_linearize(b.get(), opt.eps_pd));
  detail::check(docp_assemble_schur(b.get()));
  auto st = b.download<docp_status>(DOCP_F_STATUS);
  if (st[0].code != DOCP_OK) detail::throw_status(st[0]);
  const docp_pcg_config c = detail::to_c(cfg, opt.mode);
  {
    detail::CountPcg count;
    detail::check(docp_backward_vjp(b.get(), &c));
  }
  st = b.download<docp_status>(DOCP_F_STATUS);
  if (st[0].code != DOCP_OK) detail::throw_status(st[0]);
  BackwardResult out;
  out.grad_theta = detail::to_vec(b.download<double>(DOCP_F_GRAD_THETA).data(),
                                  b.n_theta() - static_cast<Eigen::Index>(family.theta_tail.size()));
  out.lambda_tilde = detail::to_vec(b.download<double>(DOCP_F_LAMBDA_TILDE).data(), b.n_lambda());
  out.pcg_iters = b.download<int32_t>(DOCP_F_PCG_ITERS)[0];
  return out;
}

/// docp::pcg_solve (pcg.hpp:52-109) on the GPU for one stored system.
inline PcgOutcome pcg_solve(const SchurSystem& sys, const Vector& gamma_stored, const Vector& lambda0,
                            const PcgConfig& cfg, Options opt = {}) {
  require(cfg.epsilon > 0.0 && cfg.max_iters >= 0, "pcg: invalid config");
  require(gamma_stored.size() == sys.dim(), "pcg: rhs length mismatch");
  require(lambda0.size() == sys.dim(), "pcg: initial guess length mismatch");
  const int nb = sys.neg_s.n_blocks(), nx = sys.neg_s.block_dim();
  Family f;
  f.desc.family = DOCP_AFFINE_QUADRATIC;  // the system alone fixes the arithmetic; the family is a placeholder
  f.desc.n_x = nx;
  f.desc.n_u = std::max(1, sys.n_u);
  f.desc.horizon = nb - 1;
  f.desc.cost_scale = 1.0;
  detail::Batch b(f.desc, 1, opt);
  const std::size_t X = static_cast<std::size_t>(nx) * nx;
  std::vector<double> sd((nb)*X), ss((nb - 1) * X), pd((nb)*X), ps((nb - 1) * X);
  auto put_m = [&](std::vector<double>& dst, int i, const Matrix& m) {
    for (int c = 0; c < nx; ++c)
      for (int r = 0; r < nx; ++r) dst[i * X + c * nx + r] = m(r, c);
  };
  for (int i = 0; i < nb; ++i) {
    put_m(sd, i, sys.neg_s.diag[i]);
    put_m(pd, i, sys.precond.diag[i]);
  }
  for (int i = 0; i + 1 < nb; ++i) {
    put_m(ss, i, sys.neg_s.sub[i]);
    put_m(ps, i, sys.precond.super[i]);
  }
  detail::check(docp_batch_upload_schur(b.get(), sd.data(), ss.data(), pd.data(), ps.data()));
  std::vector<double> gv(sys.dim()), lv(sys.dim());
  detail::put(gv, 0, gamma_stored);
  detail::put(lv, 0, lambda0);
  b.upload(DOCP_F_GAMMA, gv);
  b.upload(DOCP_F_LAMBDA, lv);
  const docp_pcg_config c = detail::to_c(cfg, opt.mode);
  {
    detail::CountPcg count;
    detail::check(docp_pcg_solve(b.get(), &c, DOCP_F_LAMBDA));
  }
  auto st = b.download<docp_status>(DOCP_F_STATUS);
  if (st[0].code != DOCP_OK) detail::throw_status(st[0]);
  PcgOutcome out;
  out.lambda = detail::to_vec(b.download<double>(DOCP_F_LAMBDA).data(), sys.dim());
  out.iters = b.download<int32_t>(DOCP_F_PCG_ITERS)[0];
  out.final_eta = b.download<double>(DOCP_F_FINAL_ETA)[0];
  out.converged = b.download<int32_t>(DOCP_F_PCG_CONVERGED)[0] != 0;
  return out;
}

/// docp::batch_solve (batch.hpp:83-108) on the GPU: every instance warm-
/// started from its cache slot, failures isolated per instance, the cache
/// updated after the solve and its generation bumped.
inline std::vector<BatchItem> batch_solve(const Family& family, const std::vector<BatchProblem>& instances,
                                          WarmStartCache& cache, const SqpConfig& cfg, Options opt = {}) {
  if (cache.size() != instances.size()) cache.resize(instances.size());
  std::vector<BatchItem> items;
  if (!instances.empty()) {
    std::vector<const ParameterVector*> th;
    std::vector<Trajectory> z0;
    std::vector<Vector> l0;
    for (std::size_t i = 0; i < instances.size(); ++i) {
      const OcpDefinition& ocp = *instances[i].ocp;
      th.push_back(instances[i].theta);
      z0.push_back(cache.warm_z(i, ocp));
      l0.push_back(cache.warm_lambda(i, ocp));
    }
    BatchSolver s(family, static_cast<int>(instances.size()), opt);
    items = s.solve(th, z0, l0, cfg);
  }
  for (std::size_t i = 0; i < items.size(); ++i)
    if (items[i].ok) cache.store(i, items[i].result.z, items[i].result.lambda);
  cache.bump_generation();
  return items;
}

}  // namespace docp::gpu
