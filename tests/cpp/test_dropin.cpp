// test_dropin.cpp — the C++ drop-in (include/docp_gpu.hpp) against the
// reference's own functions, in the style of the reference's Catch2 suite
// (proj/tests/test_sqp.cpp, test_backward.cpp, test_pcg.cpp, test_batch.cpp).
//
// Both sides run in this binary: docp::X is the reference header-only CPU
// implementation (compiled against oracle/eigen_lite, test infrastructure),
// docp::gpu::X is the CUDA path through libdocp_cuda.so. PARITY mode must
// be bit-identical for the affine-quadratic family; cart-pole and FAST mode
// must match iteration counts and agree to 1e-9 relative.
// Needs a GPU; built by build.py when the reference headers are present.
#include <catch2/catch_amalgamated.hpp>

#include <cmath>
#include <random>

#include "docp/bench/generators.hpp"
#include "docp/bench/train.hpp"
#include "docp_gpu.hpp"

using namespace docp;

namespace {

gpu::Options parity() { return gpu::Options{}; }
gpu::Options fast() {
  gpu::Options o;
  o.mode = DOCP_PCG_FAST;
  return o;
}

bool same(const Vector& a, const Vector& b) {
  if (a.size() != b.size()) return false;
  for (Eigen::Index i = 0; i < a.size(); ++i)
    if (!(a[i] == b[i])) return false;
  return true;
}

bool same(const Matrix& a, const Matrix& b) {
  if (a.rows() != b.rows() || a.cols() != b.cols()) return false;
  for (Eigen::Index c = 0; c < a.cols(); ++c)
    for (Eigen::Index r = 0; r < a.rows(); ++r)
      if (!(a(r, c) == b(r, c))) return false;
  return true;
}

double rel(const Vector& a, const Vector& b) {
  return (a - b).norm() / std::max(1.0, b.norm());
}

AffineQuadratic instance(int nx, int nu, int T, unsigned seed) {
  std::mt19937_64 rng(seed);
  return bench::random_convex_instance(nx, nu, T, rng);
}

Vector loss_grad(const Trajectory& z, unsigned seed) {
  std::mt19937_64 rng(seed);
  std::normal_distribution<double> n(0.0, 1.0);
  Vector g(z.flat_size());
  for (Eigen::Index i = 0; i < g.size(); ++i) g[i] = n(rng);
  return g;
}

}  // namespace

TEST_CASE("gpu sqp_solve reproduces sqp_solve bit for bit (affine-quadratic)") {
  for (unsigned seed : {1u, 2u, 3u}) {
    AffineQuadratic p = instance(8, 4, 30, seed);
    OcpDefinition ocp = p.make_ocp();
    ParameterVector theta = p.make_theta();
    Trajectory z0(8, 4, 30);
    SqpConfig cfg;
    cfg.max_sqp_iters = 5;
    SolveResult cpu = sqp_solve(ocp, theta, z0, Vector::Zero(ocp.dual_size()), cfg);
    SolveResult dev = gpu::sqp_solve(gpu::family_of(p), ocp, theta, z0, Vector::Zero(ocp.dual_size()), cfg, parity());
    CHECK(same(dev.z.flatten(), cpu.z.flatten()));
    CHECK(same(dev.lambda, cpu.lambda));
    CHECK(dev.sqp_iters == cpu.sqp_iters);
    CHECK(dev.converged == cpu.converged);
    CHECK(dev.pcg_iters == cpu.pcg_iters);
    CHECK(dev.step_sizes == cpu.step_sizes);
    CHECK(dev.kkt_inf_norm == cpu.kkt_inf_norm);
    // the cached matrices the backward pass consumes
    for (int t = 0; t <= 30; ++t) {
      CHECK(same(dev.qp.Q[t], cpu.qp.Q[t]));
      CHECK(same(dev.qp.q[t], cpu.qp.q[t]));
      CHECK(same(dev.schur.neg_s.diag[t], cpu.schur.neg_s.diag[t]));
      CHECK(same(dev.schur.precond.diag[t], cpu.schur.precond.diag[t]));
    }
    for (int t = 0; t < 30; ++t) {
      CHECK(same(dev.qp.A[t], cpu.qp.A[t]));
      CHECK(same(dev.qp.B[t], cpu.qp.B[t]));
      CHECK(same(dev.qp.C[t], cpu.qp.C[t]));
      CHECK(same(dev.schur.neg_s.sub[t], cpu.schur.neg_s.sub[t]));
      CHECK(same(dev.schur.neg_s.super[t], cpu.schur.neg_s.super[t]));
      CHECK(same(dev.schur.precond.super[t], cpu.schur.precond.super[t]));
      CHECK(same(dev.schur.precond.sub[t], cpu.schur.precond.sub[t]));
    }
    CHECK(same(dev.qp.x_s, cpu.qp.x_s));
  }
}

TEST_CASE("gpu backward_vjp reproduces backward_vjp bit for bit, one PCG solve") {
  AffineQuadratic p = instance(8, 4, 40, 7);
  OcpDefinition ocp = p.make_ocp();
  ParameterVector theta = p.make_theta();
  SqpConfig cfg;
  cfg.max_sqp_iters = 5;
  SolveResult res = sqp_solve(ocp, theta, Trajectory(8, 4, 40), Vector::Zero(ocp.dual_size()), cfg);
  Vector g = loss_grad(res.z, 11);
  Vector lt0 = Vector::Zero(ocp.dual_size());
  BackwardResult cpu = backward_vjp(res, g, lt0, ocp, theta, cfg.pcg);
  const auto before = stats::pcg_invocations().load();
  BackwardResult dev = gpu::backward_vjp(res, g, lt0, gpu::family_of(p), ocp, theta, cfg.pcg, parity());
  CHECK(stats::pcg_invocations().load() - before == 1);  // test_backward.cpp:93-107
  CHECK(same(dev.grad_theta, cpu.grad_theta));
  CHECK(same(dev.lambda_tilde, cpu.lambda_tilde));
  CHECK(dev.pcg_iters == cpu.pcg_iters);
  // warm start from the previous adjoint: fewer or equal iterations, same bits as the CPU
  BackwardResult cpu2 = backward_vjp(res, g, cpu.lambda_tilde, ocp, theta, cfg.pcg);
  BackwardResult dev2 = gpu::backward_vjp(res, g, dev.lambda_tilde, gpu::family_of(p), ocp, theta, cfg.pcg, parity());
  CHECK(dev2.pcg_iters == cpu2.pcg_iters);
  CHECK(same(dev2.grad_theta, cpu2.grad_theta));
}

TEST_CASE("a GPU SolveResult feeds the reference backward_vjp") {
  AffineQuadratic p = instance(8, 4, 30, 5);
  OcpDefinition ocp = p.make_ocp();
  ParameterVector theta = p.make_theta();
  SqpConfig cfg;
  cfg.max_sqp_iters = 5;
  SolveResult dev = gpu::sqp_solve(gpu::family_of(p), ocp, theta, Trajectory(8, 4, 30),
                                   Vector::Zero(ocp.dual_size()), cfg, parity());
  SolveResult cpu = sqp_solve(ocp, theta, Trajectory(8, 4, 30), Vector::Zero(ocp.dual_size()), cfg);
  Vector g = loss_grad(cpu.z, 3);
  Vector lt0 = Vector::Zero(ocp.dual_size());
  BackwardResult from_dev = backward_vjp(dev, g, lt0, ocp, theta, cfg.pcg);
  BackwardResult from_cpu = backward_vjp(cpu, g, lt0, ocp, theta, cfg.pcg);
  CHECK(same(from_dev.grad_theta, from_cpu.grad_theta));
  CHECK(from_dev.pcg_iters == from_cpu.pcg_iters);
}

TEST_CASE("gpu pcg_solve on a reference-assembled system") {
  AffineQuadratic p = instance(8, 4, 50, 9);
  OcpDefinition ocp = p.make_ocp();
  ParameterVector theta = p.make_theta();
  QpData qp = linearize(ocp, Trajectory(8, 4, 50), theta, kDefaultEpsPd);
  SchurSystem sys = assemble_schur(qp);
  Vector gamma = assemble_gamma(qp, sys, qp.flat_b(), qp.flat_d());
  PcgConfig pc;
  SECTION("cold start, parity") {
    PcgOutcome cpu = pcg_solve(sys, gamma, Vector::Zero(sys.dim()), pc);
    PcgOutcome dev = gpu::pcg_solve(sys, gamma, Vector::Zero(sys.dim()), pc, parity());
    CHECK(dev.iters == cpu.iters);
    CHECK(dev.converged == cpu.converged);
    CHECK(dev.final_eta == cpu.final_eta);
    CHECK(same(dev.lambda, cpu.lambda));
  }
  SECTION("cold start, fast: equal count, 1e-9") {
    PcgOutcome cpu = pcg_solve(sys, gamma, Vector::Zero(sys.dim()), pc);
    PcgOutcome dev = gpu::pcg_solve(sys, gamma, Vector::Zero(sys.dim()), pc, fast());
    CHECK(dev.iters == cpu.iters);
    CHECK(rel(dev.lambda, cpu.lambda) <= 1e-9);
  }
  SECTION("exact warm start costs zero iterations") {  // test_pcg.cpp:63-78
    PcgOutcome cpu = pcg_solve(sys, gamma, Vector::Zero(sys.dim()), pc);
    PcgOutcome dev = gpu::pcg_solve(sys, gamma, cpu.lambda, pc, parity());
    PcgOutcome cpu2 = pcg_solve(sys, gamma, cpu.lambda, pc);
    CHECK(dev.iters == cpu2.iters);
    CHECK(same(dev.lambda, cpu2.lambda));
  }
  SECTION("iteration cap") {
    PcgConfig capped;
    capped.max_iters = 3;
    PcgOutcome cpu = pcg_solve(sys, gamma, Vector::Zero(sys.dim()), capped);
    PcgOutcome dev = gpu::pcg_solve(sys, gamma, Vector::Zero(sys.dim()), capped, parity());
    CHECK(dev.iters == 3);
    CHECK_FALSE(dev.converged);
    CHECK(dev.final_eta == cpu.final_eta);
    CHECK(same(dev.lambda, cpu.lambda));
  }
  SECTION("invalid config and length checks throw DimensionError") {
    PcgConfig bad;
    bad.epsilon = 0.0;
    CHECK_THROWS_AS(gpu::pcg_solve(sys, gamma, Vector::Zero(sys.dim()), bad), DimensionError);
    CHECK_THROWS_AS(gpu::pcg_solve(sys, gamma, Vector::Zero(sys.dim() - 1), pc), DimensionError);
  }
}

TEST_CASE("gpu pcg_solve reports breakdown like the reference") {  // test_pcg.cpp:80-120
  const int nb = 4, bd = 2;
  SchurSystem sys;
  sys.n_x = bd;
  sys.n_u = 1;
  sys.horizon = nb - 1;
  sys.neg_s = BlockTridiag::identity(nb, bd);
  sys.precond = BlockTridiag::identity(nb, bd);
  sys.neg_s.diag[2] = -Matrix::Identity(bd, bd);  // indefinite
  Vector gamma = Vector::Zero(nb * bd);
  gamma[4] = 1.0;
  std::string cpu_msg, dev_msg;
  int cpu_it = -1, dev_it = -2;
  try {
    pcg_solve(sys, gamma, Vector::Zero(nb * bd), PcgConfig{});
  } catch (const BreakdownError& e) {
    cpu_msg = e.what();
    cpu_it = e.iteration;
  }
  try {
    gpu::pcg_solve(sys, gamma, Vector::Zero(nb * bd), PcgConfig{}, parity());
  } catch (const BreakdownError& e) {
    dev_msg = e.what();
    dev_it = e.iteration;
  }
  CHECK(!cpu_msg.empty());
  CHECK(dev_msg == cpu_msg);
  CHECK(dev_it == cpu_it);
}

TEST_CASE("gpu batch_solve: warm cache, failure isolation, generation") {  // test_batch.cpp:7-43
  const int n = 6;
  std::vector<AffineQuadratic> probs;
  std::vector<OcpDefinition> ocps;
  std::vector<ParameterVector> thetas;
  for (int i = 0; i < n; ++i) {
    probs.push_back(instance(4, 2, 20, 100 + i));
    ocps.push_back(probs.back().make_ocp());
    thetas.push_back(probs.back().make_theta());
  }
  // instance 3 evaluates to a non-finite state cost at stage 0
  Vector vals = thetas[3].values();
  vals[0] = std::numeric_limits<double>::infinity();
  thetas[3].values() = vals;
  std::vector<BatchProblem> inst(n);
  for (int i = 0; i < n; ++i) inst[i] = BatchProblem{&ocps[i], &thetas[i]};
  SqpConfig cfg;
  cfg.max_sqp_iters = 4;
  WarmStartCache cpu_cache, dev_cache;
  for (int round = 0; round < 2; ++round) {
    auto cpu = batch_solve(inst, cpu_cache, cfg, 1);
    auto dev = gpu::batch_solve(gpu::family_of(probs[0]), inst, dev_cache, cfg, parity());
    REQUIRE(dev.size() == cpu.size());
    for (int i = 0; i < n; ++i) {
      CHECK(dev[i].ok == cpu[i].ok);
      CHECK(dev[i].error == cpu[i].error);
      if (!cpu[i].ok || !dev[i].ok) continue;
      CHECK(same(dev[i].result.z.flatten(), cpu[i].result.z.flatten()));
      CHECK(same(dev[i].result.lambda, cpu[i].result.lambda));
      CHECK(dev[i].result.pcg_iters == cpu[i].result.pcg_iters);
    }
    CHECK(dev_cache.generation() == cpu_cache.generation());
  }
  CHECK(dev_cache.warm_lambda(0, ocps[0]).cwiseAbs().maxCoeff() > 0.0);
}

TEST_CASE("gpu sqp_solve: errors and argument checks match the reference") {
  AffineQuadratic p = instance(4, 2, 10, 4);
  OcpDefinition ocp = p.make_ocp();
  ParameterVector theta = p.make_theta();
  SqpConfig cfg;
  CHECK_THROWS_AS(gpu::sqp_solve(gpu::family_of(p), ocp, theta, Trajectory(4, 2, 9), Vector::Zero(ocp.dual_size()), cfg),
                  DimensionError);
  CHECK_THROWS_AS(gpu::sqp_solve(gpu::family_of(p), ocp, theta, Trajectory(4, 2, 10), Vector::Zero(3), cfg),
                  DimensionError);
  SqpConfig bad = cfg;
  bad.step_candidates = {0.5, 1.0};
  CHECK_THROWS_AS(gpu::sqp_solve(gpu::family_of(p), ocp, theta, Trajectory(4, 2, 10), Vector::Zero(ocp.dual_size()), bad),
                  DimensionError);
  Vector vals = theta.values();
  vals[0] = std::nan("");
  ParameterVector broken = theta;
  broken.values() = vals;
  std::string cpu_msg, dev_msg;
  try {
    sqp_solve(ocp, broken, Trajectory(4, 2, 10), Vector::Zero(ocp.dual_size()), cfg);
  } catch (const EvaluationError& e) {
    cpu_msg = e.what();
  }
  try {
    gpu::sqp_solve(gpu::family_of(p), ocp, broken, Trajectory(4, 2, 10), Vector::Zero(ocp.dual_size()), cfg);
  } catch (const EvaluationError& e) {
    dev_msg = e.what();
  }
  CHECK(!cpu_msg.empty());
  CHECK(dev_msg == cpu_msg);
}

TEST_CASE("gpu cart-pole: equal iteration counts, 1e-9 relative") {
  CartpoleParams params;
  params.horizon = 40;
  OcpDefinition ocp = make_cartpole_ocp(params);
  std::mt19937_64 rng(5);
  std::uniform_real_distribution<double> u(-0.5, 0.5);
  for (int k = 0; k < 3; ++k) {
    Vector x0(4);
    x0 << u(rng), u(rng), 2.0 * u(rng), u(rng);
    ParameterVector theta = make_cartpole_theta((Vector(4) << 1, 2, 1.5, 1).finished(), 0.05, x0);
    Trajectory z0(4, 1, 40);
    z0.x.colwise() = x0;
    SqpConfig cfg;
    cfg.max_sqp_iters = 5;
    for (const gpu::Options& o : {parity(), fast()}) {
      SolveResult cpu = sqp_solve(ocp, theta, z0, Vector::Zero(ocp.dual_size()), cfg);
      SolveResult dev = gpu::sqp_solve(gpu::family_of(params), ocp, theta, z0, Vector::Zero(ocp.dual_size()), cfg, o);
      CHECK(dev.sqp_iters == cpu.sqp_iters);
      CHECK(dev.pcg_iters == cpu.pcg_iters);
      CHECK(rel(dev.z.flatten(), cpu.z.flatten()) <= 1e-9);
      CHECK(rel(dev.lambda, cpu.lambda) <= 1e-9);
      Vector g = loss_grad(cpu.z, 17 + k);
      BackwardResult bc = backward_vjp(cpu, g, Vector::Zero(ocp.dual_size()), ocp, theta, cfg.pcg);
      BackwardResult bd = gpu::backward_vjp(dev, g, Vector::Zero(ocp.dual_size()), gpu::family_of(params), ocp, theta,
                                            cfg.pcg, o);
      CHECK(bd.pcg_iters == bc.pcg_iters);
      CHECK(rel(bd.grad_theta, bc.grad_theta) <= 1e-9);
    }
  }
}

TEST_CASE("gpu BatchSolver: train_il inner loop (solve, loss, backward) matches the reference") {  // train.hpp:82-109
  const int n = 8, T = 20;
  std::vector<AffineQuadratic> probs;
  std::vector<ParameterVector> thetas;
  std::vector<const ParameterVector*> tp;
  for (int i = 0; i < n; ++i) {
    probs.push_back(instance(8, 4, T, 200 + i));
    thetas.push_back(probs.back().make_theta());
  }
  for (auto& t : thetas) tp.push_back(&t);
  OcpDefinition ocp0 = probs[0].make_ocp();
  SqpConfig cfg;
  cfg.max_sqp_iters = 5;
  gpu::BatchSolver solver(gpu::family_of(probs[0]), n, parity());
  std::vector<Trajectory> z0(n, Trajectory(8, 4, T));
  std::vector<Vector> l0(n, Vector::Zero(ocp0.dual_size()));
  auto items = solver.solve(tp, z0, l0, cfg);
  std::vector<Vector> grads, lts(n, Vector::Zero(ocp0.dual_size()));
  for (int i = 0; i < n; ++i) grads.push_back(loss_grad(items[i].result.z, 50 + i));
  auto back = solver.backward(grads, lts, cfg.pcg);
  for (int i = 0; i < n; ++i) {
    OcpDefinition ocp = probs[i].make_ocp();
    SolveResult cpu = sqp_solve(ocp, thetas[i], z0[i], l0[i], cfg);
    REQUIRE(items[i].ok);
    CHECK(same(items[i].result.z.flatten(), cpu.z.flatten()));
    BackwardResult bc = backward_vjp(cpu, grads[i], lts[i], ocp, thetas[i], cfg.pcg);
    CHECK(same(back[i].grad_theta, bc.grad_theta));
    CHECK(back[i].pcg_iters == bc.pcg_iters);
  }
}

TEST_CASE("gpu BatchSolver: rollout + rollout_backward match the reference (affine env)") {  // batch.hpp:172-258
  const int n = 5, T = 20, H = 4;
  std::mt19937_64 rng(11);
  std::vector<AffineQuadratic> probs;
  std::vector<ParameterVector> thetas;
  std::vector<const ParameterVector*> tp;
  std::vector<Vector> x0;
  for (int i = 0; i < n; ++i) {
    probs.push_back(bench::random_linear_instance(4, 2, T, rng));
    thetas.push_back(probs.back().make_theta());
    x0.push_back(probs.back().x_s);
  }
  for (auto& t : thetas) tp.push_back(&t);
  SqpConfig cfg;
  cfg.max_sqp_iters = 1;
  cfg.step_candidates = {1.0};  // make_linear_rl_task's real-time mode (train.hpp:226-230)
  gpu::BatchSolver solver(gpu::family_of(probs[0]), n, parity());
  std::vector<std::string> errs;
  auto rewards = solver.rollout(tp, x0, H, cfg, &errs);
  auto grads = solver.rollout_backward(cfg.pcg, &errs);
  for (int i = 0; i < n; ++i) {
    OcpDefinition ocp = probs[i].make_ocp();
    DiffEnv env = bench::make_affine_env(probs[i]);
    RolloutOutput roll = rollout(env, ocp, thetas[i], x0[i], H, cfg);
    Vector g = rollout_backward(roll.record, env, ocp, thetas[i], cfg.pcg);
    CHECK(errs[i].empty());
    CHECK(rewards[i] == roll.total_reward);
    CHECK(same(grads[i], g));
  }
}

TEST_CASE("gpu attitude family: sqp_solve, backward_vjp and rollouts match the reference") {  // attitude.hpp
  AttitudeParams params;
  params.inertia = (Vector(3) << 1.5, 0.7, 1.1).finished();
  params.horizon = 25;
  OcpDefinition ocp = make_attitude_ocp(params);
  ParameterVector theta =
      make_attitude_theta(Vector::Ones(3), Vector::Ones(3), (Vector(3) << 0.4, -0.8, 0.3).finished());
  SqpConfig cfg;
  cfg.max_sqp_iters = 4;  // make_attitude_rl_task (train.hpp:258-261)
  Trajectory z0(3, 3, 25);
  SolveResult cpu = sqp_solve(ocp, theta, z0, Vector::Zero(ocp.dual_size()), cfg);
  SolveResult dev = gpu::sqp_solve(gpu::family_of(params), ocp, theta, z0, Vector::Zero(ocp.dual_size()), cfg,
                                   parity());
  CHECK(same(dev.z.flatten(), cpu.z.flatten()));
  CHECK(dev.pcg_iters == cpu.pcg_iters);
  Vector g = loss_grad(cpu.z, 5);
  BackwardResult bc = backward_vjp(cpu, g, Vector::Zero(ocp.dual_size()), ocp, theta, cfg.pcg);
  BackwardResult bd =
      gpu::backward_vjp(dev, g, Vector::Zero(ocp.dual_size()), gpu::family_of(params), ocp, theta, cfg.pcg, parity());
  CHECK(same(bd.grad_theta, bc.grad_theta));
  // rollouts with the attitude RL environment (train.hpp:239-263)
  DiffEnv env = make_diff_env([params](const Vector& x, const Vector& u) { return attitude_step(params, x, u); },
                              [](const Vector& x, const Vector& u) { return -(0.1 * x.squaredNorm() + u.squaredNorm()); },
                              [](const Vector& x, const Vector& u) {
                                return std::make_pair(Vector(-0.2 * x), Vector(-2.0 * u));
                              });
  Vector x0 = theta.segment(segment::initial_state);
  RolloutOutput roll = rollout(env, ocp, theta, x0, 3, cfg);
  Vector gr = rollout_backward(roll.record, env, ocp, theta, cfg.pcg);
  gpu::BatchSolver solver(gpu::family_of(params), 1, parity());
  auto rewards = solver.rollout({&theta}, {x0}, 3, cfg);
  auto grads = solver.rollout_backward(cfg.pcg);
  CHECK(rewards[0] == roll.total_reward);
  CHECK(same(grads[0], gr));
}
