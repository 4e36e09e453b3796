// docp_gpu — the reference CLI's `solve` and `grad-check` commands on the
// B200 path.
//
// Mirrors proj/tools/docp_main.cpp: same sub-commands, global options
// (--seed, --workers, --out), outputs (solution.json, gradcheck.json with the
// "docp-bench/1" meta header), stdout lines and exit codes (2 solver
// failure, 3 invalid input). Problem files are `aq-ocp/1`
// (problems/affine_quadratic_io.hpp:9-77). Host code talks to the GPU only
// through the C ABI (include/docp_cuda.h); there is no CPU solver here.
//
// One addition: --mode parity|fast picks the PCG arithmetic.
// The default is parity, so the written solution is bit-identical to the
// reference's.
//
// grad-check follows run_grad_check (docp_main.cpp:97-175): one-shot SQP
// (max_sqp_iters = 1, alpha = {1}), the adjoint gradient of the weighted
// quadratic loss, and central finite differences with step 1e-6
// (oracle.hpp:143-158). The 2 * dim(theta) perturbed solves run as ONE
// batched GPU solve instead of a sequential loop.
#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <filesystem>
#include <fstream>
#include <iostream>
#include <sstream>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "docp_cuda.h"
#include "json_lite.hpp"

namespace {

constexpr int kExitSolverFailure = 2;
constexpr int kExitInvalidInput = 3;
constexpr const char* kProblemFormat = "aq-ocp/1";  // affine_quadratic_io.hpp:9

class InvalidInput : public std::runtime_error {
 public:
  using std::runtime_error::runtime_error;
};
/// docp::Error raised by the solver (rendered from a device status word).
class SolverFailure : public std::runtime_error {
 public:
  using std::runtime_error::runtime_error;
};

/// AffineQuadratic fields of an aq-ocp/1 file (affine_quadratic_io.hpp:40-77).
struct AqProblem {
  int n_x = 0, n_u = 0, horizon = 0;
  std::vector<double> w_x, w_u, A, B, b_affine, x_s;  // A, B column-major

  /// make_theta (affine_quadratic.hpp:27-37): [w_x | w_u | vec A | vec B | b | x_s].
  std::vector<double> theta() const {
    std::vector<double> t;
    for (const auto* v : {&w_x, &w_u, &A, &B, &b_affine, &x_s}) t.insert(t.end(), v->begin(), v->end());
    return t;
  }
  docp_problem desc() const {
    docp_problem d{};
    d.family = DOCP_AFFINE_QUADRATIC;
    d.n_x = n_x;
    d.n_u = n_u;
    d.horizon = horizon;
    d.cost_scale = 1.0;  // the file convention (affine_quadratic_io.hpp:11-12)
    return d;
  }
  /// ParameterVector::segments() of make_theta, in std::map (name) order.
  std::vector<std::pair<std::string, std::pair<int, int>>> segments() const {
    const int dyn = n_x * n_x + n_x * n_u + n_x;
    return {{"control_cost", {n_x, n_u}},
            {"dynamics", {n_x + n_u, dyn}},
            {"initial_state", {n_x + n_u + dyn, n_x}},
            {"state_cost", {0, n_x}}};
  }
};

void require_file(bool cond, const std::string& msg) {
  if (!cond) throw InvalidInput(msg);
}

/// affine_quadratic_from_json (affine_quadratic_io.hpp:40-77) + load_problem
/// (docp_main.cpp:25-38), with the same messages.
AqProblem load_problem(const std::string& path) {
  std::ifstream in(path);
  if (!in) throw InvalidInput("cannot open problem file: " + path);
  std::stringstream ss;
  ss << in.rdbuf();
  try {
    const json_lite::value j = json_lite::value::parse(ss.str());
    if (!j.contains("format") || j.at("format").as_string() != kProblemFormat)
      throw InvalidInput("problem file: missing or unsupported format key");
    AqProblem p;
    p.n_x = j.at("n_x").as_int();
    p.n_u = j.at("n_u").as_int();
    p.horizon = j.at("T").as_int();
    require_file(p.n_x >= 1 && p.n_u >= 1 && p.horizon >= 1, "problem file: dimensions must be positive");
    auto vec = [](const json_lite::value& a, int n, const char* name) {
      std::vector<double> v = a.as_doubles();
      require_file(static_cast<int>(v.size()) == n, std::string("problem file: bad length for ") + name);
      return v;
    };
    auto mat = [](const json_lite::value& a, int rows, int cols, const char* name) {
      const auto& rv = a.elements();
      require_file(static_cast<int>(rv.size()) == rows, std::string("problem file: bad row count for ") + name);
      std::vector<double> m(static_cast<std::size_t>(rows) * cols);
      for (int i = 0; i < rows; ++i) {
        std::vector<double> row = rv[i].as_doubles();
        require_file(static_cast<int>(row.size()) == cols, std::string("problem file: bad column count for ") + name);
        for (int c = 0; c < cols; ++c) m[static_cast<std::size_t>(c) * rows + i] = row[c];
      }
      return m;
    };
    p.w_x = vec(j.at("Q"), p.n_x, "Q");
    p.w_u = vec(j.at("R"), p.n_u, "R");
    p.A = mat(j.at("A"), p.n_x, p.n_x, "A");
    p.B = mat(j.at("B"), p.n_x, p.n_u, "B");
    p.b_affine = vec(j.at("b_affine"), p.n_x, "b_affine");
    p.x_s = vec(j.at("x_s"), p.n_x, "x_s");
    return p;
  } catch (const json_lite::error& e) {
    throw InvalidInput("problem file is not valid JSON: " + std::string(e.what()));
  }
}

struct GlobalOptions {
  std::uint64_t seed = 0;
  unsigned workers = 0;  // 0: DOCP_WORKERS or hardware default
  std::string out_dir = ".";
  int mode = DOCP_PCG_PARITY;
};

/// docp::default_workers (common.hpp:62-72); reported in the meta header only.
unsigned default_workers() {
  if (const char* env = std::getenv("DOCP_WORKERS")) {
    long n = std::strtol(env, nullptr, 10);
    if (n >= 1) return static_cast<unsigned>(n);
  }
  unsigned hw = std::thread::hardware_concurrency();
  return hw == 0 ? 1u : hw;
}

json_lite::value meta_header(const std::string& command, const GlobalOptions& g) {
  json_lite::value meta = json_lite::value::object();
  meta["format"] = "docp-bench/1";
  meta["command"] = command;
  meta["seed"] = static_cast<unsigned long long>(g.seed);
  meta["workers"] = g.workers == 0 ? default_workers() : g.workers;
  return meta;
}

/// bench::write_json (report_io.hpp:42-47).
void write_json(const std::filesystem::path& path, const json_lite::value& j) {
  std::ofstream out(path);
  if (!out) throw SolverFailure("cannot open output file: " + path.string());
  out << j.dump(2) << "\n";
}

void check(int rc) {
  if (rc != 0) throw std::runtime_error(std::string("docp_cuda: ") + docp_last_error());
}

/// SqpConfig defaults (sqp.hpp:7-34) with the CLI's overrides.
docp_sqp_config sqp_config(int max_sqp_iters, const std::vector<double>& alphas, int mode) {
  docp_sqp_config c{};
  c.max_sqp_iters = max_sqp_iters;
  c.n_step_candidates = static_cast<int32_t>(alphas.size());
  for (std::size_t i = 0; i < alphas.size(); ++i) c.step_candidates[i] = alphas[i];
  c.eta_armijo = 0.4;
  c.rho_penalty = 0.5;
  c.pcg.epsilon = 1e-12;
  c.pcg.max_iters = 0;
  c.pcg.mode = mode;
  c.convergence_tol = 1e-8;
  c.mu_floor_denominator = 1e-12;
  c.eps_pd = 1e-6;
  return c;
}

/// RAII batch of B affine-quadratic instances on device 0.
class Batch {
 public:
  Batch(const docp_problem& d, int n) : d_(d), n_(n) {
    check(docp_batch_create(&d_, n, 0, &b_));
    nth_ = docp_theta_size(&d_);
    nz_ = d.n_x * (d.horizon + 1) + d.n_u * d.horizon;
    nl_ = d.n_x * (d.horizon + 1);
  }
  ~Batch() { docp_batch_destroy(b_); }
  Batch(const Batch&) = delete;
  Batch& operator=(const Batch&) = delete;

  docp_batch* get() { return b_; }
  int n_z() const { return nz_; }
  int n_lambda() const { return nl_; }
  int n_theta() const { return nth_; }
  template <class T>
  void upload(int field, const std::vector<T>& v) {
    check(docp_batch_upload(b_, field, v.data(), 0));
  }
  template <class T>
  std::vector<T> download(int field, std::size_t per) {
    std::vector<T> v(per * static_cast<std::size_t>(n_));
    check(docp_batch_download(b_, field, v.data(), 0));
    return v;
  }
  /// First failing instance, rendered with the reference's exception text.
  void throw_on_failure() {
    auto st = download<docp_status>(DOCP_F_STATUS, 1);
    for (const auto& s : st) {
      if (s.code != DOCP_OK) {
        char buf[512];
        docp_format_status(&s, buf, sizeof buf);
        throw SolverFailure(buf);
      }
    }
  }

 private:
  docp_problem d_;
  int n_;
  docp_batch* b_ = nullptr;
  int nth_ = 0, nz_ = 0, nl_ = 0;
};

/// Trajectory columns (docp_main.cpp:40-54): x as T+1 columns of n_x, u as T of n_u.
json_lite::value trajectory_json(const AqProblem& p, const double* z) {
  const int nx = p.n_x, nu = p.n_u, T = p.horizon;
  json_lite::value x = json_lite::value::array(), u = json_lite::value::array();
  for (int t = 0; t <= T; ++t) {
    const double* xt = z + static_cast<std::size_t>(t) * (nx + nu);  // flat_offset (trajectory.hpp:72-74)
    x.push_back(std::vector<double>(xt, xt + nx));
    if (t < T) u.push_back(std::vector<double>(xt + nx, xt + nx + nu));
  }
  json_lite::value j = json_lite::value::object();
  j["x"] = x;
  j["u"] = u;
  return j;
}

/// run_solve (docp_main.cpp:67-95).
int run_solve(const std::string& path, const GlobalOptions& g) {
  AqProblem prob = load_problem(path);
  Batch b(prob.desc(), 1);
  b.upload(DOCP_F_THETA, prob.theta());
  b.upload(DOCP_F_Z, std::vector<double>(b.n_z(), 0.0));
  b.upload(DOCP_F_LAMBDA, std::vector<double>(b.n_lambda(), 0.0));
  const docp_sqp_config cfg = sqp_config(20, {1.0, 0.7, 0.3, 0.1, 0.01}, g.mode);
  check(docp_sqp_solve(b.get(), &cfg));
  b.throw_on_failure();
  const auto z = b.download<double>(DOCP_F_Z, b.n_z());
  const auto lam = b.download<double>(DOCP_F_LAMBDA, b.n_lambda());
  const int sqp_iters = b.download<int32_t>(DOCP_F_SQP_ITERS, 1)[0];
  const auto hist = b.download<int32_t>(DOCP_F_PCG_HISTORY, cfg.max_sqp_iters);
  const double kkt = b.download<double>(DOCP_F_KKT, 1)[0];
  const bool converged = b.download<int32_t>(DOCP_F_CONVERGED, 1)[0] != 0;

  json_lite::value out = meta_header("solve", g);
  out["problem"] = path;
  out["trajectory"] = trajectory_json(prob, z.data());
  out["lambda"] = lam;
  out["sqp_iters"] = sqp_iters;
  out["pcg_iters"] = std::vector<int>(hist.begin(), hist.begin() + sqp_iters);
  out["kkt_inf_norm"] = kkt;
  out["converged"] = converged;
  std::filesystem::create_directories(g.out_dir);
  write_json(std::filesystem::path(g.out_dir) / "solution.json", out);
  std::cout << "solved " << path << ": sqp_iters=" << sqp_iters << " kkt_inf_norm=" << kkt
            << " converged=" << (converged ? "yes" : "no") << "\n";
  return 0;
}

/// run_grad_check (docp_main.cpp:97-175).
int run_grad_check(const std::string& path, double tol, const GlobalOptions& g) {
  AqProblem prob = load_problem(path);
  const int nx = prob.n_x, nu = prob.n_u, T = prob.horizon;
  const docp_sqp_config cfg = sqp_config(1, {1.0}, g.mode);

  std::vector<double> check_w(nx + nu);
  for (int i = 0; i < nx + nu; ++i) check_w[i] = 1.0 + 0.5 * std::sin(static_cast<double>(i) + 1.0);
  // loss.value: sum_t x_t'(W_x x_t), then sum_t u_t'(W_u u_t) (docp_main.cpp:115-122)
  auto loss_value = [&](const double* z) {
    double acc = 0.0;
    for (int t = 0; t <= T; ++t) {
      const double* x = z + static_cast<std::size_t>(t) * (nx + nu);
      double d = x[0] * (check_w[0] * x[0]);
      for (int e = 1; e < nx; ++e) d += x[e] * (check_w[e] * x[e]);
      acc += d;
    }
    for (int t = 0; t < T; ++t) {
      const double* u = z + static_cast<std::size_t>(t) * (nx + nu) + nx;
      double d = u[0] * (check_w[nx] * u[0]);
      for (int e = 1; e < nu; ++e) d += u[e] * (check_w[nx + e] * u[e]);
      acc += d;
    }
    return acc;
  };

  const std::vector<double> theta = prob.theta();
  const int nth = static_cast<int>(theta.size());

  // base solve + adjoint gradient (docp_main.cpp:130-137)
  std::vector<double> grad;
  {
    Batch b(prob.desc(), 1);
    b.upload(DOCP_F_THETA, theta);
    b.upload(DOCP_F_Z, std::vector<double>(b.n_z(), 0.0));
    b.upload(DOCP_F_LAMBDA, std::vector<double>(b.n_lambda(), 0.0));
    check(docp_sqp_solve(b.get(), &cfg));
    b.throw_on_failure();
    const auto z = b.download<double>(DOCP_F_Z, b.n_z());
    std::vector<double> gz(b.n_z());  // loss.grad: 2 W z (docp_main.cpp:123-128)
    for (int t = 0; t <= T; ++t) {
      const std::size_t o = static_cast<std::size_t>(t) * (nx + nu);
      for (int e = 0; e < nx; ++e) gz[o + e] = 2.0 * check_w[e] * z[o + e];
      if (t < T)
        for (int e = 0; e < nu; ++e) gz[o + nx + e] = 2.0 * check_w[nx + e] * z[o + nx + e];
    }
    b.upload(DOCP_F_LOSS_GRAD_Z, gz);
    b.upload(DOCP_F_LAMBDA_TILDE, std::vector<double>(b.n_lambda(), 0.0));
    check(docp_backward_vjp(b.get(), &cfg.pcg));
    b.throw_on_failure();
    grad = b.download<double>(DOCP_F_GRAD_THETA, nth);
  }

  // fd_gradient (oracle.hpp:143-158): every +-step solve in one batch,
  // instance 2i = theta + step e_i, 2i + 1 = theta - step e_i
  const double step = 1e-6;
  std::vector<double> fd(nth);
  {
    Batch b(prob.desc(), 2 * nth);
    std::vector<double> th(static_cast<std::size_t>(2 * nth) * nth);
    for (int i = 0; i < nth; ++i) {
      double* up = th.data() + static_cast<std::size_t>(2 * i) * nth;
      double* dn = up + nth;
      std::copy(theta.begin(), theta.end(), up);
      std::copy(theta.begin(), theta.end(), dn);
      up[i] = theta[i] + step;
      dn[i] = theta[i] - step;
    }
    b.upload(DOCP_F_THETA, th);
    b.upload(DOCP_F_Z, std::vector<double>(static_cast<std::size_t>(2 * nth) * b.n_z(), 0.0));
    b.upload(DOCP_F_LAMBDA, std::vector<double>(static_cast<std::size_t>(2 * nth) * b.n_lambda(), 0.0));
    check(docp_sqp_solve(b.get(), &cfg));
    b.throw_on_failure();
    const auto z = b.download<double>(DOCP_F_Z, b.n_z());
    for (int i = 0; i < nth; ++i) {
      const double up = loss_value(z.data() + static_cast<std::size_t>(2 * i) * b.n_z());
      const double down = loss_value(z.data() + static_cast<std::size_t>(2 * i + 1) * b.n_z());
      if (!std::isfinite(up) || !std::isfinite(down)) throw SolverFailure("fd_gradient: non-finite evaluation");
      fd[i] = (up - down) / (2.0 * step);
    }
  }

  json_lite::value out = meta_header("grad-check", g);
  out["problem"] = path;
  double overall = 0.0;
  for (const auto& [name, range] : prob.segments()) {
    double seg_max = 0.0;
    for (int i = range.first; i < range.first + range.second; ++i) {
      double rel = std::abs(grad[i] - fd[i]) / std::max(1e-8, std::abs(fd[i]));
      seg_max = std::max(seg_max, rel);
    }
    out["max_rel_error"][name] = seg_max;
    overall = std::max(overall, seg_max);
    std::cout << "segment " << name << ": max rel error " << seg_max << "\n";
  }
  out["overall_max_rel_error"] = overall;
  out["tolerance"] = tol;
  out["pass"] = overall <= tol;
  std::filesystem::create_directories(g.out_dir);
  write_json(std::filesystem::path(g.out_dir) / "gradcheck.json", out);
  std::cout << "overall max rel error " << overall << (overall <= tol ? " (pass)" : " (FAIL)") << "\n";
  return overall <= tol ? 0 : kExitSolverFailure;
}

void usage(std::ostream& os) {
  os << "Differentiable optimal-control solver (B200 path)\n"
        "usage: docp_gpu [--seed N] [--workers N] [--out DIR] [--mode parity|fast] <command>\n"
        "  solve <problem.json>                 solve a problem file\n"
        "  grad-check <problem.json> [--tol X]  check solver gradients against finite differences\n";
}

}  // namespace

int main(int argc, char** argv) {
  GlobalOptions g;
  std::string command, problem;
  double tol = 1e-5;
  try {
    std::vector<std::string> args(argv + 1, argv + argc);
    for (std::size_t i = 0; i < args.size(); ++i) {
      const std::string& a = args[i];
      auto next = [&]() -> const std::string& {
        if (i + 1 >= args.size()) throw InvalidInput(a + " requires an argument");
        return args[++i];
      };
      if (a == "-h" || a == "--help") {
        usage(std::cout);
        return 0;
      } else if (a == "--seed") {
        g.seed = std::stoull(next());
      } else if (a == "--workers") {
        g.workers = static_cast<unsigned>(std::stoul(next()));
      } else if (a == "--out") {
        g.out_dir = next();
      } else if (a == "--mode") {
        const std::string& m = next();
        if (m != "parity" && m != "fast") throw InvalidInput("--mode must be parity or fast");
        g.mode = m == "parity" ? DOCP_PCG_PARITY : DOCP_PCG_FAST;
      } else if (a == "--tol" && command == "grad-check") {
        tol = std::stod(next());
      } else if (command.empty()) {
        if (a != "solve" && a != "grad-check") throw InvalidInput("unknown command: " + a);
        command = a;
      } else if (problem.empty()) {
        problem = a;
      } else {
        throw InvalidInput("unexpected argument: " + a);
      }
    }
    if (command.empty() || problem.empty()) {
      usage(std::cerr);
      return 1;  // CLI11's exit code for a missing required argument
    }
  } catch (const std::logic_error& e) {  // std::stoull and friends
    std::cerr << "invalid argument: " << e.what() << "\n";
    return 1;
  } catch (const InvalidInput& e) {
    std::cerr << e.what() << "\n";
    return 1;
  }

  try {
    if (command == "solve") return run_solve(problem, g);
    return run_grad_check(problem, tol, g);
  } catch (const InvalidInput& e) {
    std::cerr << "invalid input: " << e.what() << "\n";
    return kExitInvalidInput;
  } catch (const SolverFailure& e) {
    std::cerr << "solver failure: " << e.what() << "\n";
    return kExitSolverFailure;
  } catch (const std::exception& e) {  // CUDA / ABI failures: loud, never a CPU fallback
    std::cerr << "error: " << e.what() << "\n";
    return 1;
  }
}
