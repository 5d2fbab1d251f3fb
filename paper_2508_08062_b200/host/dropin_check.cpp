// dropin_check.cpp — end-to-end checks written against the drop-in C++ API
// exactly as a user of the reference library would (cf. the reference's
// acceptance checks 1, 9, 10: proj/tests/acceptance_test.cpp:103-137,
// 511-579, 584-650). Prints one JSON object; tests/test_gpu_dropin.py
// asserts on it. Needs a B200.
#include <algorithm>
#include <cstdio>
#include <fstream>
#include <random>
#include <sstream>
#include <string>

#include "aapdhg/lp_model.hpp"
#include "aapdhg/report.hpp"
#include "aapdhg/solver.hpp"

using namespace aapdhg;

static ProblemData toy() {  // min 0 x  s.t. x = 3, x >= 0
  ProblemData p;
  p.a = SparseMatrix::from_triplets(1, 1, {{0, 0, 1.0}});
  p.g = SparseMatrix::from_triplets(0, 1, {});
  p.c = {0.0};
  p.b = {3.0};
  p.l = {0.0};
  p.u = {kInf};
  p.k = vstack(p.g, p.a);
  p.q = p.b;
  p.name = "toy";
  p.row_names_a = {"R1"};
  p.col_names = {"X1"};
  return p;
}

// transport in inequality form (demand covered, supply capacity)
static ProblemData transport(int S, int T, unsigned seed) {
  std::mt19937_64 rng(seed);
  std::uniform_int_distribution<int> cost(1, 4), amount(1, 5);
  ProblemData p;
  const int n = S * T;
  p.c.resize(std::size_t(n));
  for (auto& v : p.c) v = cost(rng);
  std::vector<Triplet> t;
  for (int j = 0; j < T; ++j) {
    for (int i = 0; i < S; ++i) t.push_back({j, i * T + j, 1.0});
    p.h.push_back(amount(rng));
  }
  for (int i = 0; i < S; ++i) {
    for (int j = 0; j < T; ++j) t.push_back({T + i, i * T + j, -1.0});
    p.h.push_back(-2.0 * amount(rng) * T / S - 5.0);
  }
  p.g = SparseMatrix::from_triplets(S + T, n, std::move(t));
  p.a = SparseMatrix::from_triplets(0, n, {});
  p.l.assign(std::size_t(n), 0.0);
  p.u.assign(std::size_t(n), kInf);
  p.k = vstack(p.g, p.a);
  p.q = p.h;
  p.name = "transport";
  for (int r = 0; r < S + T; ++r) p.row_names_g.push_back("R" + std::to_string(r + 1));
  for (int j = 0; j < n; ++j) p.col_names.push_back("X" + std::to_string(j + 1));
  return p;
}

int main() {
  std::string js = "{";
  auto put = [&](const std::string& k, const std::string& v) {
    if (js.size() > 1) js += ", ";
    js += "\"" + k + "\": " + v;
  };
  // 1. toy: plain vs accelerated (proj/test_output.txt:21)
  const ProblemData t = toy();
  SolverConfig plain;
  plain.method = Method::kPdhg;
  plain.toll = 1e-4;
  plain.tau = plain.sigma = 0.25;
  plain.max_iters = 1000;
  const SolveOutput po = solve(t, plain);
  SolverConfig accel = plain;
  accel.method = Method::kAaPdhg;
  const SolveOutput ao = solve(t, accel);
  accel.method = Method::kFaaPdhg;
  const SolveOutput fo = solve(t, accel);
  put("toy_pdhg_iterations", std::to_string(po.result.iterations));
  put("toy_pdhg_status", "\"" + std::string(status_name(po.result.status)) + "\"");
  put("toy_aa_iterations", std::to_string(ao.result.iterations));
  put("toy_faa_iterations", std::to_string(fo.result.iterations));
  put("toy_aa_x", std::to_string(ao.result.u.x[0]));

  // 2. MPS round trip (emit -> parse -> standard form) then solve
  const std::string mps = emit_mps(t);
  std::istringstream in(mps);
  const ProblemData t2 = to_standard_form(parse_mps(in));
  const SolveOutput ro = solve(t2, plain);
  put("mps_roundtrip_iterations", std::to_string(ro.result.iterations));

  // 3. safeguard bookkeeping (acceptance check 9)
  int accel_records = 0;
  bool book_ok = true;
  for (const Method m : {Method::kAaPdhg, Method::kFaaPdhg}) {
    SolverConfig c = plain;
    c.method = m;
    c.toll = 1e-9;
    c.max_iters = 5000;
    c.safeguard_d = m == Method::kAaPdhg ? 1.0 : 2.0;
    c.safeguard_eps = m == Method::kAaPdhg ? 1.0 : 0.01;
    c.m = m == Method::kAaPdhg ? 5 : 8;
    const SolveOutput o = solve(t, c);
    const double g0 = o.trajectory.front().g_norm;
    book_ok = book_ok && o.trajectory.size() == o.result.iterations + 1 &&
              o.result.i + o.result.j == o.result.iterations;
    for (const auto& r : o.trajectory) {
      if (!r.aa_step) continue;
      ++accel_records;
      book_ok = book_ok && safeguard_pass(r.g_norm, g0, r.i, c.safeguard_d, c.safeguard_eps);
    }
  }
  put("bookkeeping_ok", book_ok ? "true" : "false");
  put("accel_records", std::to_string(accel_records));

  // 4. mid-size separation (acceptance check 10 style): FAA lead over PDHG
  const ProblemData tr = transport(40, 40, 7);
  SolverConfig base;
  base.toll = 1e-14;
  base.max_iters = 3000;
  SolverConfig pc = base;
  pc.method = Method::kPdhg;
  const SolveOutput tp = solve(tr, pc);
  SolverConfig fc = base;
  fc.method = Method::kFaaPdhg;
  fc.m = 10;
  fc.safeguard_d = 10.0;
  fc.safeguard_eps = 0.01;
  const SolveOutput tf = solve(tr, fc);
  double best = 1e300;
  for (std::size_t k = 0; k < std::min(tp.trajectory.size(), tf.trajectory.size()); ++k)
    if (tp.trajectory[k].g_norm > 0.0)
      best = std::min(best, tf.trajectory[k].g_norm / tp.trajectory[k].g_norm);
  char buf[64];
  std::snprintf(buf, sizeof buf, "%.3e", best);
  put("transport_nnz", std::to_string(tr.k.nnz()));
  put("transport_best_ratio", buf);

  // 5. outputs in the reference formats
  const std::string csv = trajectory_csv(ao.trajectory);
  const std::string sum = summary_json(ao.result, accel, t);
  put("csv_rows", std::to_string(std::count(csv.begin(), csv.end(), '\n')));
  put("summary_has_status", sum.find("\"status\": \"RESIDUAL_TOL\"") != std::string::npos ? "true" : "false");

  // 6. errors map onto the reference exception types
  bool threw = false;
  try {
    SolverConfig bad;
    bad.m = 0;
    (void)solve(t, bad);
  } catch (const InputError&) {
    threw = true;
  }
  put("input_error_thrown", threw ? "true" : "false");

  // 7. sweep mode (cli.cpp:142-214): D x m cross product on 3 workers, each
  // outcome equal to the same case solved alone
  SolverConfig sb;
  sb.method = Method::kAaPdhg;
  sb.toll = 1e-4;
  sb.tau = sb.sigma = 0.25;
  const std::vector<SweepCase> cases = sweep_cases(sb, {1.0, 1e-300}, {}, {2, 5}, {});
  const std::vector<SweepOutcome> sw = solve_sweep(t, cases, 3, {0});
  bool sweep_ok = sw.size() == 4;
  std::string names;
  for (std::size_t i = 0; i < cases.size() && sweep_ok; ++i) {
    names += (i ? "," : "") + cases[i].name;
    const SolveOutput alone = solve(t, cases[i].cfg);
    sweep_ok = sw[i].ok && sw[i].output.result.iterations == alone.result.iterations &&
               sw[i].output.result.u.x == alone.result.u.x &&
               sw[i].output.trajectory.size() == alone.trajectory.size();
    if (!sweep_ok)
      std::fprintf(stderr, "sweep case %s: ok %d error '%s' iterations %zu vs %zu alone, records %zu vs %zu\n",
                   cases[i].name.c_str(), int(sw[i].ok), sw[i].error.c_str(),
                   sw[i].output.result.iterations, alone.result.iterations,
                   sw[i].output.trajectory.size(), alone.trajectory.size());
  }
  put("sweep_ok", sweep_ok ? "true" : "false");
  js += ", \"sweep_names\": \"" + names + "\"";
  js += "}";
  std::printf("%s\n", js.c_str());
  return 0;
}
