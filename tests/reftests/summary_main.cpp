// summary_main.cpp — prints summary_json / trajectory_csv of fixed results
// (test infrastructure). Compiled twice by oracle/Makefile: against the
// reference's own report.cpp (_ref/reftests/summary_ref) and against the
// drop-in (_ref/reftests/summary_dropin); tests/test_report_format.py
// compares the outputs byte for byte.
#include <cmath>
#include <cstdio>
#include <limits>
#include <string>
#include <vector>

#include "aapdhg/lp_model.hpp"
#include "aapdhg/report.hpp"
#include "aapdhg/solver.hpp"

using namespace aapdhg;

int main() {
  const double vals[] = {1.0, 0.9, 1e-6, 1e-4, 0.00012345, 123456789.0, 1e15, 1e16, 2.5e-300,
                         -3.75, 0.1 + 0.2, 1.0 / 3.0, 6.02214076e23, -0.0, 1e300,
                         std::numeric_limits<double>::quiet_NaN(),
                         std::numeric_limits<double>::infinity(), 12345678901234567.0};
  int idx = 0;
  for (double v : vals) {
    SolveResult r;
    r.status = idx % 2 ? SolveStatus::kKktTol : SolveStatus::kResidualTol;
    r.iterations = 12345 + idx;
    r.i = 17;
    r.j = 12345 + idx - 17;
    r.aa_failures = 2;
    r.g_norm = v;
    r.kkt.r_gap = v * 0.5;
    r.kkt.r_primal = 1e-7;
    r.kkt.r_dual = 3e-8;
    r.objective = -v;
    r.steps.tau = 0.0765142689325563;
    r.steps.sigma = 0.0765142689325563;
    r.wall_seconds = 1.25;
    SolverConfig cfg;
    cfg.method = idx % 3 == 0 ? Method::kAaPdhg : idx % 3 == 1 ? Method::kFaaPdhg : Method::kPdhg;
    cfg.m = 10;
    cfg.safeguard_d = idx % 2 ? 1.0 : 0.5;
    cfg.safeguard_eps = 1.0;
    cfg.filter.c_s = std::sqrt(1.0 - 0.99 * 0.99);
    cfg.filter.kappa_bar = 1e4;
    cfg.toll = 1e-6;
    cfg.kkt_terminate = idx % 2 == 1;
    if (idx % 4 == 2) cfg.aa.d_hat = {0.5, 1.0, v};
    ProblemData p;
    p.name = idx % 5 == 0 ? "tab\there \"quoted\"\n" : "config" + std::to_string(idx);
    p.maximize = idx % 2 == 0;
    std::fputs(summary_json(r, cfg, p).c_str(), stdout);
    std::vector<TrajectoryRecord> recs(2);
    recs[0].k = 0;
    recs[0].g_norm = v;
    recs[1].k = 1;
    recs[1].aa_step = true;
    recs[1].objective = v * 3;
    std::fputs(trajectory_csv(recs).c_str(), stdout);
    ++idx;
  }
  return 0;
}
