// aapdhg/aapdhg.hpp — drop-in C++ API of the B200 AA-PDHG / FAA-PDHG solver.
//
// Source-compatible with the reference library's public interface for the
// solve path (namespace aapdhg; the reference's per-module header names —
// solver.hpp, lp_model.hpp, sparse_linalg.hpp, pdhg_core.hpp, anderson.hpp,
// filtering.hpp, report.hpp, errors.hpp, vec.hpp — each include this file).
// Reference declarations mirrored (paths relative to the reference checkout):
//   errors            proj/include/aapdhg/errors.hpp:8-30
//   Vec, kInf, dot..  proj/include/aapdhg/vec.hpp:12-55
//   SparseMatrix ..   proj/include/aapdhg/sparse_linalg.hpp:10-72
//   ProblemData ..    proj/include/aapdhg/lp_model.hpp:14-68
//   Iterate ..        proj/include/aapdhg/pdhg_core.hpp:9-45
//   AAParams          proj/include/aapdhg/anderson.hpp:21-25
//   FilterParams      proj/include/aapdhg/filtering.hpp:14-17
//   solver types/API  proj/include/aapdhg/solver.hpp:15-99
//   report            proj/include/aapdhg/report.hpp:11-20 (in aapdhg/report.hpp)
// Every numeric entry point runs on the sm_100a library through the C-ABI in
// aapdhg_cuda.h; there is no CPU fallback.
#pragma once

#include <cmath>
#include <cstddef>
#include <cstdint>
#include <iosfwd>
#include <limits>
#include <stdexcept>
#include <string>
#include <unordered_map>
#include <utility>
#include <vector>

namespace aapdhg {

// ---- errors ------------------------------------------------------------------
struct Error : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct InputError : Error {  // bad input / configuration
  using Error::Error;
};
struct UnsupportedError : Error {  // deliberately out of scope
  using Error::Error;
};
struct SingularError : Error {  // degenerate small solve (AA falls back)
  using Error::Error;
};
struct DimensionError : Error {  // size mismatch
  using Error::Error;
};

// ---- dense vectors -----------------------------------------------------------
using Vec = std::vector<double>;
inline constexpr double kInf = std::numeric_limits<double>::infinity();

double dot(const Vec& a, const Vec& b);
double nrm2sq(const Vec& a);
inline double nrm2(const Vec& a) { return std::sqrt(nrm2sq(a)); }
void axpy(double alpha, const Vec& x, Vec& y);
Vec sub(const Vec& a, const Vec& b);
Vec add(const Vec& a, const Vec& b);
Vec scaled(const Vec& a, double alpha);

// ---- sparse matrices ---------------------------------------------------------
struct Triplet {
  int row = 0;
  int col = 0;
  double val = 0.0;
};

// CSR; column indices strictly increasing per row.
struct SparseMatrix {
  int nrows = 0;
  int ncols = 0;
  std::vector<int> row_ptr;
  std::vector<int> col_idx;
  std::vector<double> vals;

  // Sorts by (row, col) and sums duplicates (left to right).
  static SparseMatrix from_triplets(int nrows, int ncols, std::vector<Triplet> entries);
  std::size_t nnz() const { return vals.size(); }
};

SparseMatrix vstack(const SparseMatrix& a, const SparseMatrix& b);

// Products on the device (CSR-ordered sums: bit-identical to the reference).
void matvec(const SparseMatrix& m, const Vec& v, Vec& out);
// Column-major dense matrix, sparse_linalg.hpp:46-58 (test support / small
// algebra; the device path keeps its p x p systems in shared memory).
struct DenseMatrix {
  int nrows = 0;
  int ncols = 0;
  std::vector<double> data;  // nrows * ncols, column-major
  DenseMatrix() = default;
  DenseMatrix(int r, int c) : nrows(r), ncols(c), data(std::size_t(r) * std::size_t(c), 0.0) {}
  double& at(int i, int j) { return data[std::size_t(j) * std::size_t(nrows) + std::size_t(i)]; }
  double at(int i, int j) const { return data[std::size_t(j) * std::size_t(nrows) + std::size_t(i)]; }
  static DenseMatrix identity(int n);
};

Vec matvec(const SparseMatrix& m, const Vec& v);
void matvec_transpose(const SparseMatrix& m, const Vec& v, Vec& out);
Vec matvec_transpose(const SparseMatrix& m, const Vec& v);
double power_iteration_norm(const SparseMatrix& m, int max_iters, double rel_tol,
                            std::uint64_t seed);

// ---- the LP ------------------------------------------------------------------
struct RawLP {
  std::string name;
  bool maximize = false;
  std::string objective_name;
  std::vector<std::string> row_names;
  std::vector<char> row_sense;  // 'E', 'G', 'L'
  std::vector<std::string> col_names;
  Vec obj_coeffs;
  std::vector<Triplet> entries;
  Vec rhs;
  Vec lower, upper;
  std::vector<bool> is_integer;
  std::unordered_map<std::string, int> row_index;
  std::unordered_map<std::string, int> col_index;
};

// min c'x  s.t.  Gx >= h, Ax = b, l <= x <= u;  K = [G; A], q = [h; b].
struct ProblemData {
  SparseMatrix g, a;
  Vec c, h, b;
  Vec l, u;
  SparseMatrix k;
  Vec q;
  bool maximize = false;
  std::string name;
  std::vector<std::string> row_names_g, row_names_a, col_names;

  int n() const { return int(c.size()); }
  int m1() const { return g.nrows; }
  int m2() const { return a.nrows; }
};

enum class LambdaTag { kZero, kNonpos, kNonneg, kFree };
using LambdaSpec = std::vector<LambdaTag>;

RawLP parse_mps(std::istream& in);
RawLP parse_mps_file(const std::string& path);
ProblemData to_standard_form(const RawLP& raw);
LambdaSpec build_lambda_set(const Vec& l, const Vec& u);
std::string emit_mps(const ProblemData& p);

// ---- iterates / parameters ------------------------------------------------------
struct Iterate {
  Vec x;
  Vec y;
};

struct StepSizes {
  double tau = 0.0;
  double sigma = 0.0;
};

// projections, pdhg_core.hpp (host helpers; the device path fuses them)
Vec project_box(const Vec& x, const Vec& l, const Vec& u);
Vec project_dual(const Vec& y, int m1);
Vec project_lambda(const Vec& v, const LambdaSpec& spec);
Iterate project_feasible(const Iterate& u, const ProblemData& p);
Iterate pdhg_step(const Iterate& u, const ProblemData& p, const StepSizes& s);
std::pair<Vec, double> fixed_point_residual(const Iterate& u, const Iterate& tu);
// <Mu, v>, M = [[I, tau K'], [sigma K, I]], tau == sigma (pdhg_core.hpp:39-42;
// a diagnostic of the reference, products on the device)
double m_inner_product(const Vec& u, const Vec& v, const ProblemData& p, const StepSizes& s);
Vec concat_iterate(const Iterate& u);
Iterate split_iterate(const Vec& v, int n);

struct AAParams {
  double beta = 1.0;
  Vec d_hat;           // empty = identity
  double eta = 1e-10;  // applied as eta * ||dG||_F^2
};

struct FilterParams {
  double c_s = 0.2;
  double kappa_bar = 1e9;
};

// ---- Anderson memory, anderson.hpp:12-48 -------------------------------------------
// Columns oldest to newest, equal counts, at most `capacity` pairs.
struct AAMemory {
  std::vector<Vec> du_cols;
  std::vector<Vec> dg_cols;
  std::size_t capacity = 5;
  std::size_t size() const { return du_cols.size(); }
  bool empty() const { return du_cols.empty(); }
};

// Appends at the newest end, evicts the oldest beyond capacity.
void memory_push(AAMemory& mem, Vec du, Vec dg);
// beta * Dhat * v (empty d_hat: identity).
Vec damp(const AAParams& params, const Vec& v);
// The accelerated candidate u - H g (anderson.hpp:36-41), on the device
// (aapdhg_cuda_aa_apply: the regularised Gram, Cholesky and mix of the solve
// loop). Throws SingularError when the normal equations are not PD.
Vec aa_apply(const AAMemory& mem, const AAParams& params, const Vec& u, const Vec& g);
// Alg-1 test oracles (anderson.hpp:43-48): affine weights minimising
// ||sum alpha_i r_i|| with sum alpha = 1 (minimum-norm solution for a
// degenerate Gram), and (1-beta) sum alpha_i points_i + beta sum alpha_i images_i.
Vec standard_aa_weights(const std::vector<Vec>& residuals);
Vec standard_aa_step(const std::vector<Vec>& points, const std::vector<Vec>& images,
                     const Vec& weights, double beta);

// ---- QR, sparse_linalg.hpp:60-72 -------------------------------------------------------
struct QRFactors {
  DenseMatrix q;  // n x p, orthonormal columns
  DenseMatrix r;  // p x p, upper triangular, nonnegative diagonal
};
// On the device: R from the double-double Gram F'F (aapdhg_cuda_economy_qr),
// Q = F R^{-1}. p <= n (DimensionError otherwise); SingularError for
// rank-deficient columns.
QRFactors economy_qr(const DenseMatrix& f);
// R X = B for upper-triangular R; SingularError when a diagonal entry is
// <= 1e-14 ||R||_F.
DenseMatrix back_substitute(const DenseMatrix& r, const DenseMatrix& b);
Vec back_substitute(const DenseMatrix& r, const Vec& b);

// ---- FAA filtering, filtering.hpp:14-59 -------------------------------------------
using ColumnList = std::vector<Vec>;

struct FilteredMemory {
  ColumnList e;  // iterate differences
  ColumnList f;  // residual differences
  QRFactors qr;  // economy QR of f
  std::size_t size() const { return f.size(); }
  bool empty() const { return f.empty(); }
};

std::pair<ColumnList, ColumnList> reverse_columns(ColumnList e, ColumnList f);
// The kept sets below come from the device FAA step (aapdhg_cuda_faa_op).
std::pair<ColumnList, ColumnList> angle_filter(ColumnList e, ColumnList f, double c_s);
Vec length_bounds(const ColumnList& f, double c_s);
std::pair<ColumnList, ColumnList> length_filter(ColumnList e, ColumnList f, double c_s,
                                                double kappa_bar);
FilteredMemory build_filtered_memory(ColumnList e, ColumnList f, const FilterParams& params);
// w = R^{-1} Q'g (as the least squares of the kept f, on the device), then
// u + beta Dhat g - sum_j (e_j + beta Dhat f_j) w_j.
Vec filtered_aa_apply(const FilteredMemory& fm, const AAParams& params, const Vec& u,
                      const Vec& g);

// ---- solver ------------------------------------------------------------------
enum class Method { kPdhg, kAaPdhg, kFaaPdhg };

enum class SolveStatus { kResidualTol, kKktTol, kMaxIters, kTimeout, kFixedPointStart };

// B200 extension (not in the reference): order of the device reductions.
// kAuto = kSerial for n + m <= 65536 (bit-identical to the reference), else
// kTree (deterministic blocked trees).
enum class Reduction { kAuto, kSerial, kTree };

struct SolverConfig {
  Method method = Method::kPdhg;
  std::size_t m = 5;
  double safeguard_d = 1.0;
  double safeguard_eps = 1.0;
  AAParams aa;
  FilterParams filter;
  double toll = 1e-4;
  double kkt_eps = 1e-4;
  bool kkt_terminate = false;
  std::size_t max_iters = 100000;
  double max_wall_seconds = 3600.0;
  double tau = 0.0;
  double sigma = 0.0;
  Reduction reduction = Reduction::kAuto;  // B200 extension
  int device = 0;                          // B200 extension: CUDA device
};

struct KktMetrics {
  double r_gap = 0.0;
  double r_primal = 0.0;
  double r_dual = 0.0;
  double max() const;
};

struct TrajectoryRecord {
  std::size_t k = 0;
  double g_norm = 0.0;
  bool aa_step = false;
  std::size_t i = 0;
  std::size_t j = 0;
  KktMetrics kkt;
  double objective = 0.0;
  double elapsed_s = 0.0;
};

struct SolveResult {
  SolveStatus status = SolveStatus::kMaxIters;
  Iterate u;
  Vec lambda;
  std::size_t iterations = 0;
  std::size_t i = 0;
  std::size_t j = 0;
  std::size_t aa_failures = 0;
  double g_norm = 0.0;
  KktMetrics kkt;
  double objective = 0.0;
  StepSizes steps;
  double wall_seconds = 0.0;
};

struct SolveOutput {
  SolveResult result;
  std::vector<TrajectoryRecord> trajectory;
};

bool safeguard_pass(double g_norm, double g0_norm, std::size_t i, double d, double eps);
std::pair<KktMetrics, Vec> kkt_metrics(const Iterate& u, const ProblemData& p,
                                       const LambdaSpec& spec);
StepSizes select_step_sizes(const ProblemData& p, const SolverConfig& cfg);
SolveOutput solve(const ProblemData& p, const SolverConfig& cfg, const Iterate& u0);
SolveOutput solve(const ProblemData& p, const SolverConfig& cfg);

// A problem kept resident on the device for repeated solves (sweeps).
class DeviceProblem {
 public:
  explicit DeviceProblem(const ProblemData& p, int device = 0);
  ~DeviceProblem();
  DeviceProblem(const DeviceProblem&) = delete;
  DeviceProblem& operator=(const DeviceProblem&) = delete;
  SolveOutput solve(const SolverConfig& cfg, const Iterate& u0) const;
  SolveOutput solve(const SolverConfig& cfg) const;
  void* handle() const { return h_; }

 private:
  const ProblemData* p_;
  void* h_ = nullptr;
};

// ---- sweep mode ---------------------------------------------------------------
// The CLI's --sweep-D/--sweep-eps/--sweep-m/--sweep-kappa-bar cross product
// (proj/src/cli.cpp:155-180), with the same case names ("D0.5_eps1_m10" ...).
struct SweepCase {
  SolverConfig cfg;
  std::string name;
};
std::vector<SweepCase> sweep_cases(const SolverConfig& base, const std::vector<double>& d,
                                   const std::vector<double>& eps,
                                   const std::vector<std::size_t>& m,
                                   const std::vector<double>& kappa_bar);

struct SweepOutcome {
  bool ok = false;
  std::string error;   // the exception message when !ok
  SolveOutput output;  // valid when ok
};
// Runs the cases on `workers` threads (cli.cpp:184-209: AAPDHG_SWEEP_WORKERS
// when workers == 0). Each worker keeps one DeviceProblem resident on its
// device (devices are assigned round-robin; several workers per GPU run
// concurrently on their own streams — small LPs leave a GPU mostly idle) and
// takes cases from a shared counter. Outcomes are in case order.
std::vector<SweepOutcome> solve_sweep(const ProblemData& p, const std::vector<SweepCase>& cases,
                                      std::size_t workers = 0,
                                      const std::vector<int>& devices = {0});

// (report: status_name / method_name / trajectory_csv / summary_json are
// declared in aapdhg/report.hpp only, as in the reference — code that does
// not include it may define its own status_name, e.g. acceptance_test.cpp)

}  // namespace aapdhg
