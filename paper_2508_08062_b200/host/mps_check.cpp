// mps_check — round trip of the drop-in's MPS front end at scale (SURVEY.md
// §8(f) f3; tests/test_gpu_dropin.py): builds a random four-block LP with
// E, G and L rows, integer markers and every bound type, writes it with
// emit_mps, reads it back with parse_mps_file (mmap + threaded COLUMNS
// tokenising) and to_standard_form (device CSR assembly), and checks the
// result equals the original exactly. Prints one JSON line.
//   mps_check <rows> <cols> <nnz_per_col> <seed> <path>
//   mps_check parse <path>        (the reader alone, host only)
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <fstream>
#include <random>
#include <string>
#include <vector>

#include "aapdhg/aapdhg.hpp"

using namespace aapdhg;

// `mps_check parse <path>`: the reader alone (host only, no device): the
// RawLP as JSON, or {"error": kind, "what": message}
static int parse_only(const char* path) {
  try {
    const RawLP lp = parse_mps_file(path);
    double osum = 0.0, esum = 0.0, rsum = 0.0;
    long long rowsum = 0, colsum = 0;
    for (double v : lp.obj_coeffs) osum += v;
    for (const Triplet& t : lp.entries) {
      esum += t.val;
      rowsum += t.row;
      colsum += t.col;
    }
    for (double v : lp.rhs) rsum += v;
    int nint = 0;
    for (bool b : lp.is_integer) nint += b;
    int ninf_lo = 0, ninf_up = 0;
    for (double v : lp.lower) ninf_lo += std::isinf(v);
    for (double v : lp.upper) ninf_up += std::isinf(v);
    std::string senses(lp.row_sense.begin(), lp.row_sense.end());
    std::printf("{\"name\": \"%s\", \"objective\": \"%s\", \"maximize\": %s, \"rows\": %zu, "
                "\"cols\": %zu, \"entries\": %zu, \"senses\": \"%s\", \"obj_sum\": %.17g, "
                "\"entry_sum\": %.17g, \"rhs_sum\": %.17g, \"row_index_sum\": %lld, "
                "\"col_index_sum\": %lld, \"integer\": %d, \"inf_lower\": %d, "
                "\"inf_upper\": %d, \"first_col\": \"%s\", \"last_col\": \"%s\"}\n",
                lp.name.c_str(), lp.objective_name.c_str(), lp.maximize ? "true" : "false",
                lp.row_names.size(), lp.col_names.size(), lp.entries.size(), senses.c_str(), osum,
                esum, rsum, rowsum, colsum, nint, ninf_lo, ninf_up,
                lp.col_names.empty() ? "" : lp.col_names.front().c_str(),
                lp.col_names.empty() ? "" : lp.col_names.back().c_str());
    return 0;
  } catch (const UnsupportedError& e) {
    std::printf("{\"error\": \"UnsupportedError\", \"what\": \"%s\"}\n", e.what());
  } catch (const InputError& e) {
    std::printf("{\"error\": \"InputError\", \"what\": \"%s\"}\n", e.what());
  }
  return 3;
}

int main(int argc, char** argv) {
  if (argc == 3 && std::string(argv[1]) == "parse") return parse_only(argv[2]);
  if (argc != 6) {
    std::fprintf(stderr, "usage: mps_check <rows> <cols> <nnz_per_col> <seed> <path>\n");
    return 2;
  }
  const int m = std::atoi(argv[1]), n = std::atoi(argv[2]), per = std::atoi(argv[3]);
  const uint64_t seed = std::strtoull(argv[4], nullptr, 10);
  const std::string path = argv[5];
  std::mt19937_64 rng(seed);
  std::uniform_int_distribution<int> row(0, m - 1);
  std::normal_distribution<double> val(0.0, 1.0);
  std::uniform_int_distribution<int> sense(0, 2);

  // the RawLP a modeller would write
  RawLP raw;
  raw.name = "RT";
  raw.objective_name = "COST";
  for (int r = 0; r < m; ++r) {
    raw.row_names.push_back("R" + std::to_string(r));
    raw.row_sense.push_back("EGL"[sense(rng)]);
    raw.rhs.push_back(val(rng));
  }
  for (int j = 0; j < n; ++j) {
    raw.col_names.push_back("C" + std::to_string(j));
    raw.obj_coeffs.push_back(val(rng));
    const int kind = int(rng() % 5);
    raw.lower.push_back(kind == 1 ? -kInf : kind == 2 ? -1.5 : 0.0);
    raw.upper.push_back(kind == 3 ? 4.25 : kind == 4 ? 1.0 : kInf);
    raw.is_integer.push_back(false);
    std::vector<int> rows;
    while (int(rows.size()) < std::min(per, m)) {  // distinct rows per column
      const int r = row(rng);
      bool dup = false;
      for (int q : rows) dup = dup || q == r;
      if (!dup) rows.push_back(r);
    }
    for (int r : rows) raw.entries.push_back({r, j, val(rng)});
  }
  const auto t0 = std::chrono::steady_clock::now();
  ProblemData want = to_standard_form(raw);
  const auto t1 = std::chrono::steady_clock::now();
  {
    std::ofstream out(path);
    out << emit_mps(want);
  }
  const auto t2 = std::chrono::steady_clock::now();
  const RawLP back = parse_mps_file(path);
  const auto t3 = std::chrono::steady_clock::now();
  const ProblemData got = to_standard_form(back);
  const auto t4 = std::chrono::steady_clock::now();
  auto secs = [](auto a, auto b) { return std::chrono::duration<double>(b - a).count(); };

  bool same = got.n() == want.n() && got.m1() == want.m1() && got.m2() == want.m2() &&
              got.k.row_ptr == want.k.row_ptr && got.k.col_idx == want.k.col_idx &&
              got.k.vals == want.k.vals && got.c == want.c && got.q == want.q &&
              got.l == want.l && got.u == want.u && got.row_names_g == want.row_names_g &&
              got.row_names_a == want.row_names_a && got.col_names == want.col_names;
  std::ifstream f(path, std::ios::binary | std::ios::ate);
  const long long bytes = static_cast<long long>(f.tellg());
  std::printf("{\"rows\": %d, \"cols\": %d, \"nnz\": %zu, \"file_bytes\": %lld, "
              "\"standard_form_s\": %.4f, \"emit_s\": %.4f, \"parse_s\": %.4f, "
              "\"reparse_standard_form_s\": %.4f, \"parse_MB_per_s\": %.1f, \"identical\": %s}\n",
              m, n, want.k.vals.size(), bytes, secs(t0, t1), secs(t1, t2), secs(t2, t3),
              secs(t3, t4), double(bytes) / 1e6 / secs(t2, t3), same ? "true" : "false");
  return same ? 0 : 1;
}
