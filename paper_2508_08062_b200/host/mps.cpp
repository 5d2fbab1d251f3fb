// mps.cpp — the drop-in's MPS front end: free-format
// fixed-section MPS (NAME, OBJSENSE, ROWS, COLUMNS with integer MARKERs,
// RHS, BOUNDS; RANGES rejected) into RawLP, for MIPLIB-scale files.
//
// The file is memory-mapped and scanned once for line starts and section
// headers. The COLUMNS section — nearly all of a large file — is cut into
// line-aligned chunks that worker threads tokenise on their own: field
// splitting, std::from_chars numbers and row-name lookups in a read-only
// hash table. A sequential pass then assigns column indices in order of
// first appearance, applies the integer markers and appends the
// coefficients in file order, so the RawLP is exactly what a one-pass
// reader builds (same column order, same entry order, objective
// coefficients summed in file order). Errors carry the offending line
// number; the first one in file order wins.
// Accepted language and error kinds follow the reference reader
// (proj/src/lp_model.cpp:49-224, proj/tests/test_lp_model.cpp): InputError
// for malformed input, UnsupportedError for RANGES.
#include <fcntl.h>
#include <sys/mman.h>
#include <sys/stat.h>
#include <unistd.h>

#include <algorithm>
#include <cctype>
#include <charconv>
#include <cstring>
#include <istream>
#include <iterator>
#include <string>
#include <string_view>
#include <thread>
#include <unordered_map>
#include <vector>

#include "aapdhg/aapdhg.hpp"

namespace aapdhg {
namespace {

struct SvHash {
  using is_transparent = void;
  std::size_t operator()(std::string_view s) const { return std::hash<std::string_view>{}(s); }
};
using NameMap = std::unordered_map<std::string_view, int, SvHash, std::equal_to<>>;

struct Line {
  std::size_t no;        // 1-based line number
  std::string_view text; // without the line terminator
};

bool blank(char c) { return c == ' ' || c == '\t' || c == '\r' || c == '\v' || c == '\f'; }

// up to `cap` whitespace-separated fields; returns the field count (the
// count keeps growing past cap, so over-long records are detected)
int split(std::string_view s, std::string_view* f, int cap) {
  int n = 0;
  std::size_t i = 0;
  while (true) {
    while (i < s.size() && blank(s[i])) ++i;
    if (i >= s.size()) break;
    const std::size_t b = i;
    while (i < s.size() && !blank(s[i])) ++i;
    if (n < cap) f[n] = s.substr(b, i - b);
    ++n;
  }
  return n;
}

[[noreturn]] void bad(std::size_t line, const std::string& what) {
  throw InputError("MPS line " + std::to_string(line) + ": " + what);
}

double to_number(std::string_view s, std::size_t line) {
  double v = 0.0;
  const char* b = s.data();
  const char* e = s.data() + s.size();
  if (!s.empty() && *b == '+') ++b;  // from_chars takes no leading '+'
  const auto r = std::from_chars(b, e, v);
  if (r.ec != std::errc() || r.ptr != e || b == e) bad(line, "not a number: '" + std::string(s) + "'");
  return v;
}

bool is_header(std::string_view t) { return !t.empty() && !blank(t[0]); }
bool is_comment(std::string_view t) { return !t.empty() && t[0] == '*'; }

// One COLUMNS record after tokenising: the column name, up to two
// (row, value) pairs (row -1: the objective), or an integer marker.
struct ColRec {
  std::string_view col;
  int32_t row[2];
  double val[2];
  int8_t npairs;
  int8_t marker;  // 0 none, 1 INTORG, 2 INTEND
  std::size_t line;
};

struct ChunkOut {
  std::vector<ColRec> recs;
  std::size_t err_line = 0;  // first error of the chunk (0: none)
  std::string err;
};

void tokenise_columns(const std::vector<Line>& lines, std::size_t a, std::size_t b,
                      const NameMap& rows, std::string_view objective, ChunkOut& out) {
  out.recs.reserve(b - a);
  std::string_view f[6];
  for (std::size_t i = a; i < b; ++i) {
    const Line& ln = lines[i];
    if (is_comment(ln.text)) continue;
    try {
      const int nf = split(ln.text, f, 6);
      if (nf == 0) continue;
      ColRec r{};
      r.line = ln.no;
      r.col = f[0];
      if (nf >= 3 && f[1] == "'MARKER'") {
        if (f[2] == "'INTORG'") r.marker = 1;
        else if (f[2] == "'INTEND'") r.marker = 2;
        else bad(ln.no, "unknown MARKER type " + std::string(f[2]));
        out.recs.push_back(r);
        continue;
      }
      if (nf != 3 && nf != 5) bad(ln.no, "COLUMNS record needs 3 or 5 fields");
      r.npairs = int8_t((nf - 1) / 2);
      for (int q = 0; q < r.npairs; ++q) {
        const std::string_view rn = f[1 + 2 * q];
        r.val[q] = to_number(f[2 + 2 * q], ln.no);
        if (rn == objective) {
          r.row[q] = -1;
        } else {
          const auto it = rows.find(rn);
          if (it == rows.end()) bad(ln.no, "row '" + std::string(rn) + "' is not declared in ROWS");
          r.row[q] = it->second;
        }
      }
      out.recs.push_back(r);
    } catch (const InputError& e) {
      out.err_line = ln.no;
      out.err = e.what();
      return;  // later lines of the chunk cannot come first
    }
  }
}

int column_of(RawLP& lp, std::string_view name) {
  const auto it = lp.col_index.find(std::string(name));
  if (it != lp.col_index.end()) return it->second;
  const int idx = int(lp.col_names.size());
  lp.col_names.emplace_back(name);
  lp.col_index.emplace(lp.col_names.back(), idx);
  lp.obj_coeffs.push_back(0.0);
  lp.lower.push_back(0.0);
  lp.upper.push_back(kInf);
  lp.is_integer.push_back(false);
  return idx;
}

enum class Section { kNone, kRows, kColumns, kRhs, kBounds, kDone };

RawLP parse_buffer(std::string_view text) {
  // line index (terminators \n or \r\n; a last line without one counts)
  std::vector<Line> lines;
  lines.reserve(text.size() / 24 + 16);
  std::size_t pos = 0, no = 0;
  while (pos < text.size()) {
    const void* nl = std::memchr(text.data() + pos, '\n', text.size() - pos);
    const std::size_t end = nl ? std::size_t(static_cast<const char*>(nl) - text.data()) : text.size();
    std::string_view t = text.substr(pos, end - pos);
    if (!t.empty() && t.back() == '\r') t.remove_suffix(1);
    lines.push_back({++no, t});
    pos = end + 1;
  }

  RawLP lp;
  Section sec = Section::kNone;
  bool seen_rows = false, seen_columns = false, sense_pending = false;
  std::vector<std::string> row_storage;
  std::string_view f[6];
  auto set_sense = [&](std::string_view w) { lp.maximize = w == "MAX" || w == "MAXIMIZE"; };

  for (std::size_t i = 0; i < lines.size() && sec != Section::kDone; ++i) {
    const Line& ln = lines[i];
    if (is_comment(ln.text)) continue;
    const int nf = split(ln.text, f, 6);
    if (nf == 0) continue;
    if (is_header(ln.text)) {
      sense_pending = false;
      if (f[0] == "NAME") {
        if (nf > 1) lp.name = std::string(f[1]);
      } else if (f[0] == "OBJSENSE") {
        if (nf > 1) set_sense(f[1]);
        else sense_pending = true;
      } else if (f[0] == "ROWS") {
        sec = Section::kRows;
        seen_rows = true;
      } else if (f[0] == "COLUMNS") {
        if (!seen_rows) bad(ln.no, "COLUMNS section without a ROWS section before it");
        seen_columns = true;
        // the whole COLUMNS section in parallel chunks
        std::size_t e = i + 1;
        while (e < lines.size() && !(is_header(lines[e].text) && !is_comment(lines[e].text))) ++e;
        NameMap rows;
        rows.reserve(lp.row_names.size() * 2 + 1);
        for (std::size_t r = 0; r < lp.row_names.size(); ++r) rows.emplace(lp.row_names[r], int(r));
        const std::size_t nl = e - (i + 1);
        const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
        const std::size_t nt = std::min<std::size_t>(std::min<std::size_t>(hw, 32),
                                                     std::max<std::size_t>(1, nl / 65536));
        std::vector<ChunkOut> outs(nt);
        std::vector<std::thread> th;
        const std::size_t per = (nl + nt - 1) / std::max<std::size_t>(nt, 1);
        for (std::size_t t = 0; t < nt; ++t) {
          const std::size_t a = i + 1 + t * per, b = std::min(e, a + per);
          if (a >= b) continue;
          if (t + 1 == nt || nt == 1)
            tokenise_columns(lines, a, b, rows, lp.objective_name, outs[t]);
          else
            th.emplace_back(tokenise_columns, std::cref(lines), a, b, std::cref(rows),
                            std::string_view(lp.objective_name), std::ref(outs[t]));
        }
        for (auto& t : th) t.join();
        // in file order: the first error, column indices, markers, entries
        bool integer = false;
        std::string_view prev_name;
        int prev_col = -1;
        for (ChunkOut& o : outs) {
          for (const ColRec& r : o.recs) {
            if (r.marker) {
              integer = r.marker == 1;
              continue;
            }
            const int c = (prev_col >= 0 && r.col == prev_name) ? prev_col : column_of(lp, r.col);
            prev_name = r.col;
            prev_col = c;
            if (integer) lp.is_integer[std::size_t(c)] = true;  // relaxed: kept as a flag
            for (int q = 0; q < r.npairs; ++q) {
              if (r.row[q] < 0) lp.obj_coeffs[std::size_t(c)] += r.val[q];
              else lp.entries.push_back({r.row[q], c, r.val[q]});
            }
          }
          if (o.err_line) throw InputError(o.err);
        }
        sec = Section::kColumns;
        i = e - 1;
      } else if (f[0] == "RHS") {
        if (!seen_columns) bad(ln.no, "RHS section before COLUMNS");
        sec = Section::kRhs;
      } else if (f[0] == "RANGES") {
        throw UnsupportedError("MPS line " + std::to_string(ln.no) +
                               ": RANGES sections are not supported");
      } else if (f[0] == "BOUNDS") {
        if (!seen_columns) bad(ln.no, "BOUNDS section before COLUMNS");
        sec = Section::kBounds;
      } else if (f[0] == "ENDATA") {
        sec = Section::kDone;
      } else {
        bad(ln.no, "unknown section '" + std::string(f[0]) + "'");
      }
      continue;
    }
    if (sense_pending) {  // OBJSENSE value on its own line
      set_sense(f[0]);
      sense_pending = false;
      continue;
    }
    switch (sec) {
      case Section::kNone:
        bad(ln.no, "record outside any section");
      case Section::kRows: {
        if (nf != 2) bad(ln.no, "ROWS record needs 2 fields");
        const char kind = char(std::toupper(static_cast<unsigned char>(f[0][0])));
        if (f[0].size() != 1 || (kind != 'N' && kind != 'E' && kind != 'G' && kind != 'L'))
          bad(ln.no, "row type must be N, E, G or L");
        if (kind == 'N') {
          if (lp.objective_name.empty()) lp.objective_name = std::string(f[1]);
          break;  // further N rows are free rows: ignored
        }
        const std::string name(f[1]);
        if (lp.row_index.count(name)) bad(ln.no, "row '" + name + "' declared twice");
        lp.row_index.emplace(name, int(lp.row_names.size()));
        lp.row_names.push_back(name);
        lp.row_sense.push_back(kind);
        lp.rhs.push_back(0.0);
        break;
      }
      case Section::kRhs: {
        if (nf != 3 && nf != 5) bad(ln.no, "RHS record needs 3 or 5 fields");
        for (int q = 0; 2 + 2 * q < nf; ++q) {
          const std::string_view rn = f[1 + 2 * q];
          const double v = to_number(f[2 + 2 * q], ln.no);
          if (rn == lp.objective_name) continue;  // objective constant: not modelled
          const auto it = lp.row_index.find(std::string(rn));
          if (it == lp.row_index.end()) bad(ln.no, "RHS for undeclared row '" + std::string(rn) + "'");
          lp.rhs[std::size_t(it->second)] = v;
        }
        break;
      }
      case Section::kBounds: {
        if (nf != 3 && nf != 4) bad(ln.no, "BOUNDS record needs 3 or 4 fields");
        const auto it = lp.col_index.find(std::string(f[2]));
        if (it == lp.col_index.end()) bad(ln.no, "BOUNDS for unknown column '" + std::string(f[2]) + "'");
        const std::size_t c = std::size_t(it->second);
        const std::string_view k = f[0];
        const bool takes_value = k == "UP" || k == "LO" || k == "FX" || k == "UI" || k == "LI";
        if (takes_value && nf != 4) bad(ln.no, "bound type " + std::string(k) + " needs a value");
        const double v = takes_value ? to_number(f[3], ln.no) : 0.0;
        if (k == "UP" || k == "UI") {
          lp.upper[c] = v;
        } else if (k == "LO" || k == "LI") {
          lp.lower[c] = v;
        } else if (k == "FX") {
          lp.lower[c] = v;
          lp.upper[c] = v;
        } else if (k == "FR") {
          lp.lower[c] = -kInf;
          lp.upper[c] = kInf;
        } else if (k == "MI") {
          lp.lower[c] = -kInf;
        } else if (k == "PL") {
          lp.upper[c] = kInf;
        } else if (k == "BV") {
          lp.lower[c] = 0.0;
          lp.upper[c] = 1.0;
        } else {
          bad(ln.no, "unknown bound type '" + std::string(k) + "'");
        }
        break;
      }
      default:
        break;
    }
  }
  if (!seen_rows || !seen_columns) throw InputError("MPS input lacks a ROWS or COLUMNS section");
  if (lp.objective_name.empty()) throw InputError("MPS input declares no objective (N) row");
  return lp;
}

}  // namespace

RawLP parse_mps(std::istream& in) {
  const std::string text{std::istreambuf_iterator<char>(in), std::istreambuf_iterator<char>()};
  return parse_buffer(text);
}

RawLP parse_mps_file(const std::string& path) {
  const int fd = ::open(path.c_str(), O_RDONLY);
  if (fd < 0) throw InputError("cannot open MPS file " + path);
  struct stat st {};
  if (::fstat(fd, &st) != 0) {
    ::close(fd);
    throw InputError("cannot stat MPS file " + path);
  }
  const std::size_t len = std::size_t(st.st_size);
  if (len == 0) {
    ::close(fd);
    return parse_buffer(std::string_view());
  }
  void* map = ::mmap(nullptr, len, PROT_READ, MAP_PRIVATE, fd, 0);
  ::close(fd);
  if (map == MAP_FAILED) throw InputError("cannot map MPS file " + path);
  ::madvise(map, len, MADV_SEQUENTIAL);
  try {
    RawLP lp = parse_buffer(std::string_view(static_cast<const char*>(map), len));
    ::munmap(map, len);
    return lp;
  } catch (...) {
    ::munmap(map, len);
    throw;
  }
}

}  // namespace aapdhg
