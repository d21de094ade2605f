// batchlp/mps.hpp — free-format MPS ingest and export of the B200 drop-in
// (SURVEY §8(f) item 4), so the paper's instances reach the device solver.
//
// Same surface and semantics as the reference's reader/writer (reference
// proj/include/batchlp/mps.hpp:45-434): MpsParseError carries the 1-based
// line, MpsModel holds the LpProblem plus names, the integrality set and the
// warnings. Sections NAME, ROWS, COLUMNS, RHS, RANGES, BOUNDS, ENDATA; the
// first N row is the objective, later N rows stay as free rows; RANGES on
// L: [b - |r|, b], G: [b, b + |r|], E: [b, b + r] (r >= 0) or [b + r, b];
// bound keys LO UP FX FR MI PL BV (BV: [0, 1] and integral; UP keeps the
// default lower bound 0); INTORG / INTEND markers collect integer columns.
// The writer emits two-sided rows as L rows plus a range and round-trips
// every value with %.17g.
//
// Host-side I/O only: the parsed problem is uploaded to the GPU by the
// solve that uses it (include/batchlp/device.hpp).
#ifndef BATCHLP_B200_MPS_HPP
#define BATCHLP_B200_MPS_HPP

#include <cctype>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <fstream>
#include <istream>
#include <map>
#include <optional>
#include <ostream>
#include <sstream>
#include <stdexcept>
#include <string>
#include <vector>

#include "batchlp/problem.hpp"

namespace batchlp {

class MpsParseError : public std::runtime_error {
 public:
  MpsParseError(int line, const std::string& what)
      : std::runtime_error("mps:" + std::to_string(line) + ": " + what), line_(line) {}
  int line() const { return line_; }

 private:
  int line_;
};

struct MpsModel {
  std::string name;
  LpProblem problem;
  std::vector<int> integer_columns;
  std::vector<std::string> row_names;  // constraint rows; the objective is not listed
  std::vector<std::string> column_names;
  std::string objective_name;
  std::vector<std::string> warnings;
};

namespace mps_detail {

inline std::vector<std::string> split_fields(const std::string& text) {
  std::vector<std::string> out;
  std::istringstream words(text);
  for (std::string w; words >> w;) out.push_back(std::move(w));
  return out;
}

inline double number(const std::string& field, int line) {
  const char* s = field.c_str();
  char* stop = nullptr;
  const double v = std::strtod(s, &stop);
  if (stop == s || *stop != '\0') throw MpsParseError(line, "cannot parse number '" + field + "'");
  return v;
}

inline std::string exact(double v) {
  char text[40];
  std::snprintf(text, sizeof text, "%.17g", v);
  return text;
}

// One pass over the file; each section's data lines go to their handler.
class Reader {
 public:
  MpsModel read(std::istream& in) {
    std::string raw;
    while (std::getline(in, raw)) {
      ++line_;
      if (!raw.empty() && raw.back() == '\r') raw.pop_back();
      if (raw.empty() || raw.front() == '*') continue;  // blank / comment
      const std::vector<std::string> f = split_fields(raw);
      if (f.empty()) continue;
      if (!std::isspace(static_cast<unsigned char>(raw.front()))) {
        if (!header(f)) break;  // ENDATA
        continue;
      }
      data(f);
    }
    if (!have_objective_) throw MpsParseError(line_, "no objective (N) row declared");
    return finish();
  }

 private:
  enum class Part { kNone, kRows, kColumns, kRhs, kRanges, kBounds };
  struct Row {
    char sense = 'N';
    double rhs = 0.0;
    std::optional<double> range;
  };

  bool header(const std::vector<std::string>& f) {
    const std::string& k = f[0];
    if (k == "NAME") model_.name = f.size() > 1 ? f[1] : std::string();
    else if (k == "ROWS") part_ = Part::kRows;
    else if (k == "COLUMNS") part_ = Part::kColumns;
    else if (k == "RHS") part_ = Part::kRhs;
    else if (k == "RANGES") part_ = Part::kRanges;
    else if (k == "BOUNDS") part_ = Part::kBounds;
    else if (k == "ENDATA") return false;
    else throw MpsParseError(line_, "unknown section '" + k + "'");
    return true;
  }

  void data(const std::vector<std::string>& f) {
    switch (part_) {
      case Part::kRows: return row_entry(f);
      case Part::kColumns: return column_entry(f);
      case Part::kRhs: return pair_entries(f, "RHS", "rhs", [&](Row& r, double v) { r.rhs = v; });
      case Part::kRanges:
        return pair_entries(f, "RANGES", "range", [&](Row& r, double v) { r.range = v; });
      case Part::kBounds: return bound_entry(f);
      case Part::kNone: throw MpsParseError(line_, "data before any section header");
    }
  }

  void row_entry(const std::vector<std::string>& f) {
    if (f.size() != 2) throw MpsParseError(line_, "malformed ROWS entry");
    const char sense = static_cast<char>(std::toupper(static_cast<unsigned char>(f[0][0])));
    if (f[0].size() != 1 || std::string("NLGE").find(sense) == std::string::npos)
      throw MpsParseError(line_, "unknown row type '" + f[0] + "'");
    if (rows_by_name_.count(f[1])) throw MpsParseError(line_, "duplicate row name '" + f[1] + "'");
    if (sense == 'N' && !have_objective_) {
      have_objective_ = true;
      model_.objective_name = f[1];
      rows_by_name_[f[1]] = kObjective;
      return;
    }
    rows_by_name_[f[1]] = static_cast<int>(rows_.size());
    rows_.push_back(Row{sense, 0.0, std::nullopt});
    model_.row_names.push_back(f[1]);
  }

  int column(const std::string& name, bool declared_only) {
    const auto hit = cols_by_name_.find(name);
    if (hit != cols_by_name_.end()) return hit->second;
    if (declared_only) throw MpsParseError(line_, "bound on undeclared column '" + name + "'");
    const int id = static_cast<int>(model_.column_names.size());
    cols_by_name_.emplace(name, id);
    model_.column_names.push_back(name);
    cost_.push_back(0.0);
    lower_.push_back(0.0);
    upper_.push_back(kInf);
    integral_.push_back(in_int_block_);
    return id;
  }

  int row_of(const std::string& name) const {
    const auto hit = rows_by_name_.find(name);
    if (hit == rows_by_name_.end()) throw MpsParseError(line_, "unknown row '" + name + "'");
    return hit->second;
  }

  void column_entry(const std::vector<std::string>& f) {
    const bool marker = f.size() >= 3 && (f[1] == "'MARKER'" || f[2] == "'MARKER'");
    if (marker) {
      bool start = false, stop = false;
      for (const std::string& w : f) {
        start = start || w == "'INTORG'";
        stop = stop || w == "'INTEND'";
      }
      if (!start && !stop) throw MpsParseError(line_, "unrecognized marker line");
      in_int_block_ = start;
      return;
    }
    if (f.size() != 3 && f.size() != 5) throw MpsParseError(line_, "malformed COLUMNS entry");
    const int c = column(f[0], false);
    for (std::size_t k = 1; k + 1 < f.size(); k += 2) {
      const int r = row_of(f[k]);
      const double v = number(f[k + 1], line_);
      if (r == kObjective) cost_[c] += v;
      else entries_.push_back(Triplet{r, c, v});
    }
  }

  template <class Set>
  void pair_entries(const std::vector<std::string>& f, const char* section, const char* what,
                    Set set) {
    if (f.size() != 3 && f.size() != 5)
      throw MpsParseError(line_, std::string("malformed ") + section + " entry");
    for (std::size_t k = 1; k + 1 < f.size(); k += 2) {
      const int r = row_of(f[k]);
      const double v = number(f[k + 1], line_);
      if (r == kObjective)
        model_.warnings.push_back("line " + std::to_string(line_) + ": " + what +
                                  " on the objective row ignored");
      else set(rows_[r], v);
    }
  }

  void bound_entry(const std::vector<std::string>& f) {
    if (f.size() != 3 && f.size() != 4) throw MpsParseError(line_, "malformed BOUNDS entry");
    const std::string& key = f[0];
    const int c = column(f[2], true);
    const bool valued = key == "LO" || key == "UP" || key == "FX";
    if (valued && f.size() != 4) throw MpsParseError(line_, key + " bound requires a value");
    const double v = valued ? number(f[3], line_) : 0.0;
    if (key == "LO") lower_[c] = v;
    else if (key == "UP") upper_[c] = v;
    else if (key == "FX") lower_[c] = upper_[c] = v;
    else if (key == "FR") lower_[c] = -kInf, upper_[c] = kInf;
    else if (key == "MI") lower_[c] = -kInf;
    else if (key == "PL") upper_[c] = kInf;
    else if (key == "BV") lower_[c] = 0.0, upper_[c] = 1.0, integral_[c] = true;
    else throw MpsParseError(line_, "unknown bound key '" + key + "'");
  }

  // the row box of one constraint from its sense, rhs and optional range
  static Interval box(const Row& r) {
    double lo = -kInf, hi = kInf;
    if (r.sense == 'L') hi = r.rhs;
    if (r.sense == 'G') lo = r.rhs;
    if (r.sense == 'E') lo = hi = r.rhs;
    if (r.range && r.sense != 'N') {
      const double w = *r.range;
      if (r.sense == 'L') lo = hi - std::abs(w);
      else if (r.sense == 'G') hi = lo + std::abs(w);
      else if (w >= 0.0) hi = lo + w;
      else lo = hi + w;
    }
    return Interval{lo, hi};
  }

  MpsModel finish() {
    const int m = static_cast<int>(rows_.size());
    const int n = static_cast<int>(model_.column_names.size());
    Bounds rb(m);
    for (int r = 0; r < m; ++r) rb.set(r, box(rows_[r]));
    model_.problem.A = SparseMatrix::from_triplets(std::move(entries_), m, n);
    model_.problem.objective = std::move(cost_);
    model_.problem.row_bounds = std::move(rb);
    model_.problem.var_bounds.lower = std::move(lower_);
    model_.problem.var_bounds.upper = std::move(upper_);
    for (int c = 0; c < n; ++c)
      if (integral_[c]) model_.integer_columns.push_back(c);
    return std::move(model_);
  }

  static constexpr int kObjective = -1;
  MpsModel model_;
  Part part_ = Part::kNone;
  int line_ = 0;
  bool have_objective_ = false, in_int_block_ = false;
  std::vector<Row> rows_;
  std::map<std::string, int> rows_by_name_, cols_by_name_;
  std::vector<Triplet> entries_;
  std::vector<double> cost_, lower_, upper_;
  std::vector<bool> integral_;
};

}  // namespace mps_detail

inline MpsModel parse_mps(std::istream& in) { return mps_detail::Reader().read(in); }

inline MpsModel parse_mps_string(const std::string& text) {
  std::istringstream in(text);
  return parse_mps(in);
}

inline MpsModel read_mps_file(const std::string& path) {
  std::ifstream in(path);
  if (!in) throw std::runtime_error("cannot open '" + path + "'");
  return parse_mps(in);
}

// Rows R<i>, columns C<j>, objective OBJ; integer columns inside
// INTORG / INTEND markers.
inline void write_mps(std::ostream& os, const LpProblem& p,
                      const std::vector<int>& integer_columns = {},
                      const std::string& name = "BATCHLP") {
  using mps_detail::exact;
  const int m = p.num_rows(), n = p.num_cols();
  std::vector<bool> is_int(static_cast<std::size_t>(n), false);
  for (const int c : integer_columns)
    if (c >= 0 && c < n) is_int[c] = true;
  // N free, E fixed, R two-sided (written as L + range), L, G
  std::vector<char> kind(static_cast<std::size_t>(m));
  for (int r = 0; r < m; ++r) {
    const Interval b = p.row_bounds.at(r);
    kind[r] = b.is_free() ? 'N'
              : b.is_fixed() ? 'E'
              : (b.lower != -kInf && b.upper != kInf) ? 'R'
              : b.upper != kInf ? 'L'
                                : 'G';
  }
  os << "NAME          " << name << "\nROWS\n N  OBJ\n";
  for (int r = 0; r < m; ++r) os << ' ' << (kind[r] == 'R' ? 'L' : kind[r]) << "  R" << r << "\n";

  os << "COLUMNS\n";
  const CsrView byc = p.A.transpose_view();
  bool open = false;
  int markers = 0;
  for (int c = 0; c < n; ++c) {
    if (is_int[c] != open) {
      open = is_int[c];
      os << "    MARKER" << markers++ << "  'MARKER'  " << (open ? "'INTORG'" : "'INTEND'")
         << "\n";
    }
    const bool has_cost = p.objective[c] != 0.0;
    if (has_cost) os << "    C" << c << "  OBJ  " << exact(p.objective[c]) << "\n";
    for (int q = byc.offsets[c]; q < byc.offsets[c + 1]; ++q)
      os << "    C" << c << "  R" << byc.cols[q] << "  " << exact(byc.values[q]) << "\n";
    if (!has_cost && byc.offsets[c] == byc.offsets[c + 1]) os << "    C" << c << "  OBJ  0\n";
  }
  if (open) os << "    MARKER" << markers++ << "  'MARKER'  'INTEND'\n";

  os << "RHS\n";
  for (int r = 0; r < m; ++r) {
    if (kind[r] == 'N') continue;
    const Interval b = p.row_bounds.at(r);
    const double rhs = (kind[r] == 'L' || kind[r] == 'R') ? b.upper : b.lower;
    if (rhs != 0.0) os << "    RHS  R" << r << "  " << exact(rhs) << "\n";
  }
  bool ranged = false;
  for (int r = 0; r < m && !ranged; ++r) ranged = kind[r] == 'R';
  if (ranged) {
    os << "RANGES\n";
    for (int r = 0; r < m; ++r)
      if (kind[r] == 'R') {
        const Interval b = p.row_bounds.at(r);
        os << "    RNG  R" << r << "  " << exact(b.upper - b.lower) << "\n";
      }
  }

  os << "BOUNDS\n";
  for (int c = 0; c < n; ++c) {
    const Interval b = p.var_bounds.at(c);
    if (b.is_free()) {
      os << " FR BND  C" << c << "\n";
      continue;
    }
    if (b.is_fixed()) {
      os << " FX BND  C" << c << "  " << exact(b.lower) << "\n";
      continue;
    }
    if (b.lower == -kInf) os << " MI BND  C" << c << "\n";
    else if (b.lower != 0.0) os << " LO BND  C" << c << "  " << exact(b.lower) << "\n";
    if (b.upper != kInf) os << " UP BND  C" << c << "  " << exact(b.upper) << "\n";
  }
  os << "ENDATA\n";
}

}  // namespace batchlp

#endif  // BATCHLP_B200_MPS_HPP
