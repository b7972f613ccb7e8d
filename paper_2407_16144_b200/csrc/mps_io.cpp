// MPS ingestion and solution / trace reports -- the reference's declared but
// unimplemented inc/hplp/mps_io.hpp:29-94 (SPEC.md "[MODULE] mps_io"),
// implemented on the host for the B200 solver.
//
//  * parse_mps: fixed- and free-format MPS, sections NAME / OBJSENSE / ROWS /
//    COLUMNS / RHS / RANGES / BOUNDS / ENDATA, row types N/L/G/E, bound types
//    UP/LO/FX/FR/MI/PL/BV/LI/UI (integrality -- BV, LI/UI, MARKER INTORG --
//    relaxed to continuous, with a warning).  The first N row is the
//    objective, later N rows are dropped with a warning.  Default bounds
//    [0, inf); "UP < 0" on a column whose lower bound was never set makes the
//    lower bound -inf (common convention, warned).  RHS on the objective row
//    sets objective_constant = -value.  Errors throw MpsParseError(line).
//  * write_mps: normalized free MPS with 17-significant-digit numbers;
//    parse(write(parse(x))) == parse(x) exactly.
//  * write_solution_json / parse_solution_json: deterministic key order,
//    17-significant-digit numbers (bit-exact round trip), NaN as null and
//    infinities as "inf" / "-inf", vectors above a threshold elided with an
//    explicit flag, wall time segregated under "timing".
//  * write_trace_csv: fixed header, one row per TraceRecord.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <map>
#include <memory>
#include <sstream>
#include <stdexcept>
#include <string>
#include <unordered_map>
#include <vector>

#include "hplp_gpu.hpp"

namespace hplp_gpu {

namespace {

constexpr double kInf = std::numeric_limits<double>::infinity();

std::string num17(double v) {
  char buf[40];
  std::snprintf(buf, sizeof buf, "%.17g", v);
  return buf;
}

std::vector<std::string> split_ws(const std::string& s) {
  std::vector<std::string> out;
  std::istringstream is(s);
  std::string t;
  while (is >> t) out.push_back(t);
  return out;
}

std::string trim(const std::string& s) {
  const auto b = s.find_first_not_of(" \t\r");
  if (b == std::string::npos) return "";
  const auto e = s.find_last_not_of(" \t\r");
  return s.substr(b, e - b + 1);
}

// Fixed-format MPS fields (1-based columns 2-3, 5-12, 15-22, 25-36, 40-47,
// 50-61); used when a line does not tokenize as free format.  Name fields are
// positional (they may hold blanks); a numeric field is the token starting in
// its columns, so a 17-significant-digit number may run past column 36 (the
// writer then puts one pair per line).
std::vector<std::string> fixed_fields(const std::string& line) {
  static const int kStart[] = {1, 4, 14, 24, 39, 49};
  static const int kLen[] = {2, 8, 8, 12, 8, 12};
  std::vector<std::string> f;
  int consumed = 0;  // end of the last numeric token
  for (int k = 0; k < 6; ++k) {
    const int start = std::max(kStart[k], consumed);
    if (static_cast<int>(line.size()) <= start) break;
    if (k == 3 || k == 5) {  // numeric: the token from here to the next blank
      int b = start;
      while (b < static_cast<int>(line.size()) && line[b] == ' ') ++b;
      int e = b;
      while (e < static_cast<int>(line.size()) && line[e] != ' ') ++e;
      f.push_back(line.substr(b, e - b));
      consumed = e;
    } else {
      f.push_back(trim(line.substr(start, kLen[k] - (start - kStart[k]) > 0 ? kLen[k] - (start - kStart[k]) : 0)));
    }
  }
  while (!f.empty() && f.back().empty()) f.pop_back();
  return f;
}

struct Parser {
  MpsDocument* doc = nullptr;
  long line_no = 0;
  GeneralFormLP g;
  std::unordered_map<std::string, long> row_of;   // constraint rows; the objective maps to -1
  std::unordered_map<std::string, long> col_of;
  std::vector<std::string> dropped_n;             // later N rows
  std::vector<bool> lower_set;
  std::map<std::pair<long, long>, bool> seen;     // (row, col) of matrix entries
  bool integer_section = false, warned_int = false;
  // Switched on when a ROWS / COLUMNS line only parses with the fixed
  // columns (a name with a blank): from then on every data line is read by
  // column position.
  bool fixed_mode = false;

  [[noreturn]] void fail(const std::string& msg) const { throw MpsParseError(line_no, msg); }

  void warn(const std::string& w) {
    if (doc) doc->warnings.push_back("line " + std::to_string(line_no) + ": " + w);
  }

  double number(const std::string& s) const {
    if (s.empty()) fail("missing numeric value");
    char* end = nullptr;
    const double v = std::strtod(s.c_str(), &end);
    if (end == s.c_str() || *end != '\0') fail("malformed number '" + s + "'");
    return v;
  }

  long row(const std::string& name) const {
    auto it = row_of.find(name);
    if (it == row_of.end()) fail("undeclared row '" + name + "'");
    return it->second;
  }

  long col(const std::string& name) const {
    auto it = col_of.find(name);
    if (it == col_of.end()) fail("undeclared column '" + name + "'");
    return it->second;
  }

  bool is_dropped(const std::string& r) const {
    for (const auto& d : dropped_n)
      if (d == r) return true;
    return false;
  }

  void relax_warning() {
    if (!warned_int) warn("integrality relaxed to continuous bounds (LP relaxation)");
    warned_int = true;
  }

  // (row, value) pairs of a COLUMNS / RHS / RANGES line after `skip` leading
  // fields; free format first, fixed columns as the fallback.
  std::vector<std::pair<std::string, std::string>> pairs(const std::vector<std::string>& f, size_t skip) const {
    std::vector<std::pair<std::string, std::string>> out;
    for (size_t k = skip; k + 1 < f.size(); k += 2) out.push_back({f[k], f[k + 1]});
    return out;
  }

  void rows_line(const std::vector<std::string>& f) {
    if (f.size() != 2) fail("ROWS entry needs a type and a name");
    const std::string& type = f[0];
    const std::string& name = f[1];
    if (row_of.count(name) || is_dropped(name)) fail("duplicate row '" + name + "'");
    if (type == "N" || type == "n") {
      if (g.objective_name.empty()) {
        g.objective_name = name;
        row_of[name] = -1;
      } else {
        dropped_n.push_back(name);
        warn("extra objective row '" + name + "' dropped");
      }
      return;
    }
    GeneralFormRow r;
    r.name = name;
    if (type == "L" || type == "l") r.relation = RowRelation::kLessEqual;
    else if (type == "G" || type == "g") r.relation = RowRelation::kGreaterEqual;
    else if (type == "E" || type == "e") r.relation = RowRelation::kEqual;
    else fail("unknown row type '" + type + "'");
    row_of[name] = static_cast<long>(g.rows.size());
    g.rows.push_back(r);
  }

  void columns_line(std::vector<std::string> f, const std::string& raw) {
    if (f.size() >= 3 && (f[1] == "'MARKER'" || f[1] == "MARKER")) {
      const std::string& m = f.size() >= 3 ? f[2] : "";
      if (m == "'INTORG'" || m == "INTORG") integer_section = true, relax_warning();
      else if (m == "'INTEND'" || m == "INTEND") integer_section = false;
      else fail("unknown MARKER '" + m + "'");
      return;
    }
    if (fixed_mode || (f.size() != 3 && f.size() != 5)) {
      f = fixed_fields(raw);
      if (!f.empty() && f[0].empty()) f.erase(f.begin());
      if (f.size() != 3 && f.size() != 5) fail("COLUMNS entry needs a column and one or two (row, value) pairs");
      fixed_mode = true;
    }
    const std::string& cname = f[0];
    long j;
    auto it = col_of.find(cname);
    if (it == col_of.end()) {
      j = static_cast<long>(g.columns.size());
      col_of[cname] = j;
      GeneralFormColumn c;
      c.name = cname;
      g.columns.push_back(c);
      g.objective.push_back(0.0);
      lower_set.push_back(false);
    } else {
      j = it->second;
      if (j != static_cast<long>(g.columns.size()) - 1) fail("column '" + cname + "' is not contiguous in COLUMNS");
    }
    for (const auto& [rname, sval] : pairs(f, 1)) {
      const double v = number(sval);
      if (is_dropped(rname)) continue;
      const long i = row(rname);
      if (seen.count({i, j})) fail("duplicate entry (" + rname + ", " + cname + ")");
      seen[{i, j}] = true;
      if (i < 0) g.objective[j] = v;
      else g.entries.push_back(Triplet{i, j, v});
    }
  }

  void rhs_line(const std::vector<std::string>& f) {
    const size_t skip = f.size() % 2;  // optional set name
    if (f.size() < 2 || f.size() > 5) fail("RHS entry needs one or two (row, value) pairs");
    for (const auto& [rname, sval] : pairs(f, skip)) {
      const double v = number(sval);
      if (is_dropped(rname)) continue;
      const long i = row(rname);
      if (i < 0) g.objective_constant = -v;
      else g.rows[i].rhs = v;
    }
  }

  void ranges_line(const std::vector<std::string>& f) {
    const size_t skip = f.size() % 2;
    if (f.size() < 2 || f.size() > 5) fail("RANGES entry needs one or two (row, value) pairs");
    for (const auto& [rname, sval] : pairs(f, skip)) {
      const double v = number(sval);
      const long i = row(rname);
      if (i < 0) fail("RANGES on the objective row");
      g.rows[i].range = v;
    }
  }

  void bounds_line(const std::vector<std::string>& f) {
    if (f.size() < 2 || f.size() > 4) fail("BOUNDS entry needs a type, an optional set name, a column and a value");
    const std::string type = f[0];
    const bool needs_value = !(type == "FR" || type == "MI" || type == "PL" || type == "BV");
    // type [set] column [value]
    std::string cname, sval;
    if (needs_value) {
      if (f.size() == 4) cname = f[2], sval = f[3];
      else if (f.size() == 3) cname = f[1], sval = f[2];
      else fail("bound '" + type + "' needs a value");
    } else {
      if (f.size() == 4) cname = f[2], sval = f[3];  // BV with a stray value
      else if (f.size() == 3) {
        // "BV set col" or "FR col value"? a known column in the middle means no set name
        if (col_of.count(f[1]) && !col_of.count(f[2])) cname = f[1], sval = f[2];
        else cname = f[2];
      } else cname = f[1];
    }
    const long j = col(cname);
    GeneralFormColumn& c = g.columns[j];
    const double v = needs_value ? number(sval) : 0.0;
    if (type == "UP" || type == "UI") {
      if (type == "UI") relax_warning();
      c.upper = v;
      if (v < 0 && !lower_set[j] && c.lower == 0.0) {
        c.lower = -kInf;
        warn("UP bound < 0 on '" + cname + "' with no lower bound: lower set to -inf");
      }
    } else if (type == "LO" || type == "LI") {
      if (type == "LI") relax_warning();
      c.lower = v;
      lower_set[j] = true;
    } else if (type == "FX") {
      c.lower = c.upper = v;
      lower_set[j] = true;
    } else if (type == "FR") {
      c.lower = -kInf, c.upper = kInf;
      lower_set[j] = true;
    } else if (type == "MI") {
      c.lower = -kInf;
      lower_set[j] = true;
    } else if (type == "PL") {
      c.upper = kInf;
    } else if (type == "BV") {
      relax_warning();
      c.lower = 0.0, c.upper = 1.0;
      lower_set[j] = true;
    } else {
      fail("unknown bound type '" + type + "'");
    }
  }

  GeneralFormLP run(std::istream& in) {
    enum Sec { kNone, kName, kObjSense, kRows, kCols, kRhs, kRanges, kBounds, kEnd } sec = kNone;
    std::string raw;
    bool seen_rows = false;
    while (std::getline(in, raw)) {
      ++line_no;
      if (!raw.empty() && raw.back() == '\r') raw.pop_back();
      if (raw.empty() || raw[0] == '*' || trim(raw).empty()) continue;
      std::vector<std::string> f = split_ws(raw);
      if (raw[0] != ' ' && raw[0] != '\t') {  // section header
        const std::string& h = f[0];
        if (h == "NAME") {
          sec = kName;
          g.name = f.size() > 1 ? trim(raw.substr(raw.find("NAME") + 4)) : "";
          if (doc) doc->problem_name = g.name;
        } else if (h == "OBJSENSE" || h == "OBJSENCE") {
          sec = kObjSense;
          if (f.size() > 1) {
            if (f[1] == "MAX" || f[1] == "MAXIMIZE") g.maximize = true;
            else if (f[1] == "MIN" || f[1] == "MINIMIZE") g.maximize = false;
            else fail("unknown OBJSENSE '" + f[1] + "'");
          }
        } else if (h == "ROWS") {
          sec = kRows, seen_rows = true;
        } else if (h == "COLUMNS") {
          sec = kCols;
        } else if (h == "RHS") {
          sec = kRhs;
        } else if (h == "RANGES") {
          sec = kRanges;
        } else if (h == "BOUNDS") {
          sec = kBounds;
        } else if (h == "ENDATA") {
          sec = kEnd;
          break;
        } else {
          fail("unknown section '" + h + "'");
        }
        continue;
      }
      switch (sec) {
        case kObjSense:
          if (f[0] == "MAX" || f[0] == "MAXIMIZE") g.maximize = true;
          else if (f[0] == "MIN" || f[0] == "MINIMIZE") g.maximize = false;
          else fail("unknown OBJSENSE '" + f[0] + "'");
          break;
        case kRows:
          if (fixed_mode || f.size() != 2) {
            f = fixed_fields(raw);
            if (f.size() != 2) fail("ROWS entry needs a type and a name");
            fixed_mode = true;
          }
          rows_line(f);
          break;
        case kCols:
          columns_line(f, raw);
          break;
        case kRhs:
        case kRanges:
          if (fixed_mode) {  // fields 2..6: set, row, value, row, value
            f = fixed_fields(raw);
            if (!f.empty()) f.erase(f.begin());
            if (f.size() % 2 == 0) f.insert(f.begin(), "");  // keep the set-name slot
          }
          if (sec == kRhs) rhs_line(f);
          else ranges_line(f);
          break;
        case kBounds:
          if (fixed_mode) f = fixed_fields(raw);  // type, set, column, value
          bounds_line(f);
          break;
        default:
          fail("data line outside a section");
      }
    }
    if (sec != kEnd) {
      ++line_no;
      fail("missing ENDATA");
    }
    if (!seen_rows) fail("missing ROWS section");
    if (g.objective_name.empty()) fail("no objective (N) row");
    if (doc) doc->objective_row_name = g.objective_name;
    return std::move(g);
  }
};

// ---- minimal JSON value (writer schema only) --------------------------------
struct JVal {
  enum Kind { kNull, kBool, kNum, kStr, kArr, kObj } kind = kNull;
  bool b = false;
  double num = 0.0;
  std::string str;
  std::vector<JVal> arr;
  std::vector<std::pair<std::string, JVal>> obj;
  const JVal* get(const std::string& k) const {
    for (const auto& [key, v] : obj)
      if (key == k) return &v;
    return nullptr;
  }
};

struct JParser {
  const std::string& s;
  size_t p = 0;
  [[noreturn]] void fail(const std::string& m) const {
    throw std::invalid_argument("parse_solution_json: " + m + " at offset " + std::to_string(p));
  }
  void ws() {
    while (p < s.size() && (s[p] == ' ' || s[p] == '\n' || s[p] == '\t' || s[p] == '\r')) ++p;
  }
  JVal value() {
    ws();
    if (p >= s.size()) fail("unexpected end");
    const char c = s[p];
    JVal v;
    if (c == '{') {
      v.kind = JVal::kObj;
      ++p;
      ws();
      if (s[p] == '}') return ++p, v;
      while (true) {
        ws();
        JVal k = value();
        if (k.kind != JVal::kStr) fail("object key must be a string");
        ws();
        if (s[p] != ':') fail("expected ':'");
        ++p;
        v.obj.push_back({k.str, value()});
        ws();
        if (s[p] == ',') {
          ++p;
          continue;
        }
        if (s[p] == '}') return ++p, v;
        fail("expected ',' or '}'");
      }
    }
    if (c == '[') {
      v.kind = JVal::kArr;
      ++p;
      ws();
      if (s[p] == ']') return ++p, v;
      while (true) {
        v.arr.push_back(value());
        ws();
        if (s[p] == ',') {
          ++p;
          continue;
        }
        if (s[p] == ']') return ++p, v;
        fail("expected ',' or ']'");
      }
    }
    if (c == '"') {
      v.kind = JVal::kStr;
      ++p;
      while (p < s.size() && s[p] != '"') {
        if (s[p] == '\\') {
          ++p;
          const char e = s[p];
          v.str += e == 'n' ? '\n' : e == 't' ? '\t' : e;
        } else {
          v.str += s[p];
        }
        ++p;
      }
      if (p >= s.size()) fail("unterminated string");
      ++p;
      return v;
    }
    if (s.compare(p, 4, "null") == 0) return p += 4, v;
    if (s.compare(p, 4, "true") == 0) return p += 4, v.kind = JVal::kBool, v.b = true, v;
    if (s.compare(p, 5, "false") == 0) return p += 5, v.kind = JVal::kBool, v;
    char* end = nullptr;
    v.num = std::strtod(s.c_str() + p, &end);
    if (end == s.c_str() + p) fail("bad token");
    v.kind = JVal::kNum;
    p = static_cast<size_t>(end - s.c_str());
    return v;
  }
};

std::string jnum(double v) {
  if (std::isnan(v)) return "null";
  if (std::isinf(v)) return v > 0 ? "\"inf\"" : "\"-inf\"";
  return num17(v);
}

double jget_num(const JVal* v) {
  if (!v || v->kind == JVal::kNull) return std::numeric_limits<double>::quiet_NaN();
  if (v->kind == JVal::kStr) {
    if (v->str == "inf") return kInf;
    if (v->str == "-inf") return -kInf;
    throw std::invalid_argument("parse_solution_json: bad number string '" + v->str + "'");
  }
  return v->num;
}

std::string jstr(const std::string& s) {
  std::string o = "\"";
  for (char c : s) {
    if (c == '"' || c == '\\') o += '\\', o += c;
    else if (c == '\n') o += "\\n";
    else if (c == '\t') o += "\\t";
    else o += c;
  }
  return o + "\"";
}

const char* status_key(SolveStatus s) { return to_string(s); }

SolveStatus status_from(const std::string& k) {
  for (SolveStatus s : {SolveStatus::kOptimal, SolveStatus::kPrimalInfeasible, SolveStatus::kDualInfeasible,
                        SolveStatus::kPrimalDualInfeasible, SolveStatus::kIterationLimit, SolveStatus::kTimeLimit})
    if (k == to_string(s)) return s;
  throw std::invalid_argument("parse_solution_json: unknown status '" + k + "'");
}

void put_vector(std::string& o, const Vector& v, Index threshold) {
  if (static_cast<Index>(v.size()) > threshold) {
    o += "{\"elided\": true, \"length\": " + std::to_string(v.size()) + "}";
    return;
  }
  o += "[";
  for (size_t i = 0; i < v.size(); ++i) o += (i ? ", " : "") + jnum(v[i]);
  o += "]";
}

std::optional<Vector> get_vector(const JVal* v) {
  if (!v || v->kind == JVal::kNull) return std::nullopt;
  if (v->kind == JVal::kObj) return std::nullopt;  // elided
  Vector out;
  for (const JVal& e : v->arr) out.push_back(jget_num(&e));
  return out;
}

void put_cert(std::string& o, const Certificate& c, Index threshold) {
  o += "{\"source\": ";
  o += jstr(c.source == CandidateSource::kNormalizedIterate ? "normalized_iterate" : "iterate_difference");
  o += ", \"orientation\": ";
  o += jstr(c.orientation == Orientation::kNegated ? "negated" : "as_is");
  o += ", \"at_iteration\": " + std::to_string(c.at_iteration);
  o += ", \"residual\": " + jnum(c.residual) + ", \"margin\": " + jnum(c.margin) + ", \"vector\": ";
  put_vector(o, c.vector, threshold);
  o += "}";
}

std::optional<Certificate> get_cert(const JVal* v) {
  if (!v || v->kind != JVal::kObj) return std::nullopt;
  Certificate c;
  const JVal* s = v->get("source");
  c.source = s && s->str == "normalized_iterate" ? CandidateSource::kNormalizedIterate
                                                 : CandidateSource::kIterateDifference;
  const JVal* o = v->get("orientation");
  c.orientation = o && o->str == "negated" ? Orientation::kNegated : Orientation::kAsIs;
  c.at_iteration = static_cast<long>(jget_num(v->get("at_iteration")));
  c.residual = jget_num(v->get("residual"));
  c.margin = jget_num(v->get("margin"));
  if (auto vec = get_vector(v->get("vector"))) c.vector = *vec;
  return c;
}

}  // namespace

GeneralFormLP parse_mps(std::istream& in, MpsDocument* doc) {
  Parser p;
  p.doc = doc;
  return p.run(in);
}

GeneralFormLP parse_mps(const std::string& text, MpsDocument* doc) {
  std::istringstream in(text);
  return parse_mps(in, doc);
}

GeneralFormLP parse_mps_file(const std::string& path, MpsDocument* doc) {
  std::ifstream in(path);
  if (!in) throw MpsParseError(0, "cannot open '" + path + "'");
  return parse_mps(in, doc);
}

std::string write_mps(const GeneralFormLP& g) {
  const Index m = g.num_rows(), n = g.num_cols();
  auto raw_r = [&](Index i) { return g.rows[i].name.empty() ? "R" + std::to_string(i) : g.rows[i].name; };
  auto raw_c = [&](Index j) { return g.columns[j].name.empty() ? "C" + std::to_string(j) : g.columns[j].name; };
  const std::string raw_obj = g.objective_name.empty() ? "OBJ" : g.objective_name;
  // Names with blanks only survive in fixed format (8-character fields); if
  // one does not fit, free format with the blanks replaced by '_'.
  bool blanks = raw_obj.find(' ') != std::string::npos, fits = raw_obj.size() <= 8;
  for (Index i = 0; i < m; ++i) blanks |= raw_r(i).find(' ') != std::string::npos, fits &= raw_r(i).size() <= 8;
  for (Index j = 0; j < n; ++j) blanks |= raw_c(j).find(' ') != std::string::npos, fits &= raw_c(j).size() <= 8;
  const bool fixed = blanks && fits;
  auto clean = [&](std::string s) {
    if (!fixed)
      for (char& ch : s)
        if (ch == ' ') ch = '_';
    return s;
  };
  auto rname = [&](Index i) { return clean(raw_r(i)); };
  auto cname = [&](Index j) { return clean(raw_c(j)); };
  const std::string obj = clean(raw_obj);
  // one data line: fields at 1-based columns 2, 5, 15, 25, 40, 50 (fixed) or
  // blank separated (free)
  auto line = [&](std::initializer_list<std::string> f) {
    static const int kStart[] = {1, 4, 14, 24, 39, 49};
    std::string l;
    int k = 0;
    for (const std::string& x : f) {
      if (fixed) {
        if (static_cast<int>(l.size()) < kStart[k]) l.resize(kStart[k], ' ');
        else if (!x.empty() && k > 0) l += ' ';
        l += x;
      } else if (!x.empty()) {
        l += (k == 0 ? " " : (k == 1 && l.empty() ? "    " : " ")) + x;
      }
      ++k;
    }
    return l + "\n";
  };
  std::string o = "NAME " + g.name + "\n";
  if (g.maximize) o += "OBJSENSE\n    MAX\n";
  o += "ROWS\n" + line({"N", obj});
  for (Index i = 0; i < m; ++i) {
    const char* t = g.rows[i].relation == RowRelation::kLessEqual      ? "L"
                    : g.rows[i].relation == RowRelation::kGreaterEqual ? "G"
                                                                       : "E";
    o += line({t, rname(i)});
  }
  o += "COLUMNS\n";
  // entries grouped by column, in their order within the column
  std::vector<std::vector<std::pair<Index, double>>> by_col(static_cast<size_t>(n));
  for (const Triplet& t : g.entries) {
    if (t.row < 0 || t.row >= m || t.col < 0 || t.col >= n) throw std::invalid_argument("write_mps: entry out of range");
    by_col[t.col].push_back({t.row, t.value});
  }
  // fixed fields are 12 characters wide for numbers: %.17g needs up to 24, so
  // fixed-format numbers are written in free-form positions after the field
  // start (the reader takes fields by position up to the next one)
  for (Index j = 0; j < n; ++j) {
    const double cj = j < static_cast<Index>(g.objective.size()) ? g.objective[j] : 0.0;
    if (cj != 0.0 || by_col[j].empty()) o += line({"", cname(j), obj, num17(cj)});
    for (const auto& [i, v] : by_col[j]) o += line({"", cname(j), rname(i), num17(v)});
  }
  o += "RHS\n";
  if (g.objective_constant != 0.0) o += line({"", "RHS", obj, num17(-g.objective_constant)});
  for (Index i = 0; i < m; ++i)
    if (g.rows[i].rhs != 0.0) o += line({"", "RHS", rname(i), num17(g.rows[i].rhs)});
  bool any_range = false;
  for (Index i = 0; i < m; ++i) any_range |= g.rows[i].range.has_value();
  if (any_range) {
    o += "RANGES\n";
    for (Index i = 0; i < m; ++i)
      if (g.rows[i].range) o += line({"", "RNG", rname(i), num17(*g.rows[i].range)});
  }
  o += "BOUNDS\n";
  for (Index j = 0; j < n; ++j) {
    const double lo = g.columns[j].lower, up = g.columns[j].upper;
    const std::string c = cname(j);
    if (lo == -kInf && up == kInf) {
      o += line({"FR", "BND", c});
    } else if (lo == up) {
      o += line({"FX", "BND", c, num17(lo)});
    } else {
      if (lo == -kInf) o += line({"MI", "BND", c});
      else if (lo != 0.0 || (up < 0.0)) o += line({"LO", "BND", c, num17(lo)});
      if (up != kInf) o += line({"UP", "BND", c, num17(up)});
    }
  }
  o += "ENDATA\n";
  return o;
}

std::string write_solution_json(const SolutionReport& r, const JsonWriteOptions& opt) {
  const Index th = opt.vector_elision_threshold;
  std::string o = "{\n";
  o += "  \"instance\": " + jstr(r.instance) + ",\n";
  o += "  \"status\": " + jstr(status_key(r.status)) + ",\n";
  o += "  \"primal_objective\": " + jnum(r.primal_objective) + ",\n";
  o += "  \"dual_objective\": " + jnum(r.dual_objective) + ",\n";
  o += "  \"kkt\": {\"primal\": " + jnum(r.kkt.primal_residual) + ", \"dual\": " + jnum(r.kkt.dual_residual) +
       ", \"gap\": " + jnum(r.kkt.gap_residual) + ", \"max\": " + jnum(r.kkt.max_relative) + "},\n";
  o += "  \"iterations\": " + std::to_string(r.iterations) + ",\n";
  o += "  \"epochs\": " + std::to_string(r.epochs) + ",\n";
  o += "  \"spmv_count\": " + std::to_string(r.spmv_count) + ",\n";
  o += "  \"eta\": " + jnum(r.eta) + ",\n";
  o += "  \"sigma_estimate\": " + jnum(r.sigma_estimate) + ",\n";
  o += "  \"primal_solution\": ";
  if (r.primal_solution) put_vector(o, *r.primal_solution, th);
  else o += "null";
  o += ",\n  \"dual_solution\": ";
  if (r.dual_solution) put_vector(o, *r.dual_solution, th);
  else o += "null";
  o += ",\n  \"primal_certificate\": ";
  if (r.primal_certificate) put_cert(o, *r.primal_certificate, th);
  else o += "null";
  o += ",\n  \"dual_certificate\": ";
  if (r.dual_certificate) put_cert(o, *r.dual_certificate, th);
  else o += "null";
  o += ",\n  \"config\": [";
  for (size_t k = 0; k < r.config_echo.size(); ++k)
    o += std::string(k ? ", " : "") + "[" + jstr(r.config_echo[k].first) + ", " + jstr(r.config_echo[k].second) + "]";
  o += "]";
  if (opt.include_timing) o += ",\n  \"timing\": {\"solve_seconds\": " + jnum(r.solve_seconds) + "}";
  o += "\n}\n";
  return o;
}

SolutionReport parse_solution_json(const std::string& text) {
  JParser jp{text};
  const JVal root = jp.value();
  if (root.kind != JVal::kObj) throw std::invalid_argument("parse_solution_json: top level must be an object");
  SolutionReport r;
  if (const JVal* v = root.get("instance")) r.instance = v->str;
  const JVal* st = root.get("status");
  if (!st || st->kind != JVal::kStr) throw std::invalid_argument("parse_solution_json: missing status");
  r.status = status_from(st->str);
  r.primal_objective = jget_num(root.get("primal_objective"));
  r.dual_objective = jget_num(root.get("dual_objective"));
  if (const JVal* k = root.get("kkt")) {
    r.kkt.primal_residual = jget_num(k->get("primal"));
    r.kkt.dual_residual = jget_num(k->get("dual"));
    r.kkt.gap_residual = jget_num(k->get("gap"));
    r.kkt.max_relative = jget_num(k->get("max"));
  }
  r.iterations = static_cast<long>(jget_num(root.get("iterations")));
  r.epochs = static_cast<long>(jget_num(root.get("epochs")));
  r.spmv_count = static_cast<long>(jget_num(root.get("spmv_count")));
  r.eta = jget_num(root.get("eta"));
  r.sigma_estimate = jget_num(root.get("sigma_estimate"));
  r.primal_solution = get_vector(root.get("primal_solution"));
  r.dual_solution = get_vector(root.get("dual_solution"));
  r.primal_certificate = get_cert(root.get("primal_certificate"));
  r.dual_certificate = get_cert(root.get("dual_certificate"));
  if (const JVal* c = root.get("config"))
    for (const JVal& kv : c->arr)
      if (kv.arr.size() == 2) r.config_echo.push_back({kv.arr[0].str, kv.arr[1].str});
  if (const JVal* t = root.get("timing")) r.solve_seconds = jget_num(t->get("solve_seconds"));
  return r;
}

std::string write_trace_csv(const std::vector<TraceRecord>& trace) {
  std::string o =
      "iteration,epoch,inner,fixed_point_residual,kkt_primal,kkt_dual,kkt_gap,kkt_max,partition_n,partition_b1,"
      "partition_b2,candidate_norm_normalized,candidate_norm_difference,wall_seconds\n";
  for (const TraceRecord& t : trace) {
    o += std::to_string(t.iteration) + "," + std::to_string(t.epoch) + "," + std::to_string(t.inner) + "," +
         num17(t.fixed_point_residual) + "," + num17(t.kkt.primal_residual) + "," + num17(t.kkt.dual_residual) + "," +
         num17(t.kkt.gap_residual) + "," + num17(t.kkt.max_relative) + "," + std::to_string(t.partition.n_set.size()) +
         "," + std::to_string(t.partition.b1_set.size()) + "," + std::to_string(t.partition.b2_set.size()) + "," +
         num17(t.candidate_norm_normalized) + "," + num17(t.candidate_norm_difference) + "," + num17(t.wall_seconds) +
         "\n";
  }
  return o;
}

}  // namespace hplp_gpu
