// sdf_reader.h -- native SDF delay reader (host C++), included by glsim_cuda.cu.
//
// Design ingest for the path: one pass over the SDF text
// straight to the flat arrays the engine takes -- arc_rows [R][2] (rise, fall
// per condition row, gates in order, pins in order, 2^(k-1) rows each) and
// pin_ic [sum k] -- with the semantics of the reference's parse_sdf
// (pkg/src/glsim/sdf.py:229-503) as restated in paper_2203_06117_b200/sdf.py:
// s-expression lexer ("//" comments, quoted strings); one DELAYFILE form;
// TIMESCALE (1|10|100 s..fs), DIVIDER; CELL / INSTANCE / DELAY ABSOLUTE with
// IOPATH, COND-qualified IOPATH (conjunctions of pin literals, later entries
// overwrite earlier ones) and INTERCONNECT; min:typ:max values collapsed to a
// corner; everything else skipped with the reference's warning text.
//
// Errors carry the reference's messages and positions.  Input the
// restatement does not cover byte for byte -- non-ASCII text, numbers Python
// float() reads but this reader does not (inf, nan, underscores), negative
// delays (their message prints a Python float), nested forms inside a delay
// value, an empty DIVIDER -- returns SDF_FALLBACK and the caller uses the
// Python reader.
#pragma once
#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <string>
#include <string_view>
#include <unordered_map>
#include <vector>

#include "vcd_reader.h"  // py_repr

namespace gssdf {

enum Status { SDF_OK = 0, SDF_PARSE = 1, SDF_SEMANTIC = 2, SDF_FALLBACK = 3 };

// the netlist side of the annotation (gate and net names, cells, wiring)
struct Design {
  std::vector<std::string> gate_names, net_names;
  std::vector<int> gate_cell;                 // [G]
  std::vector<std::vector<std::string>> cell_inputs;
  std::vector<std::string> cell_output;
  std::vector<int64_t> pin_off;               // [G+1]
  std::vector<int64_t> pin_net;               // [sum k]
  std::vector<int64_t> out_net;               // [G]
};

struct Result {
  std::vector<int64_t> arc_rows;  // [R*2]
  std::vector<int64_t> pin_ic;    // [sum k]
  int64_t timescale_fs = 1000000;
  std::vector<std::string> warnings;
  std::string msg;
  int64_t line = 0, col = 0;      // position of a parse error (0 = none)
};

struct Kids {        // a list's elements: node indices (a view into one flat store)
  const int *p = nullptr;
  size_t n = 0;
  size_t size() const { return n; }
  bool empty() const { return n == 0; }
  int operator[](size_t i) const { return p[i]; }
  int back() const { return p[n - 1]; }
  const int *begin() const { return p; }
  const int *end() const { return p + n; }
};

struct Node {        // a token or a list
  bool list = false;
  int32_t line = 0, col = 0;      // (documents beyond 2^31 lines or columns fall back)
  std::string_view text;          // token
  Kids kids;                      // list: set once the whole document is read
  int64_t kbeg = 0;               // list: first element in the flat store
};

struct Fail {
  Status st;
  std::string msg;
  int64_t line, col;
};

inline bool py_space(unsigned char c) {
  return c == ' ' || (c >= 9 && c <= 13) || (c >= 28 && c <= 31);
}

inline std::string_view py_strip(std::string_view s) {
  size_t a = 0, b = s.size();
  while (a < b && py_space((unsigned char)s[a])) ++a;
  while (b > a && py_space((unsigned char)s[b - 1])) --b;
  return s.substr(a, b - a);
}

inline std::string upper(std::string_view s) {
  std::string o(s);
  for (auto &c : o)
    if (c >= 'a' && c <= 'z') c = (char)(c - 'a' + 'A');
  return o;
}

// a decimal number Python float() reads the same way strtod does
inline bool plain_number(std::string_view f) {
  size_t i = 0, n = f.size();
  if (i < n && (f[i] == '+' || f[i] == '-')) ++i;
  size_t d0 = i;
  while (i < n && f[i] >= '0' && f[i] <= '9') ++i;
  size_t nd = i - d0;
  if (i < n && f[i] == '.') {
    ++i;
    size_t f0 = i;
    while (i < n && f[i] >= '0' && f[i] <= '9') ++i;
    nd += i - f0;
  }
  if (nd == 0) return false;
  if (i < n && (f[i] == 'e' || f[i] == 'E')) {
    ++i;
    if (i < n && (f[i] == '+' || f[i] == '-')) ++i;
    size_t e0 = i;
    while (i < n && f[i] >= '0' && f[i] <= '9') ++i;
    if (i == e0) return false;
  }
  return i == n;
}

// could Python float() accept it even though plain_number() does not?
inline bool maybe_py_float(std::string_view f) {
  std::string l;
  for (char c : f) {
    if (py_space((unsigned char)c)) continue;
    l += (char)(c >= 'A' && c <= 'Z' ? c - 'A' + 'a' : c);
  }
  std::string_view v(l);
  if (!v.empty() && (v[0] == '+' || v[0] == '-')) v.remove_prefix(1);
  if (v == "inf" || v == "infinity" || v == "nan") return true;
  for (char c : l)
    if (!((c >= '0' && c <= '9') || c == '+' || c == '-' || c == '.' || c == '_' || c == 'e'))
      return false;
  return true;
}

class Reader {
 public:
  Reader(const char *text, int64_t len, const Design &d, int corner, const std::string &path,
         Result &r)
      : t_(text), n_(len), d_(d), corner_(corner), path_(path), r_(r) {}

  Status run() {
    for (int64_t i = 0; i < n_; ++i)
      if ((unsigned char)t_[i] >= 0x80 || t_[i] == 0) return SDF_FALLBACK;
    try {
      lex_and_build();
      annotate();
    } catch (const Fail &f) {
      r_.msg = f.msg;
      r_.line = f.line;
      r_.col = f.col;
      return f.st;
    }
    return SDF_OK;
  }

 private:
  const char *t_;
  int64_t n_;
  const Design &d_;
  int corner_;  // 0 min, 1 typ, 2 max
  std::string path_;
  Result &r_;
  std::vector<Node> nodes_;
  std::vector<int> store_;  // list elements, one run per list
  int root_ = -1;
  std::string divider_ = "/";
  std::unordered_map<std::string_view, int> gate_index_, net_index_;
  std::vector<int64_t> row_off_;  // first arc row of (gate, pin): pin_off-indexed

  [[noreturn]] void parse_fail(const std::string &m, int64_t line, int64_t col) {
    throw Fail{SDF_PARSE, m, line, col};
  }
  [[noreturn]] void fallback() { throw Fail{SDF_FALLBACK, "", 0, 0}; }

  // ---- lexer + s-expressions (sdf.py _lex / _sexprs)
  void lex_and_build() {
    if (n_ >= INT32_MAX) fallback();
    nodes_.reserve((size_t)(n_ / 4 + 16));
    std::vector<int> stack;         // open lists
    std::vector<size_t> mark;       // their first element on `pending`
    std::vector<int> pending;       // elements of the open lists, innermost last
    std::vector<size_t> kn;         // element count per node (lists)
    store_.reserve((size_t)(n_ / 4 + 16));
    Node root;
    root.list = true;
    root.line = root.col = 1;
    nodes_.push_back(root);
    root_ = 0;
    stack.push_back(0);
    mark.push_back(0);
    int64_t i = 0, line = 1, col = 1;
    auto token = [&](std::string_view s, int64_t l, int64_t c) {
      Node nd;
      nd.line = (int32_t)l;
      nd.col = (int32_t)c;
      nd.text = s;
      nodes_.push_back(nd);
      pending.push_back((int)nodes_.size() - 1);
    };
    auto close = [&]() {  // move the innermost list's elements to the store
      const int id = stack.back();
      const size_t m = mark.back();
      nodes_[id].kbeg = (int64_t)store_.size();
      if (kn.size() < nodes_.size()) kn.resize(nodes_.size() * 2 + 16, 0);
      kn[id] = pending.size() - m;
      store_.insert(store_.end(), pending.begin() + (long)m, pending.end());
      pending.resize(m);
      stack.pop_back();
      mark.pop_back();
    };
    while (i < n_) {
      const char c = t_[i];
      if (c == '\n') {
        ++i;
        ++line;
        col = 1;
      } else if (c == ' ' || c == '\t' || c == '\r') {
        ++i;
        ++col;
      } else if (c == '/' && i + 1 < n_ && t_[i + 1] == '/') {
        while (i < n_ && t_[i] != '\n') ++i;
      } else if (c == '(') {
        Node nd;
        nd.list = true;
        nd.line = (int32_t)line;
        nd.col = (int32_t)col;
        nodes_.push_back(nd);
        const int id = (int)nodes_.size() - 1;
        pending.push_back(id);
        stack.push_back(id);
        mark.push_back(pending.size());
        ++i;
        ++col;
      } else if (c == ')') {
        if (stack.size() == 1) parse_fail("unbalanced ')'", line, col);
        close();
        ++i;
        ++col;
      } else if (c == '"') {
        int64_t j = i + 1;
        while (j < n_ && t_[j] != '"') ++j;
        if (j >= n_) parse_fail("unterminated string", line, col);
        // a quoted "(" or ")" is a parenthesis to the Python reader
        if (j - i - 1 == 1 && (t_[i + 1] == '(' || t_[i + 1] == ')')) fallback();
        token(std::string_view(t_ + i + 1, (size_t)(j - i - 1)), line, col);
        col += j + 1 - i;
        i = j + 1;
      } else {
        int64_t j = i;
        while (j < n_) {
          const char x = t_[j];
          if (x == ' ' || x == '\t' || x == '\r' || x == '\n' || x == '(' || x == ')' || x == '"')
            break;
          ++j;
        }
        token(std::string_view(t_ + i, (size_t)(j - i)), line, col);
        col += j - i;
        i = j;
      }
    }
    if (stack.size() != 1) {
      const Node &o = nodes_[stack.back()];
      parse_fail("unbalanced '('", o.line, o.col);
    }
    close();  // the document's top-level forms
    if (kn.size() < nodes_.size()) kn.resize(nodes_.size(), 0);
    for (size_t k = 0; k < nodes_.size(); ++k)
      if (nodes_[k].list) nodes_[k].kids = Kids{store_.data() + nodes_[k].kbeg, kn[k]};
  }

  const Node &N(int id) const { return nodes_[id]; }
  // keyword of a form: its first element upper-cased when that is a token
  bool keyword(int id, std::string *kw) const {
    const Node &n = N(id);
    if (!n.list || n.kids.empty() || N(n.kids[0]).list) return false;
    *kw = upper(N(n.kids[0]).text);
    return true;
  }
  std::string kw_or_none(int id) const {
    std::string k;
    return keyword(id, &k) ? k : std::string("None");
  }
  // position of a form: its first token, descending into first elements
  bool where(int id, int64_t *line, int64_t *col) const {
    const Node *n = &N(id);
    while (n->list) {
      if (n->kids.empty()) return false;
      n = &N(n->kids[0]);
    }
    *line = n->line;
    *col = n->col;
    return true;
  }
  [[noreturn]] void fail(const std::string &m, int form, bool semantic = false) {
    int64_t line = 0, col = 0;
    const bool has = where(form, &line, &col);
    if (semantic) {
      throw Fail{SDF_SEMANTIC, has ? path_ + ":" + std::to_string(line) + ": " + m : m, 0, 0};
    }
    throw Fail{SDF_PARSE, m, has ? line : 0, has ? col : 0};
  }
  void warn(const std::string &m, int form) {
    int64_t line = 0, col = 0;
    const bool has = where(form, &line, &col);
    r_.warnings.push_back((has ? path_ + ":" + std::to_string(line) : path_) + ": " + m);
  }

  // ---- annotation (sdf.py parse_sdf / _SdfReader)
  void annotate() {
    const int64_t G = (int64_t)d_.gate_names.size();
    for (int64_t g = 0; g < G; ++g) gate_index_[d_.gate_names[g]] = (int)g;  // last wins
    for (size_t i = 0; i < d_.net_names.size(); ++i) net_index_[d_.net_names[i]] = (int)i;
    row_off_.assign(d_.pin_net.size() + 1, 0);
    int64_t rows = 0;
    for (int64_t g = 0; g < G; ++g) {
      const int64_t k = d_.pin_off[g + 1] - d_.pin_off[g];
      for (int64_t p = 0; p < k; ++p) {
        row_off_[d_.pin_off[g] + p] = rows;
        rows += (int64_t)1 << (k - 1);
      }
    }
    r_.arc_rows.assign((size_t)rows * 2, 0);
    r_.pin_ic.assign(d_.pin_net.size(), 0);
    r_.timescale_fs = 1000000;
    const Node &top = N(root_);
    std::string kw;
    if (top.kids.size() != 1 || !keyword(top.kids[0], &kw) || kw != "DELAYFILE")
      parse_fail("expected a single (DELAYFILE ...) form", 1, 1);
    const Node &df = N(top.kids[0]);
    for (size_t a = 1; a < df.kids.size(); ++a) {
      const int item = df.kids[a];
      if (!keyword(item, &kw)) {
        int64_t line = 0, col = 0;
        where(item, &line, &col);
        parse_fail("expected a (KEYWORD ...) form", line, col);
      }
      if (kw == "TIMESCALE") {
        timescale(item);
      } else if (kw == "DIVIDER") {
        const Node &it = N(item);
        if (it.kids.size() > 1 && !N(it.kids[1]).list) {
          divider_ = std::string(N(it.kids[1]).text);
          if (divider_.empty()) fallback();
        }
      } else if (kw == "CELL") {
        cell(item);
      }
    }
  }

  void timescale(int item) {
    std::string spec;
    const Node &it = N(item);
    for (size_t a = 1; a < it.kids.size(); ++a)
      if (!N(it.kids[a]).list) spec += N(it.kids[a]).text;
    size_t k = spec.size();
    while (k > 0 && spec[k - 1] >= 'a' && spec[k - 1] <= 'z') --k;
    const std::string num = spec.substr(0, k), unit = spec.substr(k);
    static const char *units[] = {"s", "ms", "us", "ns", "ps", "fs"};
    static const int64_t fs[] = {1000000000000000ll, 1000000000000ll, 1000000000ll, 1000000ll,
                                 1000ll, 1ll};
    int ui = -1;
    for (int u = 0; u < 6; ++u)
      if (unit == units[u]) ui = u;
    if (ui < 0 || !(num == "1" || num == "10" || num == "100")) {
      int64_t line = 0, col = 0;
      where(item, &line, &col);
      parse_fail("bad TIMESCALE " + gsvcd::py_repr(spec) +
                     " (expected 1|10|100 s|ms|us|ns|ps|fs)",
                 line, col);
    }
    r_.timescale_fs = std::stoll(num) * fs[ui];
  }

  void cell(int form) {
    const Node &f = N(form);
    bool have_inst = false, inst_named = false;
    std::string_view inst;
    std::string kw;
    for (size_t a = 1; a < f.kids.size(); ++a) {
      const int sub = f.kids[a];
      const bool is_kw = keyword(sub, &kw);
      if (is_kw && kw == "CELLTYPE") continue;
      if (is_kw && kw == "INSTANCE") {
        inst_named = false;
        const Node &s = N(sub);
        for (size_t b = 1; b < s.kids.size(); ++b)
          if (!N(s.kids[b]).list) {
            inst = N(s.kids[b]).text;
            inst_named = true;
            break;
          }
        have_inst = true;
      } else if (is_kw && kw == "DELAY") {
        if (!have_inst) fail("DELAY before INSTANCE in CELL", sub);
        delay(sub, inst_named ? &inst : nullptr);
      } else if (is_kw && (kw == "TIMINGCHECK" || kw == "LABEL" || kw == "TIMINGENV")) {
        warn("skipping unsupported " + kw + " section", sub);
      } else {
        warn("skipping unsupported CELL entry " + (is_kw ? kw : std::string("None")), sub);
      }
    }
  }

  void delay(int form, const std::string_view *inst) {
    const Node &f = N(form);
    std::string kw;
    for (size_t a = 1; a < f.kids.size(); ++a) {
      const int sub = f.kids[a];
      const bool is_kw = keyword(sub, &kw);
      if (is_kw && kw == "ABSOLUTE") {
        const Node &s = N(sub);
        for (size_t b = 1; b < s.kids.size(); ++b) entry(s.kids[b], inst);
      } else if (is_kw && (kw == "PATHPULSE" || kw == "PATHPULSEPERCENT")) {
        warn("skipping " + kw + " entry (pulse handling is a simulator setting)", sub);
      } else {
        warn("skipping unsupported DELAY section " + (is_kw ? kw : std::string("None")), sub);
      }
    }
  }

  void entry(int e, const std::string_view *inst) {
    std::string kw;
    const bool is_kw = keyword(e, &kw);
    if (is_kw && kw == "IOPATH") {
      iopath(e, inst, nullptr);
    } else if (is_kw && kw == "COND") {
      const Node &en = N(e);
      std::string k2;
      if (en.kids.size() < 2 || !keyword(en.kids.back(), &k2) || k2 != "IOPATH")
        fail("COND must wrap an IOPATH entry", e);
      std::vector<int> expr(en.kids.begin() + 1, en.kids.end() - 1);
      if (expr.size() == 1 && N(expr[0]).list) {
        const Kids &in = N(expr[0]).kids;
        expr.assign(in.begin(), in.end());
      }
      std::string cond;
      bool any = false;
      for (int x : expr)
        if (!N(x).list) {
          if (any) cond += ' ';
          cond += N(x).text;
          any = true;
        }
      if (!any) fail("COND requires a condition expression", e);
      iopath(en.kids.back(), inst, &cond);
    } else if (is_kw && kw == "INTERCONNECT") {
      interconnect(e);
    } else if (is_kw && (kw == "PATHPULSE" || kw == "PATHPULSEPERCENT")) {
      warn("skipping " + kw + " entry (pulse handling is a simulator setting)", e);
    } else {
      warn("skipping unsupported delay entry " + (is_kw ? kw : std::string("None")), e);
    }
  }

  int gate_of(const std::string_view *inst, int form) {
    if (!inst) fail("IOPATH requires a named INSTANCE", form);
    auto it = gate_index_.find(*inst);
    if (it == gate_index_.end()) fail("unknown instance " + gsvcd::py_repr(std::string(*inst)), form, true);
    return it->second;
  }

  int input_pin(int g, std::string_view name) const {
    const auto &ins = d_.cell_inputs[d_.gate_cell[g]];
    for (size_t i = 0; i < ins.size(); ++i)
      if (ins[i] == name) return (int)i;
    return -1;
  }

  void iopath(int e, const std::string_view *inst, const std::string *cond) {
    const int g = gate_of(inst, e);
    const Node &en = N(e);
    if (en.kids.size() < 4)
      fail("IOPATH needs input port, output port and at least one delay value", e);
    const Node &src = N(en.kids[1]), &dst = N(en.kids[2]);
    if (src.list) {
      warn("skipping edge-qualified IOPATH", e);
      return;
    }
    if (dst.list) fail("IOPATH output port must be a pin name", e);
    if (dst.text != d_.cell_output[d_.gate_cell[g]])
      fail("gate " + gsvcd::py_repr(std::string(*inst)) + ": unknown output pin " +
               gsvcd::py_repr(std::string(dst.text)),
           e, true);
    const int pin = input_pin(g, src.text);
    if (pin < 0)
      fail("gate " + gsvcd::py_repr(std::string(*inst)) + ": unknown input pin " +
               gsvcd::py_repr(std::string(src.text)),
           e, true);
    int64_t rise = 0, fall = 0;
    for (size_t a = 3; a < en.kids.size(); ++a) {  // every value is read (and checked)
      const int64_t v = value(en.kids[a], e);
      if (a == 3) rise = fall = v;
      if (a == 4) fall = v;
    }
    if (en.kids.size() > 5) warn("ignoring IOPATH delay values beyond rise/fall", e);
    const int64_t k = d_.pin_off[g + 1] - d_.pin_off[g];
    const int64_t nrows = (int64_t)1 << (k - 1);
    int64_t *rows = r_.arc_rows.data() + 2 * row_off_[d_.pin_off[g] + pin];
    if (!cond) {
      for (int64_t r = 0; r < nrows; ++r) {
        rows[2 * r] = rise;
        rows[2 * r + 1] = fall;
      }
      return;
    }
    // literals of the conjunction, all validated before any row is touched
    std::vector<std::pair<int, int>> lits;
    std::string_view cs(*cond);
    size_t pos = 0;
    while (true) {
      const size_t nx = cs.find("&&", pos);
      std::string_view term = py_strip(cs.substr(pos, nx == std::string_view::npos ? cs.npos : nx - pos));
      if (term.empty()) fail("empty term in COND expression", e);
      std::string_view name;
      int want;
      const size_t eq = term.find("==");
      if (eq != std::string_view::npos) {
        name = py_strip(term.substr(0, eq));
        std::string_view val = py_strip(term.substr(eq + 2));
        if (!(val == "0" || val == "1" || val == "1'b0" || val == "1'b1"))
          fail("unsupported COND comparison value " + gsvcd::py_repr(std::string(val)), e);
        want = (val == "1" || val == "1'b1") ? 1 : 0;
      } else if (term[0] == '!') {
        name = py_strip(term.substr(1));
        want = 0;
      } else {
        name = term;
        want = 1;
      }
      const int q = input_pin(g, name);
      if (q < 0)
        fail("gate " + gsvcd::py_repr(std::string(*inst)) + ": COND references unknown pin " +
                 gsvcd::py_repr(std::string(name)),
             e, true);
      if (q == pin)
        fail("gate " + gsvcd::py_repr(std::string(*inst)) + ": COND references the switching pin " +
                 gsvcd::py_repr(std::string(name)),
             e, true);
      lits.emplace_back(q, want);
      if (nx == std::string_view::npos) break;
      pos = nx + 2;
    }
    int64_t mask = 0, bits = 0;
    for (auto &l : lits) {
      const int side = l.first < pin ? l.first : l.first - 1;  // index among the other pins
      const int64_t bit = (int64_t)1 << side;
      if ((mask & bit) && (((bits & bit) != 0) != (l.second != 0))) return;  // contradiction
      mask |= bit;
      if (l.second) bits |= bit;
    }
    for (int64_t r = 0; r < nrows; ++r)
      if ((r & mask) == bits) {
        rows[2 * r] = rise;
        rows[2 * r + 1] = fall;
      }
  }

  void interconnect(int e) {
    const Node &en = N(e);
    if (en.kids.size() != 4)
      fail("INTERCONNECT needs source port, destination port and one delay value", e);
    const Node &src = N(en.kids[1]), &dst = N(en.kids[2]);
    if (src.list || dst.list) fail("INTERCONNECT ports must be names", e);
    const int64_t v = value(en.kids[3], e);
    const std::string s(src.text), t(dst.text);
    const int64_t net = source_net(s, e);
    int g = 0, pin = 0;
    sink_pin(t, e, &g, &pin);
    if (d_.pin_net[d_.pin_off[g] + pin] != net)
      fail("INTERCONNECT " + gsvcd::py_repr(s) + " -> " + gsvcd::py_repr(t) +
               " does not match netlist connectivity",
           e, true);
    r_.pin_ic[d_.pin_off[g] + pin] = v;
  }

  int64_t source_net(const std::string &src, int e) {
    const size_t at = src.rfind(divider_);
    if (at != std::string::npos) {
      const std::string gname = src.substr(0, at), pname = src.substr(at + divider_.size());
      auto it = gate_index_.find(std::string_view(gname));
      if (it == gate_index_.end()) fail("unknown instance " + gsvcd::py_repr(gname), e, true);
      const int g = it->second;
      if (pname != d_.cell_output[d_.gate_cell[g]])
        fail("INTERCONNECT source " + gsvcd::py_repr(src) + " is not a driver pin", e, true);
      return d_.out_net[g];
    }
    auto it = net_index_.find(std::string_view(src));
    if (it == net_index_.end()) fail("unknown net " + gsvcd::py_repr(src), e, true);
    return it->second;
  }

  void sink_pin(const std::string &dst, int e, int *g, int *pin) {
    const size_t at = dst.rfind(divider_);
    if (at == std::string::npos)
      fail("INTERCONNECT destination " + gsvcd::py_repr(dst) + " must name a gate input pin",
           e, true);
    const std::string gname = dst.substr(0, at), pname = dst.substr(at + divider_.size());
    auto it = gate_index_.find(std::string_view(gname));
    if (it == gate_index_.end()) fail("unknown instance " + gsvcd::py_repr(gname), e, true);
    *g = it->second;
    *pin = input_pin(*g, pname);
    if (*pin < 0)
      fail("gate " + gsvcd::py_repr(gname) + ": unknown pin " + gsvcd::py_repr(pname), e, true);
  }

  // (v), (min:typ:max) with blanks, or () -> integer fs
  int64_t value(int form, int e) {
    const Node &f = N(form);
    if (!f.list) fail("delay value must be parenthesized", e);
    std::string joined;
    std::string_view spec;
    if (f.kids.size() == 1 && !N(f.kids[0]).list) {
      spec = N(f.kids[0]).text;  // the usual single token, no copy
    } else {
      for (int x : f.kids) {
        if (N(x).list) fallback();  // str() of a nested form: Python list repr
        joined += N(x).text;
      }
      spec = joined;
    }
    if (spec.empty()) return 0;
    std::string_view fields[3];
    size_t nf = 0, p = 0;
    while (true) {
      const size_t c = spec.find(':', p);
      const std::string_view fld = spec.substr(p, c == std::string_view::npos ? spec.npos : c - p);
      if (nf < 3) fields[nf] = fld;
      ++nf;
      if (c == std::string_view::npos) break;
      p = c + 1;
    }
    if (nf == 1) fields[1] = fields[2] = fields[0];
    else if (nf != 3) fail("bad delay value " + gsvcd::py_repr(std::string(spec)), form);
    double num[3];
    bool have[3];
    for (int i = 0; i < 3; ++i) {
      have[i] = !fields[i].empty();
      if (!have[i]) continue;
      if (!plain_number(fields[i])) {
        // Python float() may still read it (inf, nan, 1_0, surrounding
        // spaces): let the Python reader decide; anything else is no number
        if (maybe_py_float(fields[i])) fallback();
        fail("bad delay number " + gsvcd::py_repr(std::string(fields[i])), form);
      }
      char buf[64];
      if (fields[i].size() >= sizeof buf) fallback();
      memcpy(buf, fields[i].data(), fields[i].size());
      buf[fields[i].size()] = 0;
      num[i] = std::strtod(buf, nullptr);
    }
    int pick = corner_;
    if (!have[pick]) {
      static const int order[] = {1, 0, 2};  // typ, min, max
      pick = -1;
      for (int o : order)
        if (have[o]) {
          pick = o;
          break;
        }
    }
    if (pick < 0) return 0;
    const double v = num[pick];
    if (!std::isfinite(v) || v < 0) fallback();  // negative: message prints a Python float
    const double s = v * (double)r_.timescale_fs;
    if (!(s < 4.0e18)) fallback();
    return (int64_t)std::nearbyint(s);  // round half to even, as Python round()
  }
};

inline Status parse(const char *text, int64_t len, const Design &d, int corner,
                    const std::string &path, Result &r) {
  Reader rd(text, len, d, corner, path, r);
  return rd.run();
}

}  // namespace gssdf
