// vcd_reader.h -- native VCD stimulus reader (host C++), included by glsim_cuda.cu.
//
// The stimulus document immediately upstream of the path:
// one streaming pass over the text produces the per-input CSR waveforms K1
// consumes (pi_off / pi_times / pi_init), with the semantics of the
// reference's parse_vcd (pkg/src/glsim/waveform.py:101-198) as restated in
// paper_2203_06117_b200/waveform.py: whitespace tokens; `$keyword ... $end`
// sections across lines, of which only `$timescale` (1|10|100 s..fs) and
// `$var` (scalar inputs; aliases of a bound input ignored) matter; `#t`
// time marks scaled to fs and non-decreasing; `0 1 x X z Z` scalar changes
// (x/z read as 0) on bound identifiers, at or before time 0 setting the
// initial value; repeated values collapse; two changes at one time mark
// leave the later one; `b B r R` vector/real changes skip their identifier.
//
// Errors carry the reference's messages (ParseError with the 1-based line,
// SemanticError).  Input the restatement does not cover byte for byte --
// non-ASCII text, Unicode line/space separators, integers beyond int64 --
// returns VCD_FALLBACK and the caller uses the Python reader.
#pragma once
#include <cstdint>
#include <cstdio>
#include <deque>
#include <string>
#include <string_view>
#include <unordered_map>
#include <vector>

namespace gsvcd {

enum Status { VCD_OK = 0, VCD_PARSE = 1, VCD_SEMANTIC = 2, VCD_FALLBACK = 3 };

struct Result {
  std::vector<int64_t> pi_off, pi_times;
  std::vector<uint8_t> pi_init;
  int64_t duration = 0;
  std::string msg;  // error message (reference wording)
  int64_t line = 0; // 1-based line of a parse error
};

// Python repr() of an ASCII string (the messages quote tokens with !r)
inline std::string py_repr(const std::string &s) {
  const bool sq = s.find('\'') != std::string::npos, dq = s.find('"') != std::string::npos;
  const char q = (sq && !dq) ? '"' : '\'';
  std::string o(1, q);
  for (unsigned char c : s) {
    if (c == '\\') o += "\\\\";
    else if (c == (unsigned char)q) { o += '\\'; o += (char)c; }
    else if (c == '\n') o += "\\n";
    else if (c == '\r') o += "\\r";
    else if (c == '\t') o += "\\t";
    else if (c < 0x20 || c == 0x7f) {
      char b[8];
      snprintf(b, sizeof b, "\\x%02x", c);
      o += b;
    } else o += (char)c;
  }
  o += q;
  return o;
}

// Python int() of an ASCII token: optional sign, digits with single
// underscores between them.  Returns false if malformed; *overflow if it
// does not fit int64.
inline bool py_int(const char *p, const char *e, int64_t *v, bool *overflow) {
  *overflow = false;
  bool neg = false;
  if (p < e && (*p == '+' || *p == '-')) neg = *p++ == '-';
  if (p == e || !(*p >= '0' && *p <= '9')) return false;
  unsigned long long acc = 0;
  bool prev_us = false;
  for (; p < e; ++p) {
    if (*p == '_') {
      if (prev_us) return false;
      prev_us = true;
      continue;
    }
    if (!(*p >= '0' && *p <= '9')) return false;
    prev_us = false;
    if (acc > (~0ull - 9) / 10) *overflow = true;
    acc = acc * 10 + (unsigned)(*p - '0');
  }
  if (prev_us) return false;
  if (acc > (unsigned long long)INT64_MAX + (neg ? 1ull : 0ull)) *overflow = true;
  *v = neg ? (int64_t)(0 - acc) : (int64_t)acc;
  return true;
}

inline bool is_ws(unsigned char c) { return c == ' ' || c == '\t' || c == '\n' || c == '\r'; }

inline Status parse(const char *text, int64_t len, const std::vector<std::string> &pi_names,
                    Result &R) {
  const int P = (int)pi_names.size();
  // bytes the Python reader would split or decode differently
  for (int64_t i = 0; i < len; ++i) {
    const unsigned char c = (unsigned char)text[i];
    if (c >= 0x80 || c == 0x0b || c == 0x0c || (c >= 0x1c && c <= 0x1f) || c == 0) return VCD_FALLBACK;
  }
  std::unordered_map<std::string, int> pi_of;
  pi_of.reserve(P * 2 + 1);
  for (int i = 0; i < P; ++i) pi_of[pi_names[i]] = i;  // a repeated name: the last index
  std::deque<std::string> idents;                   // storage behind the keys below
  std::unordered_map<std::string_view, int> bound;  // identifier -> input
  std::vector<int> bound_refs(P, 0);            // how many identifiers map to each input
  std::vector<uint8_t> value(P, 0), initial(P, 0);
  std::vector<std::vector<int64_t>> tog(P);
  int64_t scale = -1, now = -1, duration = 0;

  // line/token cursor over the text (lines end at \n, \r\n or \r)
  int64_t pos = 0, lineno = 1;
  auto next_token = [&](const char **b, const char **e, int64_t *tok_line) -> bool {
    while (pos < len) {
      const char c = text[pos];
      if (c == '\n') { ++pos; ++lineno; continue; }
      if (c == '\r') { ++pos; if (pos < len && text[pos] == '\n') ++pos; ++lineno; continue; }
      if (c == ' ' || c == '\t') { ++pos; continue; }
      break;
    }
    if (pos >= len) return false;
    const int64_t s = pos;
    while (pos < len && !is_ws((unsigned char)text[pos])) ++pos;
    *b = text + s;
    *e = text + pos;
    *tok_line = lineno;
    return true;
  };
  auto fail_parse = [&](const std::string &m, int64_t line) {
    R.msg = m;
    R.line = line;
    return VCD_PARSE;
  };
  static const char *units[] = {"s", "ms", "us", "ns", "ps", "fs"};
  static const int64_t unit_fs[] = {1000000000000000ll, 1000000000000ll, 1000000000ll, 1000000ll,
                                    1000ll, 1ll};
  const char *b, *e;
  int64_t tl;
  while (next_token(&b, &e, &tl)) {
    const char c = *b;
    if (c == '$') {
      const std::string kw(b, e);
      std::vector<std::string> body;
      bool closed = false;
      int64_t end_line = tl;
      while (next_token(&b, &e, &end_line)) {
        if (e - b == 4 && std::string(b, e) == "$end") {
          closed = true;
          break;
        }
        body.emplace_back(b, e);
      }
      if (!closed) {
        // the Python reader reports the line count of the document
        int64_t nlines = 0;
        {
          int64_t i = 0;
          while (i < len) {
            ++nlines;
            while (i < len && text[i] != '\n' && text[i] != '\r') ++i;
            if (i < len) {
              if (text[i] == '\r' && i + 1 < len && text[i + 1] == '\n') ++i;
              ++i;
            }
          }
        }
        return fail_parse("unterminated " + kw + " section", nlines);
      }
      if (kw == "$timescale") {
        std::string spec;
        for (auto &t : body) spec += t;
        size_t k = spec.size();
        while (k > 0 && spec[k - 1] >= 'a' && spec[k - 1] <= 'z') --k;
        const std::string num = spec.substr(0, k), unit = spec.substr(k);
        int ui = -1;
        for (int u = 0; u < 6; ++u)
          if (unit == units[u]) ui = u;
        if (ui < 0 || !(num == "1" || num == "10" || num == "100"))
          return fail_parse("bad $timescale " + py_repr(spec), end_line);
        scale = std::stoll(num) * unit_fs[ui];
      } else if (kw == "$var") {
        if (body.size() < 4) return fail_parse("malformed $var declaration", end_line);
        const std::string &width = body[1], &ident = body[2], &name = body[3];
        auto it = pi_of.find(name);
        if (it == pi_of.end()) continue;
        const int pi = it->second;
        if (width != "1") {
          R.msg = "vector variable (" + width + " bits) bound to input net " + py_repr(name);
          return VCD_SEMANTIC;
        }
        if (bound_refs[pi] > 0) continue;  // an alias of an input that is already bound
        auto old = bound.find(std::string_view(ident));
        if (old != bound.end()) {
          --bound_refs[old->second];
          old->second = pi;
        } else {
          idents.push_back(ident);
          bound.emplace(std::string_view(idents.back()), pi);
        }
        ++bound_refs[pi];
      }
      continue;
    }
    if (c == '#') {
      int64_t t = 0;
      bool ovf = false;
      if (!py_int(b + 1, e, &t, &ovf)) return fail_parse("bad time mark " + py_repr(std::string(b, e)), tl);
      if (ovf) return VCD_FALLBACK;
      if (scale < 0) return fail_parse("missing $timescale before time marks", tl);
      if (t != 0 && (t > INT64_MAX / scale || t < INT64_MIN / scale)) return VCD_FALLBACK;
      t *= scale;
      if (t < now) return fail_parse("non-monotonic time mark #" + std::string(b + 1, e), tl);
      now = t;
      if (t > duration) duration = t;
    } else if (c == '0' || c == '1' || c == 'x' || c == 'X' || c == 'z' || c == 'Z') {
      auto it = bound.find(std::string_view(b + 1, (size_t)(e - b - 1)));
      if (it != bound.end()) {
        const int pi = it->second;
        const uint8_t v = c == '1' ? 1 : 0;
        const int64_t t = now > 0 ? now : 0;
        if (t <= 0) {
          initial[pi] = v;
          value[pi] = v;
        } else if (v != value[pi]) {
          auto &tv = tog[pi];
          if (!tv.empty() && tv.back() == t) tv.pop_back();  // later change at one mark wins
          else tv.push_back(t);
          value[pi] = v;
        }
      }
    } else if (c == 'b' || c == 'B' || c == 'r' || c == 'R') {
      // vector/real change: skip its identifier, the next token of this line
      const int64_t save_pos = pos, save_line = lineno;
      int64_t nl = 0;
      if (next_token(&b, &e, &nl) && nl != tl) {
        pos = save_pos;
        lineno = save_line;
      }
    }
  }
  for (int i = 0; i < P; ++i) {
    if (bound_refs[pi_of[pi_names[i]]] == 0) {
      // first unbound input in declaration order (pi_names order)
      R.msg = "VCD declares no scalar variable for input net " + py_repr(pi_names[i]);
      return VCD_SEMANTIC;
    }
  }
  // per input position, the waveform of its name (a repeated name maps every
  // position to the last one, like the name-keyed waveform map)
  R.pi_off.assign(P + 1, 0);
  R.pi_init.assign(P, 0);
  int64_t n = 0;
  for (int i = 0; i < P; ++i) {
    R.pi_off[i] = n;
    n += (int64_t)tog[pi_of[pi_names[i]]].size();
  }
  R.pi_off[P] = n;
  R.pi_times.resize(n);
  for (int i = 0; i < P; ++i) {
    const int src = pi_of[pi_names[i]];
    std::copy(tog[src].begin(), tog[src].end(), R.pi_times.begin() + R.pi_off[i]);
    R.pi_init[i] = initial[src];
  }
  R.duration = duration;
  return VCD_OK;
}

}  // namespace gsvcd
