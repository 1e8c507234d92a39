// netlist_reader.h -- the netlist JSON document (reference parse_netlist,
// pkg/src/glsim/netlist.py:190-275) read straight into flat arrays, the
// format immediately upstream of the design upload:
// no per-gate objects, so a 10M-gate netlist reads in seconds.
//
// Scope: a document the reference accepts.  Anything the reference would
// reject -- malformed JSON, a missing or mistyped field, an unknown cell or
// pin, a net with two drivers or none -- makes the reader answer
// "unsupported" and the caller runs its own reader, which raises the
// reference's exact error.  JSON semantics follow Python's json module:
// duplicate object keys keep the last value, NaN / Infinity are accepted as
// values (and then fail any string check), strings may not hold raw control
// characters, \uXXXX escapes (surrogate pairs combined) decode to UTF-8.
//
// Nets are interned as the reference does: the inputs first, then one output
// net per gate in document order (gate i drives net P + i).
#pragma once
#include <cstdint>
#include <cstring>
#include <deque>
#include <string>
#include <string_view>
#include <unordered_map>
#include <vector>

namespace gsnl {

struct Cell {
  std::string name;
  std::vector<std::string> pins;  // input pins, in order
  std::string out;
};

// a list of names as one byte blob with [n+1] offsets
struct Names {
  std::string blob;
  std::vector<int64_t> off{0};
  void add(std::string_view s) {
    blob.append(s.data(), s.size());
    off.push_back((int64_t)blob.size());
  }
  size_t size() const { return off.size() - 1; }
};

struct Result {
  std::string name;
  Names pis, pos, gates, outs;      // outs: gate output net names
  std::vector<int64_t> gate_cell;   // [G] index into the cell list
  std::vector<int64_t> pin_off;     // [G+1]
  std::vector<int64_t> pin_net;     // [sum k], cell pin order
};

// ---------------------------------------------------------------- JSON
struct Value;
using Object = std::vector<std::pair<std::string, Value>>;
struct Value {
  enum Kind { NUL, BOOL, NUM, STR, ARR, OBJ } kind = NUL;
  std::string s;
  std::vector<Value> arr;
  Object obj;
  // last value of `key` (Python dict semantics), or null
  const Value *get(std::string_view key) const {
    const Value *v = nullptr;
    for (const auto &kv : obj)
      if (kv.first == key) v = &kv.second;
    return v;
  }
};

class Parser {
 public:
  Parser(const char *p, size_t n) : p_(p), end_(p + n) {}
  bool parse(Value &out) {
    ws();
    if (!value(out, 0)) return false;
    ws();
    return p_ == end_;
  }
  // cursor interface for streaming a large document
  const char *pos() const { return p_; }
  bool at_end() { ws(); return p_ == end_; }
  bool eat(char c) {
    ws();
    if (p_ < end_ && *p_ == c) { ++p_; return true; }
    return false;
  }
  bool key(std::string &k) {
    ws();
    return p_ < end_ && *p_ == '"' && str(k);
  }
  bool one(Value &v) { ws(); return value(v, 0); }
  bool skip() { ws(); return skip_value(0); }
  // a string value as a view into the text when it has no escapes, else
  // decoded into `arena` (stable storage); false if not a valid string
  bool fstr(std::string_view &out, std::deque<std::string> &arena) {
    ws();
    if (p_ >= end_ || *p_ != '"') return false;
    const char *b = p_ + 1, *q = b;
    while (q < end_ && *q != '"' && *q != '\\' && (unsigned char)*q >= 0x20) ++q;
    if (q < end_ && *q == '"') {
      out = std::string_view(b, (size_t)(q - b));
      p_ = q + 1;
      return true;
    }
    arena.emplace_back();
    if (!str(arena.back())) return false;
    out = arena.back();
    return true;
  }
  bool peek(char c) { ws(); return p_ < end_ && *p_ == c; }

 private:
  const char *p_, *end_;
  // syntax check of one value without building it
  bool skip_value(int depth) {
    if (depth > 200 || p_ >= end_) return false;
    const char c = *p_;
    if (c == '"') { std::string_view v; return skip_str(); }
    if (c == '{' || c == '[') {
      const char close = c == '{' ? '}' : ']';
      ++p_;
      ws();
      if (p_ < end_ && *p_ == close) { ++p_; return true; }
      while (true) {
        ws();
        if (c == '{') {
          if (p_ >= end_ || *p_ != '"' || !skip_str()) return false;
          ws();
          if (p_ >= end_ || *p_ != ':') return false;
          ++p_;
          ws();
        }
        if (!skip_value(depth + 1)) return false;
        ws();
        if (p_ < end_ && *p_ == ',') { ++p_; continue; }
        if (p_ < end_ && *p_ == close) { ++p_; return true; }
        return false;
      }
    }
    Value v;
    return value(v, depth);
  }
  void ws() {
    while (p_ < end_ && (*p_ == ' ' || *p_ == '\t' || *p_ == '\n' || *p_ == '\r')) ++p_;
  }
  // a string checked without building it (escapes validated)
  bool skip_str() {
    const char *q = p_ + 1;
    while (q < end_ && *q != '"' && *q != '\\' && (unsigned char)*q >= 0x20) ++q;
    if (q < end_ && *q == '"') {
      p_ = q + 1;
      return true;
    }
    std::string t;
    return str(t);
  }
  bool lit(const char *w) {
    const size_t n = strlen(w);
    if ((size_t)(end_ - p_) < n || memcmp(p_, w, n) != 0) return false;
    p_ += n;
    return true;
  }
  static void utf8(std::string &o, uint32_t c) {
    if (c < 0x80) {
      o.push_back((char)c);
    } else if (c < 0x800) {
      o.push_back((char)(0xC0 | (c >> 6)));
      o.push_back((char)(0x80 | (c & 0x3F)));
    } else if (c < 0x10000) {
      o.push_back((char)(0xE0 | (c >> 12)));
      o.push_back((char)(0x80 | ((c >> 6) & 0x3F)));
      o.push_back((char)(0x80 | (c & 0x3F)));
    } else {
      o.push_back((char)(0xF0 | (c >> 18)));
      o.push_back((char)(0x80 | ((c >> 12) & 0x3F)));
      o.push_back((char)(0x80 | ((c >> 6) & 0x3F)));
      o.push_back((char)(0x80 | (c & 0x3F)));
    }
  }
  bool hex4(uint32_t &v) {
    if (end_ - p_ < 4) return false;
    v = 0;
    for (int i = 0; i < 4; ++i) {
      const char c = *p_++;
      v <<= 4;
      if (c >= '0' && c <= '9') v |= (uint32_t)(c - '0');
      else if (c >= 'a' && c <= 'f') v |= (uint32_t)(c - 'a' + 10);
      else if (c >= 'A' && c <= 'F') v |= (uint32_t)(c - 'A' + 10);
      else return false;
    }
    return true;
  }
  bool str(std::string &o) {
    ++p_;  // opening quote
    while (p_ < end_) {
      const unsigned char c = (unsigned char)*p_;
      if (c == '"') {
        ++p_;
        return true;
      }
      if (c < 0x20) return false;  // strict: no raw control characters
      if (c != '\\') {
        o.push_back((char)c);
        ++p_;
        continue;
      }
      if (++p_ >= end_) return false;
      const char e = *p_++;
      switch (e) {
        case '"': o.push_back('"'); break;
        case '\\': o.push_back('\\'); break;
        case '/': o.push_back('/'); break;
        case 'b': o.push_back('\b'); break;
        case 'f': o.push_back('\f'); break;
        case 'n': o.push_back('\n'); break;
        case 'r': o.push_back('\r'); break;
        case 't': o.push_back('\t'); break;
        case 'u': {
          uint32_t v;
          if (!hex4(v)) return false;
          if (v >= 0xD800 && v < 0xDC00) {  // a surrogate pair, or not representable
            uint32_t lo;
            if (end_ - p_ < 6 || p_[0] != '\\' || p_[1] != 'u') return false;
            p_ += 2;
            if (!hex4(lo) || lo < 0xDC00 || lo >= 0xE000) return false;
            v = 0x10000 + ((v - 0xD800) << 10) + (lo - 0xDC00);
          } else if (v >= 0xDC00 && v < 0xE000) {
            return false;  // lone low surrogate
          }
          utf8(o, v);
          break;
        }
        default: return false;
      }
    }
    return false;
  }
  bool num() {
    const char *s = p_;
    if (p_ < end_ && *p_ == '-') ++p_;
    if (p_ < end_ && *p_ == 'I') return lit("Infinity");
    if (p_ >= end_ || !(*p_ >= '0' && *p_ <= '9')) return false;
    if (*p_ == '0') ++p_;
    else while (p_ < end_ && *p_ >= '0' && *p_ <= '9') ++p_;
    if (p_ < end_ && *p_ == '.') {
      ++p_;
      if (p_ >= end_ || !(*p_ >= '0' && *p_ <= '9')) return false;
      while (p_ < end_ && *p_ >= '0' && *p_ <= '9') ++p_;
    }
    if (p_ < end_ && (*p_ == 'e' || *p_ == 'E')) {
      ++p_;
      if (p_ < end_ && (*p_ == '+' || *p_ == '-')) ++p_;
      if (p_ >= end_ || !(*p_ >= '0' && *p_ <= '9')) return false;
      while (p_ < end_ && *p_ >= '0' && *p_ <= '9') ++p_;
    }
    return p_ > s;
  }
  bool value(Value &v, int depth) {
    if (depth > 200 || p_ >= end_) return false;
    const char c = *p_;
    if (c == '"') {
      v.kind = Value::STR;
      return str(v.s);
    }
    if (c == '{') {
      v.kind = Value::OBJ;
      ++p_;
      ws();
      if (p_ < end_ && *p_ == '}') {
        ++p_;
        return true;
      }
      while (true) {
        ws();
        if (p_ >= end_ || *p_ != '"') return false;
        std::pair<std::string, Value> kv;
        if (!str(kv.first)) return false;
        ws();
        if (p_ >= end_ || *p_ != ':') return false;
        ++p_;
        ws();
        if (!value(kv.second, depth + 1)) return false;
        v.obj.push_back(std::move(kv));
        ws();
        if (p_ < end_ && *p_ == ',') { ++p_; continue; }
        if (p_ < end_ && *p_ == '}') { ++p_; return true; }
        return false;
      }
    }
    if (c == '[') {
      v.kind = Value::ARR;
      ++p_;
      ws();
      if (p_ < end_ && *p_ == ']') {
        ++p_;
        return true;
      }
      while (true) {
        ws();
        v.arr.emplace_back();
        if (!value(v.arr.back(), depth + 1)) return false;
        ws();
        if (p_ < end_ && *p_ == ',') { ++p_; continue; }
        if (p_ < end_ && *p_ == ']') { ++p_; return true; }
        return false;
      }
    }
    if (c == 't') { v.kind = Value::BOOL; return lit("true"); }
    if (c == 'f') { v.kind = Value::BOOL; return lit("false"); }
    if (c == 'n') { v.kind = Value::NUL; return lit("null"); }
    if (c == 'N') { v.kind = Value::NUM; return lit("NaN"); }
    v.kind = Value::NUM;
    return num();
  }
};

// ---------------------------------------------------------------- netlist
// open-addressing string_view -> int64 map (linear probing, power-of-two
// capacity): the name tables of a multi-million-gate netlist, without a heap
// node per entry
class NameMap {
 public:
  explicit NameMap(size_t expect = 16) { grow(expect * 2); }
  // inserts (key, v) unless present; returns false if the key was present
  bool insert(std::string_view k, int64_t v) {
    if ((n_ + 1) * 4 > cap_ * 3) grow(cap_ * 2);
    size_t i = slot(k);
    if (used_[i]) return false;
    used_[i] = 1;
    keys_[i] = k;
    vals_[i] = v;
    ++n_;
    return true;
  }
  // value of k, or -1
  int64_t find(std::string_view k) const {
    const size_t i = slot(k);
    return used_[i] ? vals_[i] : -1;
  }

 private:
  std::vector<std::string_view> keys_;
  std::vector<int64_t> vals_;
  std::vector<char> used_;
  size_t cap_ = 0, n_ = 0;
  static uint64_t hash(std::string_view k) {
    uint64_t h = 1469598103934665603ull;  // FNV-1a, then a final mix
    for (unsigned char c : k) h = (h ^ c) * 1099511628211ull;
    h ^= h >> 33;
    h *= 0xff51afd7ed558ccdull;
    h ^= h >> 33;
    return h;
  }
  size_t slot(std::string_view k) const {
    size_t i = (size_t)hash(k) & (cap_ - 1);
    while (used_[i] && keys_[i] != k) i = (i + 1) & (cap_ - 1);
    return i;
  }
  void grow(size_t want) {
    size_t c = 16;
    while (c < want) c <<= 1;
    std::vector<std::string_view> ok;
    std::vector<int64_t> ov;
    for (size_t i = 0; i < cap_; ++i)
      if (used_[i]) {
        ok.push_back(keys_[i]);
        ov.push_back(vals_[i]);
      }
    cap_ = c;
    keys_.assign(c, std::string_view());
    vals_.assign(c, 0);
    used_.assign(c, 0);
    n_ = 0;
    for (size_t i = 0; i < ok.size(); ++i) {
      const size_t j = slot(ok[i]);
      used_[j] = 1;
      keys_[j] = ok[i];
      vals_[j] = ov[i];
      ++n_;
    }
  }
};

// false: the document is outside the reader's scope (the caller's reader
// then produces the reference's result or error).  Two passes: the top-level
// object is scanned for the (last) "name", "inputs", "outputs" and "gates"
// values; then the gates array is streamed one entry at a time, strings held
// as views into the text (decoded copies only where they carry escapes).
inline bool read(const char *text, size_t len, const std::vector<Cell> &cells, Result &R) {
  Parser top(text, len);
  const char *at[4] = {nullptr, nullptr, nullptr, nullptr};  // name, inputs, outputs, gates
  static const char *const keys[4] = {"name", "inputs", "outputs", "gates"};
  if (!top.eat('{')) return false;
  if (!top.eat('}')) {
    while (true) {
      std::string k;
      if (!top.key(k) || !top.eat(':')) return false;
      top.peek(' ');
      const char *v = top.pos();
      for (int i = 0; i < 4; ++i)
        if (k == keys[i]) at[i] = v;
      if (!top.skip()) return false;
      if (top.eat(',')) continue;
      if (top.eat('}')) break;
      return false;
    }
  }
  if (!top.at_end()) return false;
  std::deque<std::string> arena;  // decoded strings (escapes); views point here
  auto cursor = [&](const char *p) { return Parser(p, (size_t)(text + len - p)); };
  {
    if (!at[0]) return false;
    Parser q = cursor(at[0]);
    std::string_view nm;
    if (!q.fstr(nm, arena) || nm.empty()) return false;
    R.name.assign(nm.data(), nm.size());
  }
  auto str_list = [&](const char *p, Names &out) {
    if (!p) return true;  // absent: empty
    Parser q = cursor(p);
    if (!q.eat('[')) return false;
    if (q.eat(']')) return true;
    while (true) {
      std::string_view v;
      if (!q.fstr(v, arena)) return false;
      out.add(v);
      if (q.eat(',')) continue;
      return q.eat(']');
    }
  };
  if (!str_list(at[1], R.pis) || !str_list(at[2], R.pos)) return false;

  NameMap cell_ix(cells.size()), net_ix((size_t)(len / 48) + R.pis.size()),
      seen((size_t)(len / 96));
  for (size_t c = 0; c < cells.size(); ++c) cell_ix.insert(cells[c].name, (int64_t)c);
  int64_t nets = 0;
  for (size_t i = 0; i < R.pis.size(); ++i)
    if (!net_ix.insert(std::string_view(R.pis.blob).substr(R.pis.off[i],
                                                          R.pis.off[i + 1] - R.pis.off[i]),
                       nets++))
      return false;  // two drivers
  std::vector<std::string_view> pending;  // pin nets not yet driven when read
  R.pin_off.assign(1, 0);
  std::vector<std::pair<std::string_view, std::string_view>> pins;
  if (at[3]) {
    Parser gp = cursor(at[3]);
    if (!gp.eat('[')) return false;
    if (!gp.eat(']')) {
      while (true) {
        // one gate entry: {"name": str, "cell": str, "pins": {str: str}}
        std::string_view gn, cn;
        bool have_gn = false, have_cn = false, have_pins = false;
        if (!gp.eat('{')) return false;
        if (!gp.eat('}')) {
          while (true) {
            std::string_view k;
            if (!gp.fstr(k, arena) || !gp.eat(':')) return false;
            if (k == "name") {
              if (!gp.fstr(gn, arena)) return false;
              have_gn = true;
            } else if (k == "cell") {
              if (!gp.fstr(cn, arena)) return false;
              have_cn = true;
            } else if (k == "pins") {
              pins.clear();
              have_pins = true;
              if (!gp.eat('{')) return false;
              if (!gp.eat('}')) {
                while (true) {
                  std::string_view pk, pv;
                  if (!gp.fstr(pk, arena) || !gp.eat(':') || !gp.fstr(pv, arena)) return false;
                  pins.emplace_back(pk, pv);
                  if (gp.eat(',')) continue;
                  if (gp.eat('}')) break;
                  return false;
                }
              }
            } else if (!gp.skip()) {
              return false;
            }
            if (gp.eat(',')) continue;
            if (gp.eat('}')) break;
            return false;
          }
        }
        if (!have_gn || gn.empty() || !have_cn || !have_pins) return false;
        if (!seen.insert(gn, 1)) return false;  // duplicate gate name
        const int64_t ci = cell_ix.find(cn);
        if (ci < 0) return false;
        const Cell &cell = cells[ci];
        auto last = [&](std::string_view key) -> const std::string_view * {
          const std::string_view *v = nullptr;
          for (const auto &kv : pins)
            if (kv.first == key) v = &kv.second;
          return v;
        };
        for (const auto &kv : pins) {
          bool legal = kv.first == cell.out;
          for (const auto &p : cell.pins) legal |= kv.first == p;
          if (!legal) return false;
        }
        const std::string_view *ov = last(cell.out);
        if (!ov) return false;
        for (const auto &p : cell.pins) {
          const std::string_view *src = last(p);
          if (!src) return false;
          const int64_t nx = net_ix.find(*src);
          if (nx >= 0) {
            R.pin_net.push_back(nx);
          } else {  // resolved once every output is claimed
            R.pin_net.push_back(-1 - (int64_t)pending.size());
            pending.push_back(*src);
          }
        }
        if (!net_ix.insert(*ov, nets++)) return false;  // two drivers
        R.pin_off.push_back((int64_t)R.pin_net.size());
        R.gates.add(gn);
        R.gate_cell.push_back(ci);
        R.outs.add(*ov);
        if (gp.eat(',')) continue;
        if (gp.eat(']')) break;
        return false;
      }
    }
  }
  for (auto &x : R.pin_net)
    if (x < 0) {
      const int64_t nx = net_ix.find(pending[-1 - x]);
      if (nx < 0) return false;  // undriven input
      x = nx;
    }
  for (size_t i = 0; i < R.pos.size(); ++i)
    if (net_ix.find(std::string_view(R.pos.blob).substr(R.pos.off[i],
                                                        R.pos.off[i + 1] - R.pos.off[i])) < 0)
      return false;
  return true;
}

}  // namespace gsnl
