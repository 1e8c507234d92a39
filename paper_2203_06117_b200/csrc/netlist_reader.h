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

struct Result {
  std::string name;
  std::vector<std::string> pis, pos, gates;
  std::vector<int64_t> gate_cell;   // [G] index into the cell list
  std::vector<int64_t> pin_off;     // [G+1]
  std::vector<int64_t> pin_net;     // [sum k], cell pin order
  std::vector<std::string> out_names;  // [G] output net names
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
  bool skip() { Value v; ws(); return skip_value(0); }

 private:
  const char *p_, *end_;
  // syntax check of one value without building it
  bool skip_value(int depth) {
    if (depth > 200 || p_ >= end_) return false;
    const char c = *p_;
    if (c == '"') { std::string t; return str(t); }
    if (c == '{' || c == '[') {
      const char close = c == '{' ? '}' : ']';
      ++p_;
      ws();
      if (p_ < end_ && *p_ == close) { ++p_; return true; }
      while (true) {
        ws();
        if (c == '{') {
          std::string k;
          if (p_ >= end_ || *p_ != '"' || !str(k)) return false;
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
// false: the document is outside the reader's scope (the caller's reader
// then produces the reference's result or error).  Two passes: the top-level
// object is scanned for the (last) "name", "inputs", "outputs" and "gates"
// values; then the gates array is streamed one entry at a time.
inline bool read(const char *text, size_t len, const std::vector<Cell> &cells, Result &R) {
  Parser top(text, len);
  const char *at[4] = {nullptr, nullptr, nullptr, nullptr};  // name, inputs, outputs, gates
  static const char *const keys[4] = {"name", "inputs", "outputs", "gates"};
  if (!top.eat('{')) return false;
  if (!top.eat('}')) {
    while (true) {
      std::string k;
      if (!top.key(k) || !top.eat(':')) return false;
      top.eat(' ');  // (whitespace is skipped by the next call anyway)
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
  auto parse_at = [&](const char *p, Value &v) {
    Parser q(p, (size_t)(text + len - p));
    return q.one(v);
  };
  Value name, ins, outs;
  if (!at[0] || !parse_at(at[0], name) || name.kind != Value::STR || name.s.empty()) return false;
  R.name = name.s;
  auto str_list = [&](const char *p, std::vector<std::string> &out, Value &tmp) {
    if (!p) return true;  // absent: empty
    if (!parse_at(p, tmp) || tmp.kind != Value::ARR) return false;
    for (auto &x : tmp.arr) {
      if (x.kind != Value::STR) return false;
      out.push_back(std::move(x.s));
    }
    return true;
  };
  if (!str_list(at[1], R.pis, ins) || !str_list(at[2], R.pos, outs)) return false;

  std::unordered_map<std::string, int64_t> cell_ix, net_ix;
  for (size_t c = 0; c < cells.size(); ++c) cell_ix.emplace(cells[c].name, (int64_t)c);
  int64_t nets = 0;
  for (const auto &pi : R.pis)
    if (!net_ix.emplace(pi, nets++).second) return false;  // two drivers
  std::unordered_map<std::string, char> seen;
  std::vector<std::string> pending;  // pin nets not yet driven when read
  R.pin_off.assign(1, 0);
  if (at[3]) {
    Parser gp(at[3], (size_t)(text + len - at[3]));
    if (!gp.eat('[')) return false;
    if (!gp.eat(']')) {
      while (true) {
        Value e;
        if (!gp.one(e) || e.kind != Value::OBJ) return false;
        const Value *gn = e.get("name"), *cn = e.get("cell"), *pins = e.get("pins");
        if (!gn || gn->kind != Value::STR || gn->s.empty()) return false;
        if (!seen.emplace(gn->s, 1).second) return false;  // duplicate gate name
        if (!cn || cn->kind != Value::STR) return false;
        auto ci = cell_ix.find(cn->s);
        if (ci == cell_ix.end()) return false;
        if (!pins || pins->kind != Value::OBJ) return false;
        const Cell &cell = cells[ci->second];
        for (const auto &kv : pins->obj) {
          if (kv.second.kind != Value::STR) return false;
          bool legal = kv.first == cell.out;
          for (const auto &p : cell.pins) legal |= kv.first == p;
          if (!legal) return false;
        }
        const Value *ov = pins->get(cell.out);
        if (!ov) return false;
        for (const auto &p : cell.pins) {
          const Value *src = pins->get(p);
          if (!src) return false;
          auto it = net_ix.find(src->s);
          if (it != net_ix.end()) {
            R.pin_net.push_back(it->second);
          } else {  // resolved once every output is claimed
            R.pin_net.push_back(-1 - (int64_t)pending.size());
            pending.push_back(src->s);
          }
        }
        if (!net_ix.emplace(ov->s, nets++).second) return false;  // two drivers
        R.pin_off.push_back((int64_t)R.pin_net.size());
        R.gates.push_back(gn->s);
        R.gate_cell.push_back(ci->second);
        R.out_names.push_back(ov->s);
        if (gp.eat(',')) continue;
        if (gp.eat(']')) break;
        return false;
      }
    }
  }
  for (auto &x : R.pin_net)
    if (x < 0) {
      auto it = net_ix.find(pending[-1 - x]);
      if (it == net_ix.end()) return false;  // undriven input
      x = it->second;
    }
  for (const auto &po : R.pos)
    if (net_ix.find(po) == net_ix.end()) return false;
  return true;
}

}  // namespace gsnl
