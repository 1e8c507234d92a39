// vcd_writer.h -- the VCD dump of simulated waveforms (reference VcdWriter /
// write_vcd, pkg/src/glsim/report.py:144-214), native: the format
// immediately downstream of the hot path.
//
// Same bytes as the reference:
//   header   $timescale 1 fs $end / $scope module <design> $end / one
//            "$var wire 1 <id> <name> $end" per listed name / $upscope $end /
//            $enddefinitions $end;  <id> = bijective base-94 code ('!'..'~')
//            of the name's LAST position in the list (a dict keyed by name);
//   feed     per listed net and window: a window-open event (time b_w) when
//            the window's start value differs from the net's last written
//            value, then one event per toggle; all events of the fed window
//            range sorted by (time, open-before-toggle, name, value), written
//            as "#<time>" on every new time and "<value><id>" per event;
//   finish   "#<end time>".
// Names compare by their UTF-8 bytes, which orders them as Python orders str.
#pragma once
#include <algorithm>
#include <charconv>
#include <cstdint>
#include <cstring>
#include <numeric>
#include <string>
#include <string_view>
#include <vector>

namespace gsvcd {

inline void id_code(int64_t i, std::string &out) {
  ++i;
  while (i) {
    const int64_t r = (i - 1) % 94;
    i = (i - 1) / 94;
    out.push_back((char)(33 + r));
  }
}

inline void put_int(std::string &out, int64_t v) {
  char tmp[24];
  auto r = std::to_chars(tmp, tmp + sizeof(tmp), v);
  out.append(tmp, r.ptr);
}

// Per listed position: the dense rank of its name among the distinct names
// (equal names share a rank), and per rank the id code of the name's last
// position.
struct NameTable {
  std::vector<int64_t> rank;     // [num_names]
  std::vector<std::string> id;   // [num_ranks]
  void build(const char *names, const int64_t *off, int64_t n) {
    std::vector<int64_t> ix(n);
    std::iota(ix.begin(), ix.end(), 0);
    auto sv = [&](int64_t i) { return std::string_view(names + off[i], (size_t)(off[i + 1] - off[i])); };
    std::stable_sort(ix.begin(), ix.end(), [&](int64_t a, int64_t b) { return sv(a) < sv(b); });
    rank.assign(n, 0);
    int64_t r = -1;
    std::vector<int64_t> last_pos;
    for (int64_t k = 0; k < n; ++k) {
      if (k == 0 || sv(ix[k]) != sv(ix[k - 1])) {
        ++r;
        last_pos.push_back(ix[k]);
      }
      rank[ix[k]] = r;
      last_pos[r] = std::max(last_pos[r], ix[k]);
    }
    id.assign(r + 1, std::string());
    for (int64_t q = 0; q <= r; ++q) id_code(last_pos[q], id[q]);
  }
};

inline void header(std::string &out, const char *names, const int64_t *off, int64_t n,
                   const NameTable &T, const char *design) {
  out += "$timescale 1 fs $end\n$scope module ";
  out += design;
  out += " $end\n";
  for (int64_t i = 0; i < n; ++i) {
    out += "$var wire 1 ";
    out += T.id[T.rank[i]];
    out.push_back(' ');
    out.append(names + off[i], (size_t)(off[i + 1] - off[i]));
    out += " $end\n";
  }
  out += "$upscope $end\n$enddefinitions $end\n";
}

// one windowed waveform source: row r, window column c -> region of `buf`
struct Source {
  const int64_t *buf, *offsets, *counts;
  const uint8_t *initials;
  int64_t cols, col0, nbuf;
};

struct Event {
  int64_t t;
  uint64_t key;  // open(0)/toggle(1) << 63 | name rank << 1 | value
  bool operator<(const Event &o) const { return t != o.t ? t < o.t : key < o.key; }
};

// Feed windows [w_lo, w_hi) of every listed net; last[rank] is the last
// written value per distinct name (-1: none yet), updated.  Returns false on a
// region outside its buffer.
inline bool feed(std::string &out, int64_t n, const uint8_t *net_src, const int64_t *net_row,
                 const Source *src, const int64_t *bounds, int64_t w_lo, int64_t w_hi,
                 const NameTable &T, std::vector<int8_t> &last) {
  std::vector<Event> ev;
  for (int64_t i = 0; i < n; ++i) {
    const Source &S = src[net_src[i] ? 1 : 0];
    const uint64_t rk = (uint64_t)T.rank[i] << 1;
    int8_t &lv = last[T.rank[i]];
    for (int64_t w = w_lo; w < w_hi; ++w) {
      const int64_t cell = net_row[i] * S.cols + (w - w_lo) + S.col0;
      const int64_t o = S.offsets[cell], c = S.counts[cell];
      if (o < 0 || c < 0 || o + c > S.nbuf) return false;
      unsigned v = S.initials[cell] & 1u;
      if (lv != (int8_t)v) ev.push_back({bounds[w], rk | v});
      for (int64_t q = 0; q < c; ++q) {
        v ^= 1u;
        ev.push_back({S.buf[o + q], (1ull << 63) | rk | v});
      }
      lv = (int8_t)v;
    }
  }
  std::sort(ev.begin(), ev.end());
  out.reserve(out.size() + ev.size() * 6);
  bool first = true;
  int64_t cur = 0;
  for (const Event &e : ev) {
    if (first || e.t != cur) {
      out.push_back('#');
      put_int(out, e.t);
      out.push_back('\n');
      cur = e.t;
      first = false;
    }
    out.push_back((char)('0' + (e.key & 1u)));
    out += T.id[(e.key & ~(1ull << 63)) >> 1];
    out.push_back('\n');
  }
  return true;
}

}  // namespace gsvcd
