// kernels.cuh -- sm_100a kernels of the windowed gate-level re-simulation path.
//
// Layout in HBM for one chunk of Wc cycle windows (Tc = ceil(Wc/32) tiles):
//   cnt  [N][Tc*32] u32  toggles of net n in chunk window w
//   tbase[N][Tc]    u64  index in `data` of the first toggle of (n, tile t);
//                        lane j's toggles start at tbase + sum_{i<j} cnt[i]
//   init [N][Tc]    u32  window-start value bits, bit j = window t*32+j
//   data            TS   window-relative toggle times (u32, or u64 when a
//                        window is longer than 2^32 fs)
// so the 32 windows of one (net, tile) are one contiguous run of `data`:
// a warp reading one fanin tile touches exactly the sectors holding it.
//
// Kernels
//   K1 stim_segment_csr / stim_segment_win : cut primary-input waveforms into
//      windows (reference StimulusSet.build + slice_windows, waveform.py:49-63,
//      243-265), fused with the input nets' dwell/toggle sums (dwell_sweep,
//      _kernels.py:254-295, PI rows).
//   K4 gate_eval : one warp = one gate x 32 windows (lane = window).  Per lane
//      the exact Algo. 1 event loop of sim_span (_kernels.py:54-210), with the
//      window-start value (init_values, _kernels.py:213-231), the upper bound
//      (level_ub, _kernels.py:234-251) and the dwell/toggle reduction
//      (dwell_sweep) fused in; outputs are staged in shared memory, compacted
//      with a warp scan and appended to a per-CTA region (no global atomics).
//   K6 dwell_arena : dwell_sweep over a host-provided arena (compute_stats).
//   K2 zero_delay_level : init_values seam (one level, thread per gate-window).
#pragma once
#include <cstdint>
#include <climits>
#include <cuda_runtime.h>

namespace gs {

constexpr int kWarp = 32;
constexpr int kEvalWarps = 8;               // warps per K4 CTA
constexpr int kEvalThreads = kEvalWarps * kWarp;
constexpr int kSlab = 512;                  // staged output timestamps per warp (smem)
constexpr int kMaxK = 16;                   // netlist.py:17 MAX_CELL_INPUTS
constexpr long long kInf = LLONG_MAX;

// accumulator rows (each [N] int64): per-net results of one chunk
enum AccRow { ACC_T1 = 0, ACC_TC = 1, ACC_IG = 2, ACC_ICF = 3, ACC_DISC = 4, ACC_ROWS = 5 };
// error flags
enum ErrFlag { ERR_POOL = 0, ERR_CAP = 1, ERR_NFLAGS = 4 };
// K4 modes
enum Mode { MODE_STATS = 0, MODE_COUNTERS = 1, MODE_STORE = 3 };

struct DesignDev {
  int P, G, N;
  const int *order;            // [G] level order
  const int *gate_k;           // [G]
  const int *gate_pin;         // [G] first pin
  const unsigned long long *gate_lut;  // [G] k<=6: truth bits; else word offset
  const unsigned *lut_words;   // packed truth tables of k>6 cells
  const int *pin_net;          // [sum k]
  const long long *pin_ic;     // [sum k]
  const int *pin_arc;          // [sum k] first condition row of the pin
  const long long *arc;        // [R*2] (rise, fall)
  const unsigned *arc32;       // same, 32-bit (narrow kernels; null if delays >= 2^31)
};

struct ChunkDev {
  int N, Wc, Tc, Wpad;         // nets, windows, tiles, cnt row pitch (= Tc*32)
  long long w0;                // absolute index of the chunk's first window
  const long long *bnd;        // [W+1] absolute window boundaries
  unsigned *cnt;
  unsigned long long *tbase;
  unsigned *init;
  void *data;                  // TS[]
  unsigned long long pool_base, part_words;  // per-warp regions of `data`
  unsigned long long *bump;    // [gridDim.x * kEvalWarps] words used in each region
  unsigned *work;              // per-launch work counters (dynamic item fetch)
  long long *acc;              // [ACC_ROWS][N]
  int *err;                    // [ERR_NFLAGS]
  // arena mode ([G][Wpad] by gate id)
  long long *a_cnt, *a_peak, *a_filt, *a_icf, *a_disc;
  unsigned char *a_init;
  const long long *a_off;      // store offsets into a_buf
  long long *a_buf;
  long long a_nbuf;
};

struct StimDev {
  int P;
  long long W;
  // CSR form
  const long long *pi_off, *pi_times;
  const unsigned char *pi_init;
  // windowed form ([P][W])
  const long long *buf, *offsets, *counts;
  long long nbuf;
  const unsigned char *initials;
};

struct LevelArgs {
  int lo, n;                   // gates order[lo, lo+n)
  int tpi, ntg;                // tiles per item, tile groups per gate
  int pct;
  int counter;                 // index into ChunkDev::work
};

// ---------------------------------------------------------------- helpers

__device__ __forceinline__ unsigned lane_id() { return threadIdx.x & (kWarp - 1); }

template <typename T>
__device__ __forceinline__ T warp_excl_scan(T v, T *total) {
  const unsigned lane = lane_id();
  T x = v;
#pragma unroll
  for (int o = 1; o < kWarp; o <<= 1) {
    T y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= (unsigned)o) x += y;
  }
  *total = __shfl_sync(0xffffffffu, x, kWarp - 1);
  return x - v;
}

__device__ __forceinline__ long long warp_sum(long long v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__device__ __forceinline__ unsigned lut_bit(unsigned long long lut, int k,
                                            const unsigned *__restrict__ words, unsigned idx) {
  if (k <= 6) return (unsigned)(lut >> idx) & 1u;
  return (__ldg(words + lut + (idx >> 5)) >> (idx & 31)) & 1u;
}

// first index i in [0, n) with a[i] >= x (n if none)
__device__ __forceinline__ long long lower_bound(const long long *__restrict__ a, long long n,
                                                 long long x) {
  long long lo = 0, hi = n;
  while (lo < hi) {
    long long mid = (lo + hi) >> 1;
    if (__ldg(a + mid) < x) lo = mid + 1; else hi = mid;
  }
  return lo;
}

// bump-allocate `words` (warp-uniform) in this warp's private region of the
// pool; returns the absolute index in `data` (same on all lanes) or ~0ull when
// the region is full (the chunk is then re-run with more room)
__device__ __forceinline__ unsigned long long region_alloc(const ChunkDev &C,
                                                           unsigned long long &bump,
                                                           unsigned long long region,
                                                           unsigned long long words) {
  const unsigned long long old = bump;
  if (old + words > C.part_words) {
    if (lane_id() == 0) atomicExch(C.err + ERR_POOL, 1);
    return ~0ull;
  }
  bump = old + words;
  return C.pool_base + region * C.part_words + old;
}

// warp-wide sum of five per-lane partials, added by lane 0 into acc[row][net]
__device__ __forceinline__ void acc_flush(const ChunkDev &C, int net, long long t1, long long tc,
                                          long long filt, long long icf, long long disc) {
  t1 = warp_sum(t1);
  tc = warp_sum(tc);
  filt = warp_sum(filt);
  icf = warp_sum(icf);
  disc = warp_sum(disc);
  if (lane_id() == 0) {
    unsigned long long *a = reinterpret_cast<unsigned long long *>(C.acc);
    const size_t N = (size_t)C.N;
    if (t1) atomicAdd(a + ACC_T1 * N + net, (unsigned long long)t1);
    if (tc) atomicAdd(a + ACC_TC * N + net, (unsigned long long)tc);
    if (filt) atomicAdd(a + ACC_IG * N + net, (unsigned long long)filt);
    if (icf) atomicAdd(a + ACC_ICF * N + net, (unsigned long long)icf);
    if (disc) atomicAdd(a + ACC_DISC * N + net, (unsigned long long)disc);
  }
}

// ----------------------------------------------------------------- K1 (CSR)
// One warp per (input p, group of tiles); lane = window.  cut_w is the lower
// bound of b_w in p's sorted toggles (slice_windows, waveform.py:58); the
// window holds toggles [cut_w, cut_{w+1}) and starts at init ^ (cut_w & 1)
// (waveform.py:61).  Toggles land in `data` at their CSR index, so the tile
// base is pi_off[p] + cut of lane 0 and the tile is contiguous.
template <typename TS>
__global__ void __launch_bounds__(256) stim_segment_csr(StimDev S, ChunkDev C, int tpi, int ntg) {
  const unsigned lane = lane_id();
  const long long nwarps = (long long)gridDim.x * (blockDim.x / kWarp);
  const long long items = (long long)S.P * ntg;
  TS *data = reinterpret_cast<TS *>(C.data);
  for (long long it = (long long)blockIdx.x * (blockDim.x / kWarp) + threadIdx.x / kWarp;
       it < items; it += nwarps) {
    const int p = (int)(it / ntg);
    const int tg = (int)(it % ntg);
    const long long off = S.pi_off[p];
    const long long n = S.pi_off[p + 1] - off;
    const long long *seg = S.pi_times + off;
    const unsigned init = S.pi_init[p];
    long long tc = 0, t1 = 0;
    const int t_hi = min((tg + 1) * tpi, C.Tc);
    for (int t = tg * tpi; t < t_hi; ++t) {
      const int wr = t * kWarp + (int)lane;
      const bool act = wr < C.Wc;
      const long long wabs = C.w0 + wr;
      long long b_lo = 0, b_hi = 0, cut = n;
      if (act) {
        b_lo = C.bnd[wabs];
        b_hi = C.bnd[wabs + 1];
        cut = lower_bound(seg, n, b_lo);
      }
      long long nxt = __shfl_down_sync(0xffffffffu, cut, 1);
      if (act && (lane == kWarp - 1 || wr == C.Wc - 1)) nxt = lower_bound(seg, n, b_hi);
      const unsigned c = act ? (unsigned)(nxt - cut) : 0u;
      const unsigned v0 = act ? ((init ^ (unsigned)cut) & 1u) : 0u;
      const unsigned word = __ballot_sync(0xffffffffu, v0);
      const long long cut0 = __shfl_sync(0xffffffffu, cut, 0);
      if (lane == 0) {
        C.tbase[(size_t)p * C.Tc + t] = (unsigned long long)(off + cut0);
        C.init[(size_t)p * C.Tc + t] = word;
      }
      if (act) {
        C.cnt[(size_t)p * C.Wpad + wr] = c;
        TS *dst = data + off + cut;
        long long prev = 0, acc1 = 0;
        unsigned v = v0;
        for (unsigned j = 0; j < c; ++j) {
          const long long x = __ldg(seg + cut + j) - b_lo;
          dst[j] = (TS)x;
          if (v) acc1 += x - prev;
          v ^= 1u;
          prev = x;
        }
        if (v) acc1 += (b_hi - b_lo) - prev;
        t1 += acc1;
        tc += c;
      }
    }
    acc_flush(C, p, t1, tc, 0, 0, 0);
  }
}

// ------------------------------------------------------------ K1 (windowed)
// Reference-constructed StimulusSet (waveform.py:235-241): per (input, window)
// offset/count/initial are given; copy each tile into this CTA's region.
template <typename TS>
__global__ void __launch_bounds__(kEvalThreads) stim_segment_win(StimDev S, ChunkDev C, int tpi,
                                                                 int ntg) {
  const unsigned lane = lane_id();
  const int warp = threadIdx.x / kWarp;
  const unsigned long long region = (unsigned long long)blockIdx.x * kEvalWarps + warp;
  unsigned long long bump = C.bump[region];
  const long long items = (long long)S.P * ntg;
  TS *data = reinterpret_cast<TS *>(C.data);
  for (long long it = blockIdx.x + (long long)gridDim.x * warp; it < items;
       it += (long long)gridDim.x * kEvalWarps) {
    const int p = (int)(it / ntg);
    const int tg = (int)(it % ntg);
    long long tc = 0, t1 = 0;
    const int t_hi = min((tg + 1) * tpi, C.Tc);
    for (int t = tg * tpi; t < t_hi; ++t) {
      const int wr = t * kWarp + (int)lane;
      const bool act = wr < C.Wc;
      const long long wabs = C.w0 + wr;
      unsigned c = 0, v0 = 0;
      long long src = 0, b_lo = 0, b_hi = 0;
      if (act) {
        const size_t pw = (size_t)p * S.W + wabs;
        c = (unsigned)S.counts[pw];
        src = S.offsets[pw];
        v0 = S.initials[pw] & 1u;
        b_lo = C.bnd[wabs];
        b_hi = C.bnd[wabs + 1];
      }
      unsigned total;
      const unsigned ex = warp_excl_scan(c, &total);
      const unsigned long long base = total ? region_alloc(C, bump, region, total) : 0ull;
      const unsigned word = __ballot_sync(0xffffffffu, v0);
      const bool wrote = base != ~0ull;
      if (lane == 0) {
        C.tbase[(size_t)p * C.Tc + t] = wrote ? base : 0ull;
        C.init[(size_t)p * C.Tc + t] = word;
      }
      if (act) {
        C.cnt[(size_t)p * C.Wpad + wr] = wrote ? c : 0u;
        long long prev = 0, acc1 = 0;
        unsigned v = v0;
        for (unsigned j = 0; j < c; ++j) {
          const long long x = __ldg(S.buf + src + j) - b_lo;
          if (wrote) data[base + ex + j] = (TS)x;
          if (v) acc1 += x - prev;
          v ^= 1u;
          prev = x;
        }
        if (v) acc1 += (b_hi - b_lo) - prev;
        t1 += acc1;
        tc += c;
      }
    }
    acc_flush(C, p, t1, tc, 0, 0, 0);
  }
  if (lane == 0) C.bump[region] = bump;
}

// ------------------------------------------------------------------- K4
// Algo. 1 for one gate over one 32-window tile; lane = window.
//   K > 0 : fanin count fixed at compile time (fully unrolled, registers);
//   K == 0: generic k <= 16 (runtime loops).
//   TT    : time arithmetic -- unsigned (narrow: every window length plus the
//           largest interconnect and arc delay fits below 2^32-1) or long long.
// One kernel instance per (K, TT) keeps each hot loop small enough for the
// instruction cache; gates of a level are grouped by k on the host.
template <typename TT>
struct TimeTraits;
template <>
struct TimeTraits<unsigned> {
  static __device__ __forceinline__ unsigned inf() { return 0xffffffffu; }
};
template <>
struct TimeTraits<long long> {
  static __device__ __forceinline__ long long inf() { return kInf; }
};

template <typename TT>
__device__ __forceinline__ TT arc_delay(const DesignDev &D, int row, int col);
template <>
__device__ __forceinline__ unsigned arc_delay<unsigned>(const DesignDev &D, int row, int col) {
  return __ldg(D.arc32 + (size_t)row * 2 + col);
}
template <>
__device__ __forceinline__ long long arc_delay<long long>(const DesignDev &D, int row, int col) {
  return __ldg(D.arc + (size_t)row * 2 + col);
}

template <typename TS, typename TT, int MODE, int K>
__device__ __forceinline__ void eval_tile(const DesignDev &D, const ChunkDev &C, int g, int k,
                                          unsigned long long lut, const int *net,
                                          const TT *ic, const int *arc, int t, int pct,
                                          TS *slab, unsigned long long &bump,
                                          unsigned long long region, long long &acc_t1,
                                          long long &acc_tc, long long &acc_filt,
                                          long long &acc_icf, long long &acc_disc) {
  constexpr int KM = K > 0 ? K : kMaxK;
  const int kk = K > 0 ? K : k;
  const TT INF = TimeTraits<TT>::inf();
  const unsigned lane = lane_id();
  const int wr = t * kWarp + (int)lane;
  const bool act = wr < C.Wc;
  const long long wabs = C.w0 + wr;
  TS *data = reinterpret_cast<TS *>(C.data);
  long long b_lo = 0, wlen64 = 0;
  if (act) {
    b_lo = C.bnd[wabs];
    wlen64 = C.bnd[wabs + 1] - b_lo;
  }
  const TT wlen = (TT)wlen64;

  // fanin tiles: counts, bases, window-start bits (init_values + level_ub fused)
  const TS *sp[KM];
  unsigned n[KM];
  unsigned idx = 0, ub = 0;
#pragma unroll
  for (int p = 0; p < kk; ++p) {
    const int nn = net[p];
    const unsigned c = act ? __ldg(C.cnt + (size_t)nn * C.Wpad + wr) : 0u;
    const unsigned long long tb = __ldg(C.tbase + (size_t)nn * C.Tc + t);
    const unsigned iw = __ldg(C.init + (size_t)nn * C.Tc + t);
    unsigned tot;
    const unsigned ex = warp_excl_scan(c, &tot);
    sp[p] = data + tb + ex;
    n[p] = c;
    ub += c;
    idx |= ((iw >> lane) & 1u) << p;
  }
  const unsigned y0 = act ? lut_bit(lut, kk, D.lut_words, idx) : 0u;

  // output staging: smem slab when the tile's bound fits, else this warp's region
  unsigned UB;
  const unsigned ubx = warp_excl_scan(ub, &UB);
  TS *st;
  bool ok = true;
  if (UB <= (unsigned)kSlab) {
    st = slab + ubx;
  } else {
    const unsigned long long sb = region_alloc(C, bump, region, UB);
    ok = sb != ~0ull;
    st = data + (ok ? sb : 0ull) + ubx;
  }

  // ---- per-lane event loop (sim_span, _kernels.py:94-203)
  unsigned pos[KM];
  TT nxt[KM];
#pragma unroll
  for (int p = 0; p < kk; ++p) { pos[p] = 0; nxt[p] = INF; }
  unsigned need = (act && ok) ? ((1u << kk) - 1u) : 0u;
  unsigned y = y0;
  int cnt = 0, peak = 0, filt = 0, icf = 0, disc = 0;
  bool has_last = false, last_stored = false;
  TT t_last = 0;
  const int cap = (int)ub;  // peak <= #events <= sum of fanin toggles
  while (true) {
    TT tmin = INF;
#pragma unroll
    for (int p = 0; p < kk; ++p) {
      if ((need >> p) & 1u) {
        // interconnect inertial filter: drop adjacent pairs narrower than d
        const TT d = ic[p];
        unsigned q = pos[p];
        const TS *s = sp[p];
        if (d > 0) {
          while (q + 1 < n[p] && (TT)__ldg(s + q + 1) - (TT)__ldg(s + q) < d) {
            q += 2;
            ++icf;
          }
        }
        pos[p] = q;
        nxt[p] = q < n[p] ? (TT)__ldg(s + q) + d : INF;
      }
      tmin = min(tmin, nxt[p]);
    }
    if (tmin == INF) break;
    // multiple simultaneous inputs: consume every pin arriving at tmin
    unsigned sw = 0;
#pragma unroll
    for (int p = 0; p < kk; ++p) {
      if (nxt[p] == tmin) {
        pos[p] += 1;
        sw |= 1u << p;
      }
    }
    idx ^= sw;
    need = sw;
    const unsigned ny = lut_bit(lut, kk, D.lut_words, idx);
    if (ny != y) {
      // conditional SDF: max over switching arcs, rows from the post state
      const int col = ny ? 0 : 1;
      TT dly = 0;
#pragma unroll
      for (int p = 0; p < kk; ++p) {
        if ((sw >> p) & 1u) {
          const int row = (int)((idx & ((1u << p) - 1u)) | ((idx >> (p + 1)) << p));
          dly = max(dly, arc_delay<TT>(D, arc[p] + row, col));
        }
      }
      const TT t_out = tmin + dly;
      const TT thr = (TT)((unsigned long long)dly * (unsigned)pct / 100u);
      const bool have = has_last || cnt > 0;
      const TT tgt = has_last ? t_last : (cnt > 0 ? (TT)st[cnt - 1] : (TT)0);
      if (have && (t_out <= tgt || t_out - tgt < thr)) {
        // inertial rejection: the pulse is cancelled in full
        if (has_last) {
          if (!last_stored) --disc;
          has_last = false;
        } else {
          --cnt;
        }
        ++filt;
      } else {
        if (has_last && last_stored) {
          if (cnt < cap) st[cnt] = (TS)t_last; else atomicExch(C.err + ERR_CAP, 1);
          ++cnt;
          peak = max(peak, cnt);
        }
        if (t_out < wlen) {
          last_stored = true;
        } else {
          ++disc;  // lands at or past the window end
          last_stored = false;
        }
        has_last = true;
        t_last = t_out;
      }
      y = ny;
    }
  }
  if (has_last && last_stored) {
    if (cnt < cap) st[cnt] = (TS)t_last; else atomicExch(C.err + ERR_CAP, 1);
    ++cnt;
    peak = max(peak, cnt);
  }
  if (!(act && ok)) cnt = peak = 0;

  // ---- compaction: warp scan of counts, one region allocation per tile;
  // the copy out of the staging area also yields the dwell at 1 (dwell_sweep)
  unsigned CNT;
  const unsigned cx = warp_excl_scan((unsigned)cnt, &CNT);
  const unsigned long long ob = CNT ? region_alloc(C, bump, region, CNT) : 0ull;
  const bool wrote = ob != ~0ull;  // else the chunk is re-run; keep readers in bounds
  const unsigned word = __ballot_sync(0xffffffffu, y0);
  const int gnet = D.P + g;
  if (lane == 0) {
    C.tbase[(size_t)gnet * C.Tc + t] = wrote ? ob : 0ull;
    C.init[(size_t)gnet * C.Tc + t] = word;
  }
  if (act) {
    C.cnt[(size_t)gnet * C.Wpad + wr] = wrote ? (unsigned)cnt : 0u;
    TS *dst = data + (wrote ? ob + cx : 0ull);
    unsigned v = y0;
    long long prev = 0, t1 = 0;
    for (int j = 0; j < cnt; ++j) {
      const TS x = st[j];
      if (wrote) dst[j] = x;
      if (v) t1 += (long long)x - prev;
      v ^= 1u;
      prev = (long long)x;
    }
    if (v) t1 += wlen64 - prev;
    acc_t1 += t1;
    acc_tc += cnt;
    acc_filt += filt;
    acc_icf += icf;
    acc_disc += disc;
    if (MODE & MODE_COUNTERS) {
      const size_t gw = (size_t)g * C.Wpad + wr;
      C.a_cnt[gw] = cnt;
      C.a_peak[gw] = peak;
      C.a_filt[gw] = filt;
      C.a_icf[gw] = icf;
      C.a_disc[gw] = disc;
      C.a_init[gw] = (unsigned char)y0;
    }
    if ((MODE & MODE_STORE) == MODE_STORE) {
      // store pass: the (g, w) region of the reference arena layout receives
      // every slot the lane ever wrote, [0, peak) (waveform.py:340-345)
      const long long o = C.a_off[(size_t)g * C.Wpad + wr];
      if (o >= 0 && o + peak <= C.a_nbuf) {
        for (int j = 0; j < peak; ++j) C.a_buf[o + j] = (long long)st[j] + b_lo;
      } else if (peak) {
        atomicExch(C.err + ERR_CAP, 1);
      }
    }
  }
  __syncwarp();
}

// One launch per (logic level, fanin-count group); the level barrier is the
// launch boundary.  Persistent grid with dynamic work fetching: each warp takes
// the next item (gate, group of tpi tiles) from a per-launch counter, and owns
// a private output region (no CTA barrier, no global atomics on the data path).
template <typename TS, typename TT, int MODE, int K>
__global__ void __launch_bounds__(kEvalThreads) gate_eval(DesignDev D, ChunkDev C, LevelArgs A) {
  constexpr int KM = K > 0 ? K : kMaxK;
  __shared__ TS s_slab[kEvalWarps][kSlab];
  const int warp = threadIdx.x / kWarp;
  const unsigned lane = lane_id();
  const unsigned long long region = (unsigned long long)blockIdx.x * kEvalWarps + warp;
  unsigned long long bump = C.bump[region];
  const long long items = (long long)A.n * A.ntg;
  TS *slab = s_slab[warp];
  while (true) {
    long long it = 0;
    if (lane == 0) it = (long long)atomicAdd(C.work + A.counter, 1u);
    it = __shfl_sync(0xffffffffu, it, 0);
    if (it >= items) break;
    const int j = (int)(it / A.ntg);
    const int tg = (int)(it % A.ntg);
    const int g = __ldg(D.order + A.lo + j);
    const int k = K > 0 ? K : __ldg(D.gate_k + g);
    const int pin0 = __ldg(D.gate_pin + g);
    const unsigned long long lut = __ldg(D.gate_lut + g);
    const int t_lo = tg * A.tpi;
    const int t_hi = min(t_lo + A.tpi, C.Tc);
    int net[KM], arc[KM];
    TT ic[KM];
#pragma unroll
    for (int p = 0; p < (K > 0 ? K : k); ++p) {
      net[p] = __ldg(D.pin_net + pin0 + p);
      ic[p] = (TT)__ldg(D.pin_ic + pin0 + p);
      arc[p] = __ldg(D.pin_arc + pin0 + p);
    }
    long long t1 = 0, tc = 0, filt = 0, icf = 0, disc = 0;
    for (int t = t_lo; t < t_hi; ++t)
      eval_tile<TS, TT, MODE, K>(D, C, g, k, lut, net, ic, arc, t, A.pct, slab, bump, region,
                                 t1, tc, filt, icf, disc);
    acc_flush(C, D.P + g, t1, tc, filt, icf, disc);
  }
  if (lane == 0) C.bump[region] = bump;
}

// chunk accumulators -> run accumulators [t1 | tc | ig | filtered, icf, disc]
__global__ void acc_commit(const long long *__restrict__ acc, long long *__restrict__ out, int N) {
  __shared__ unsigned long long part[3];
  if (threadIdx.x < 3) part[threadIdx.x] = 0;
  __syncthreads();
  unsigned long long f = 0, ic = 0, di = 0;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < N;
       i += (long long)gridDim.x * blockDim.x) {
    out[i] += acc[ACC_T1 * (size_t)N + i];
    out[N + i] += acc[ACC_TC * (size_t)N + i];
    const long long ig = acc[ACC_IG * (size_t)N + i];
    out[2 * (size_t)N + i] += ig;
    f += (unsigned long long)ig;
    ic += (unsigned long long)acc[ACC_ICF * (size_t)N + i];
    di += (unsigned long long)acc[ACC_DISC * (size_t)N + i];
  }
  for (int o = 16; o > 0; o >>= 1) {
    f += __shfl_xor_sync(0xffffffffu, f, o);
    ic += __shfl_xor_sync(0xffffffffu, ic, o);
    di += __shfl_xor_sync(0xffffffffu, di, o);
  }
  if (lane_id() == 0) {
    atomicAdd(&part[0], f);
    atomicAdd(&part[1], ic);
    atomicAdd(&part[2], di);
  }
  __syncthreads();
  if (threadIdx.x < 3 && part[threadIdx.x])
    atomicAdd(reinterpret_cast<unsigned long long *>(out + 3 * (size_t)N + threadIdx.x),
              part[threadIdx.x]);
}

// ------------------------------------------------------------------- K6
// dwell_sweep (_kernels.py:254-295) over explicit arena arrays: warp per
// (net, 32 windows); lane = window.
struct DwellArgs {
  int N, P;
  const unsigned char *net_kind;
  const long long *net_slot;
  const long long *sbuf, *soff, *scnt;
  const unsigned char *sinit;
  long long sW;  // stimulus row pitch (windows)
  const long long *gbuf, *goff, *gcnt;
  const unsigned char *ginit;
  long long gW;  // arena row pitch
  const long long *bnd;
  long long w_lo, w_hi, w_off;
  long long *t0, *t1, *tc;
};

__global__ void dwell_arena(DwellArgs A) {
  const unsigned lane = lane_id();
  const long long nwarps = (long long)gridDim.x * (blockDim.x / kWarp);
  const long long Wn = A.w_hi - A.w_lo;
  const long long tiles = (Wn + kWarp - 1) / kWarp;
  for (long long it = (long long)blockIdx.x * (blockDim.x / kWarp) + threadIdx.x / kWarp;
       it < (long long)A.N * tiles; it += nwarps) {
    const int n = (int)(it / tiles);
    const long long w = A.w_lo + (it % tiles) * kWarp + lane;
    long long a0 = 0, a1 = 0, c = 0;
    if (w < A.w_hi) {
      const long long s = A.net_slot[n];
      const long long *buf;
      long long off;
      unsigned v;
      if (A.net_kind[n] == 0) {
        off = A.soff[s * A.sW + w];
        c = A.scnt[s * A.sW + w];
        v = A.sinit[s * A.sW + w];
        buf = A.sbuf;
      } else {
        const long long j = s * A.gW + (w - A.w_off);
        off = A.goff[j];
        c = A.gcnt[j];
        v = A.ginit[j];
        buf = A.gbuf;
      }
      long long prev = A.bnd[w];
      for (long long i = 0; i < c; ++i) {
        const long long x = buf[off + i];
        if (v) a1 += x - prev; else a0 += x - prev;
        v ^= 1u;
        prev = x;
      }
      const long long e = A.bnd[w + 1];
      if (v) a1 += e - prev; else a0 += e - prev;
    }
    a0 = warp_sum(a0);
    a1 = warp_sum(a1);
    c = warp_sum(c);
    if (lane == 0) {
      atomicAdd(reinterpret_cast<unsigned long long *>(A.t0 + n), (unsigned long long)a0);
      atomicAdd(reinterpret_cast<unsigned long long *>(A.t1 + n), (unsigned long long)a1);
      atomicAdd(reinterpret_cast<unsigned long long *>(A.tc + n), (unsigned long long)c);
    }
  }
}

// ------------------------------------------------------------------- K2
// init_values (_kernels.py:213-231) for one level: vals[out][w] = lut[idx].
__global__ void zero_delay_level(DesignDev D, unsigned char *vals, long long W, int lo, int n) {
  const long long total = (long long)n * W;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < total;
       i += (long long)gridDim.x * blockDim.x) {
    const int g = D.order[lo + (int)(i / W)];
    const long long w = i % W;
    const int k = D.gate_k[g], p0 = D.gate_pin[g];
    unsigned idx = 0;
    for (int p = 0; p < k; ++p) idx |= (unsigned)(vals[(size_t)D.pin_net[p0 + p] * W + w] & 1u) << p;
    vals[(size_t)(D.P + g) * W + w] = (unsigned char)lut_bit(D.gate_lut[g], k, D.lut_words, idx);
  }
}

}  // namespace gs
