// kernels_lean.cuh -- K4 gate_eval for the hot instances: fanin count K = 1..4
// and 32-bit window-relative time (every window length plus the largest
// interconnect and arc delay stays below 2^32 - 1).  Same chunk layout and
// same results as the generic kernel in kernels.cuh; built around what the
// benchmark activities look like (0.2 - 1.7 fanin toggles and
// 0.2 - 0.8 output toggles per gate-window), where most windows of a gate see
// no input transition at all or exactly one.
//
// One CTA = one gate x a super-tile of 4 consecutive 128-window tiles; warp i
// owns tile i of it and lane l windows 4l .. 4l+3 of that tile.
//   (A) per warp: per pin the tile's count row (prefetched by cp.async
//       during the previous tile) and warp scans (two pins per scan) -> the
//       lane's window offsets in the pin's segment; the window-start input
//       vectors by a 4x4 bit transpose; the pins' segments staged into the
//       warp's shared-memory slab by one TMA bulk copy (cp.async.bulk,
//       completion on an mbarrier) per pin, each issued by its own lane and
//       overlapped with the classification.  Windows with no input
//       transition keep their window-start value and are finished by the
//       lane that owns them; the others go to the CTA's worklists by class
//       (one, two, three or more transitions), positioned by one warp scan
//       of the lane's packed class counts and one shared-memory atomic;
//   (M) the whole CTA works the pooled lists of its 4 tiles, so the few busy
//       windows of each tile fill whole warps: three or more transitions
//       through sim_span's event loop with its lazy interconnect filter
//       (the loop windows take the first warps), two in closed form (the
//       interconnect pair filter of a same-pin pair, _kernels.py:96-117,
//       included) and one as a single Algo. 1 step (_kernels.py:94-203, one
//       iteration) -- these two dealt over the warps without loop windows,
//       so the warps reach the barrier together;
//   (C) per warp: warp scan of the output counts, one pool allocation, the
//       outputs copied out of the staging area; per-net dwell / toggle /
//       filter sums.
// Tiles whose fanin toggles do not fit the slab read their segments in place
// (generic pointers) and stage outputs in the pool; all their active windows
// then go through (M)'s event loop.
#pragma once
#include "kernels.cuh"

namespace gs {

#ifndef GS_LEAN_WARPS
#define GS_LEAN_WARPS 4   // warps per CTA (dev A/B knob)
#endif
// CTAs per SM each fixed-K instance is built for (launch bounds), given as
// the count of 4-warp CTAs
#ifndef GS_LEAN_CTAS2
#define GS_LEAN_CTAS2 8   // CTAs per SM of the k <= 2 instances (dev A/B knob)
#endif
#ifndef GS_LEAN_CTAS3
#define GS_LEAN_CTAS3 7   // CTAs per SM of the k = 3 instances (dev A/B knob)
#endif
#ifndef GS_LEAN_CTAS4
#define GS_LEAN_CTAS4 6   // CTAs per SM of the k = 4 instances (dev A/B knob)
#endif
template <int K>
__host__ __device__ constexpr int lean_ctas() {
  return (K <= 2 ? GS_LEAN_CTAS2 : K == 3 ? GS_LEAN_CTAS3 : GS_LEAN_CTAS4) * 4 / GS_LEAN_WARPS;
}

constexpr int kLeanWarps = GS_LEAN_WARPS;
constexpr int kLeanThreads = kLeanWarps * kWarp;
constexpr int kSuper = kLeanWarps;         // tiles per CTA step (one per warp)
constexpr int kPool = kSuper * kTile;      // windows per CTA step

// per-warp part: staged segments and tile state
template <int K, int SLAB>
struct alignas(16) LeanWarp {
  unsigned slab[SLAB];                       // staged fanin segments, then outputs
  // the next tile's fanin count rows, start-bit words and tile bases,
  // prefetched (cp.async) while the current tile is evaluated
  alignas(16) unsigned pcnt[K][kTile];
  alignas(16) unsigned pinit[K][4];
  alignas(16) unsigned long long ptb[K];
  alignas(16) unsigned offs[K][kTile + 4];   // pin p: window w's toggles start at offs[p][w]
  alignas(16) unsigned cnt[kTile];           // stored toggles per window
  unsigned long long tb[K];                  // in place: pin p's tile base in `data`
  unsigned long long stage;                  // generic address of the output staging area
  unsigned stage_at;                         // ... its slab offset (staged statistics runs)
  unsigned seg[K];                           // staged: pin p's segment at slab[seg[p]]
  int t;                                     // tile index
  int in_smem;
  unsigned long long mbar;                   // bulk-copy completion
};

// worklist classes of a window (by its input transitions); list c occupies
// [kListAt[c], kListAt[c] + kPool) of LeanShared::list
enum LeanClass : unsigned { kQuiet = 0, kSingle = 1, kTwo = 2, kLoop = 3 };
constexpr unsigned kListBits = 10;                 // per-class field of a packed count
constexpr unsigned kListMask = (1u << kListBits) - 1u;

template <int K>
struct LeanShared {
  // worklists of a step, one region of kPool entries per class: loop
  // windows at 0, two-transition windows at kPool, single-transition windows
  // at 2 kPool; then one sink slot per thread for the stores of windows that
  // need no list
  unsigned short list[3 * kPool + kLeanThreads];
  unsigned arcs[K * (1 << (K - 1)) * 2];
  unsigned ic[K];                            // the gate's interconnect delays, by pin
  unsigned dtab[K <= 2 ? (1 << (2 * K)) * 2 : K * (1 << K) * 2];
  unsigned nlist[2];                         // packed list lengths (single | two << 10 |
                                             // loop << 20), double-buffered by step parity
  unsigned item;
};

// staged words per warp that the occupancy leaves in 228 KB of shared memory
// (1 KB per CTA reserved)
template <int K>
__host__ __device__ constexpr int lean_slab_words() {
  return (int)(((233472 / lean_ctas<K>() - 1024 - sizeof(LeanShared<K>) - 64) / kLeanWarps -
                sizeof(LeanWarp<K, 4>) + 16) / 16 * 4);
}

template <int K>
struct alignas(16) LeanSmem {
  LeanWarp<K, lean_slab_words<K>()> w[kLeanWarps];
  LeanShared<K> s;
};

template <int K>
constexpr size_t lean_smem_bytes() {
  return sizeof(LeanSmem<K>);
}

// ---------------------------------------------------------------- TMA bulk
__device__ __forceinline__ unsigned smem_addr(const void *p) {
  return (unsigned)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(unsigned long long *bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count)
               : "memory");
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long *bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long *bar, unsigned parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_addr(bar)),
      "r"(parity)
      : "memory");
}
// global -> shared bulk copy (16-byte aligned, multiple of 16 bytes)
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, unsigned bytes,
                                         unsigned long long *bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_addr(dst)),
      "l"(src), "r"(bytes), "r"(smem_addr(bar))
      : "memory");
}
__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// delay of a single switching pin p (post-transition inputs idx, edge col)
template <int K>
__device__ __forceinline__ unsigned dtab_pin(const unsigned *dtab, unsigned p, unsigned idx,
                                             unsigned col) {
  if constexpr (K <= 2) return dtab[((((1u << p) << K) | idx) << 1) | col];
  else return dtab[(((p << K) | idx) << 1) | col];
}

struct LeanAcc {
  long long t1 = 0, tc = 0;
  unsigned filt = 0, icf = 0;
  int disc = 0;
};

// condition tables of one gate -> smem: arcs[(p << (K-1) | row) * 2 + col],
// then the delay table of the event step: k <= 2 by (switching pin set,
// post-transition inputs, edge) -- the max over the switching arcs of the
// conditioned delay (K:139-151); k = 3, 4 by (single pin, inputs, edge),
// simultaneous pins taking the max of their entries.  One warp builds it.
template <int K>
__device__ __forceinline__ void build_dtab(unsigned *arcs, unsigned *dtab,
                                           const unsigned *__restrict__ arc32,
                                           const int (&arc)[K]) {
  constexpr int R = 1 << (K - 1);
  const int lane = (int)lane_id();
  for (int i = lane; i < K * R * 2; i += kWarp) {
    const int pp = i / (2 * R), rc = i % (2 * R);
    int a = arc[0];
#pragma unroll
    for (int q = 1; q < K; ++q) a = pp == q ? arc[q] : a;
    arcs[i] = __ldg(arc32 + (size_t)a * 2 + rc);
  }
  __syncwarp();
  // condition row of pin pp: the other pins' values (pp's own bit removed)
  auto row_of = [](unsigned id, unsigned pp) {
    return (id & ((1u << pp) - 1u)) | ((id >> (pp + 1)) << pp);
  };
  if constexpr (K <= 2) {
    for (int i = lane; i < (1 << (2 * K)) * 2; i += kWarp) {
      const unsigned col = i & 1, id = (i >> 1) & ((1u << K) - 1), sw = (unsigned)i >> (K + 1);
      unsigned dmax = 0;
      for (unsigned pp = 0; pp < (unsigned)K; ++pp)
        if ((sw >> pp) & 1u) dmax = max(dmax, arcs[((pp * R) + row_of(id, pp)) * 2 + col]);
      dtab[i] = dmax;
    }
  } else {
    for (int i = lane; i < K * (1 << K) * 2; i += kWarp) {
      const unsigned col = i & 1, id = (i >> 1) & ((1u << K) - 1), pp = (unsigned)i >> (K + 1);
      dtab[i] = arcs[((pp * R) + row_of(id, pp)) * 2 + col];
    }
  }
}

// ---------------------------------------------------- worklist windows
// A worklist entry: window (7 bits) | start input vector (4) | warp (2).
__device__ __forceinline__ unsigned short wl_entry(int w, unsigned ix, int warp) {
  return (unsigned short)((unsigned)w | (ix << 7) | ((unsigned)warp << 11));
}

// the sources of a tile's fanin segments: the slab (SMEM, shared-memory
// addressing) or the segments in place
template <bool SMEM, int K, int SLAB>
__device__ __forceinline__ void tile_sources(const ChunkDev &C, LeanWarp<K, SLAB> &T,
                                             const unsigned *(&src)[K]) {
  unsigned *data = reinterpret_cast<unsigned *>(C.data);
#pragma unroll
  for (int p = 0; p < K; ++p) src[p] = SMEM ? &T.slab[T.seg[p]] : data + T.tb[p];
}
// a tile's output staging area (the slab for staged statistics runs)
template <bool SMEM, int MODE, int K, int SLAB>
__device__ __forceinline__ unsigned *tile_stage(LeanWarp<K, SLAB> &T) {
  if (SMEM && MODE == MODE_STATS) return &T.slab[T.stage_at];
  return reinterpret_cast<unsigned *>(T.stage);
}

// cp.async of tile t's fanin count rows (a 16-byte piece per lane), the
// tile's start-bit words (16 bytes) and tile bases (8 bytes) into the
// warp's prefetch buffers; completed by cp.async.wait_all + __syncwarp.
template <int K, int SLAB>
__device__ __forceinline__ void prefetch_tile(const ChunkDev &C, const int (&net)[K], int t,
                                              LeanWarp<K, SLAB> &T, unsigned lane) {
  const int Tw = C.Wpad / 32;
#pragma unroll
  for (int p = 0; p < K; ++p)
    __pipeline_memcpy_async(&T.pcnt[p][lane * kWPL],
                            C.cnt + (size_t)net[p] * C.Wpad + (size_t)t * kTile + lane * kWPL, 16);
  if (lane < (unsigned)K) {
    int n = net[0];
#pragma unroll
    for (int p = 1; p < K; ++p) n = lane == (unsigned)p ? net[p] : n;
    __pipeline_memcpy_async(&T.ptb[lane], C.tbase + (size_t)n * C.Tc + t, 8);
    __pipeline_memcpy_async(&T.pinit[lane][0], C.init + (size_t)n * Tw + (size_t)t * (kTile / 32),
                            16);
  }
  __pipeline_commit();
}

// sim_span's event loop (_kernels.py:94-203) over one window with three or
// more input transitions, the interconnect pair filter applied lazily as
// sim_span's refresh does (_kernels.py:96-117).  Outputs go to the tile's
// staging area at the window's slot.
template <int MODE, int K, bool PCT100, bool SMEM, int SLAB>
__device__ __forceinline__ void loop_window(const ChunkDev &C, int g, unsigned lut,
                                            const unsigned (&ic)[K], int pct,
                                            const unsigned *dtab, LeanWarp<K, SLAB> &T, int w,
                                            unsigned idx, LeanAcc &acc) {
  constexpr unsigned INF = 0xffffffffu;
  // staged: cursors are absolute slab indices (one base for every pin);
  // in place: per-pin segment pointers and relative cursors
  const unsigned *src[K];
  tile_sources<SMEM, K, SLAB>(C, T, src);
  auto at = [&](int p, unsigned q) -> unsigned { return SMEM ? T.slab[q] : src[p][q]; };
  unsigned *stage = tile_stage<SMEM, MODE, K, SLAB>(T);
  const int base_w = T.t * kTile;
  unsigned cur[K], end[K], nxt[K], so = 0;
  int icf = 0;
  auto refresh = [&](int p) {
    unsigned q = cur[p];
    const unsigned d = ic[p];
    if constexpr (SMEM) {  // unconditional slab loads, as in the event loop
      unsigned t0 = T.slab[q], t1 = T.slab[q + 1];
      if (d > 0) {
        bool narrow = q + 1 < end[p] && t1 - t0 < d;
        while (narrow) {
          q += 2;
          ++icf;
          t0 = T.slab[q];
          t1 = T.slab[q + 1];
          narrow = q + 1 < end[p] && t1 - t0 < d;
        }
        cur[p] = q;
      }
      nxt[p] = q < end[p] ? t0 + d : INF;
    } else {
      if (d > 0) {
        while (q + 1 < end[p] && at(p, q + 1) - at(p, q) < d) {
          q += 2;
          ++icf;
        }
        cur[p] = q;
      }
      nxt[p] = q < end[p] ? at(p, q) + d : INF;
    }
  };
#pragma unroll
  for (int p = 0; p < K; ++p) {
    const unsigned a = T.offs[p][w];
    const unsigned b0 = SMEM ? T.seg[p] : 0u;
    cur[p] = b0 + a;
    end[p] = b0 + T.offs[p][w + 1];
    so += a;
    refresh(p);
  }
  const unsigned y0 = (unsigned)(lut >> idx) & 1u;
  const unsigned wlen = __ldg(C.wlen32 + base_w + w);
  unsigned y = y0, t_last = 0, t_stored = 0, dt = 0, t1w = 0, dv = y0;
  int cnt = 0, peak = 0, filt = 0, disc = 0;
  bool has_last = false, last_stored = false;
  while (true) {
    unsigned tmin = nxt[0];
#pragma unroll
    for (int p = 1; p < K; ++p) tmin = min(tmin, nxt[p]);
    if (tmin == INF) break;
    // every pin arriving at tmin switches (MSI), then advances
    unsigned sw = 0;
#pragma unroll
    for (int p = 0; p < K; ++p) sw |= (nxt[p] == tmin ? 1u : 0u) << p;
    idx ^= sw;
    // the switching pins advance: predicated per pin (no divergent branch);
    // only a narrow pair (rare) enters the filter loop
    auto advance_pins = [&]() {
#pragma unroll
      for (int p = 0; p < K; ++p) {
        const bool adv = (sw >> p) & 1u;
        unsigned q = cur[p] + (adv ? 1u : 0u);
        const unsigned d = ic[p];
        if constexpr (SMEM) {
          // staged: both candidate toggles loaded unconditionally (a cursor at
          // most two words past the segment still reads inside the warp's
          // shared-memory slice), so no pin takes a divergent branch
          unsigned t0 = T.slab[q], t1 = T.slab[q + 1];
          if (d > 0) {  // the gate's pin: uniform across the CTA
            bool narrow = adv && q + 1 < end[p] && t1 - t0 < d;
            while (narrow) {
              q += 2;
              ++icf;
              t0 = T.slab[q];
              t1 = T.slab[q + 1];
              narrow = q + 1 < end[p] && t1 - t0 < d;
            }
          }
          cur[p] = q;
          nxt[p] = adv ? (q < end[p] ? t0 + d : INF) : nxt[p];
        } else {
          if (d > 0) {
            bool narrow = adv && q + 1 < end[p] && at(p, q + 1) - at(p, q) < d;
            while (narrow) {
              q += 2;
              ++icf;
              narrow = q + 1 < end[p] && at(p, q + 1) - at(p, q) < d;
            }
          }
          cur[p] = q;
          const unsigned v = adv && q < end[p] ? at(p, q) + d : INF;
          nxt[p] = adv ? v : nxt[p];
        }
      }
    };
    if constexpr (SMEM && K >= 3) {
      // one switching pin (the common case): its cursor fetched by selects,
      // advanced once, written back -- instead of K predicated advances
      if ((sw & (sw - 1u)) == 0u) {
        const unsigned ps = (unsigned)__ffs(sw) - 1u;
        unsigned q = cur[0], e = end[0], d = ic[0];
#pragma unroll
        for (int k = 1; k < K; ++k) {
          q = ps == (unsigned)k ? cur[k] : q;
          e = ps == (unsigned)k ? end[k] : e;
          d = ps == (unsigned)k ? ic[k] : d;
        }
        q += 1;
        unsigned t0 = T.slab[q], t1 = T.slab[q + 1];
        bool narrow = d > 0 && q + 1 < e && t1 - t0 < d;
        while (narrow) {
          q += 2;
          ++icf;
          t0 = T.slab[q];
          t1 = T.slab[q + 1];
          narrow = q + 1 < e && t1 - t0 < d;
        }
        const unsigned nv = q < e ? t0 + d : INF;
#pragma unroll
        for (int k = 0; k < K; ++k) {
          cur[k] = ps == (unsigned)k ? q : cur[k];
          nxt[k] = ps == (unsigned)k ? nv : nxt[k];
        }
      } else {
        advance_pins();
      }
    } else {
      advance_pins();
    }
    // output side (K:136-193)
    const unsigned ny = (unsigned)(lut >> idx) & 1u;
    const bool chg = ny != y;
    const unsigned dly = dtab_delay<K>(dtab, sw, idx, ny ? 0 : 1);
    const unsigned t_out = tmin + dly;
    const unsigned thr = PCT100 ? dly : (unsigned)((unsigned long long)dly * (unsigned)pct / 100u);
    bool cancel;
    if constexpr (PCT100) {
      // only the pending edge can be cancelled at 100 %: stored edges are final
      cancel = chg && has_last && (t_out <= t_last || t_out - t_last < thr);
    } else {
      const bool have = has_last || cnt > 0;
      const unsigned tgt = has_last ? t_last : t_stored;
      cancel = chg && have && (t_out <= tgt || t_out - tgt < thr);
    }
    const bool emit = chg && !cancel;
    const bool pop = !PCT100 && cancel && !has_last;
    disc -= (cancel && has_last && !last_stored) ? 1 : 0;
    if (!PCT100) {
      cnt -= pop ? 1 : 0;
      if (pop && cnt > 0) t_stored = stage[so + cnt - 1];
    }
    filt += cancel ? 1 : 0;
    const bool store = emit && has_last && last_stored;
    if (store) stage[so + cnt] = t_last;
    if (!PCT100) t_stored = store ? t_last : t_stored;
    cnt += store ? 1 : 0;
    if (MODE != MODE_STATS) peak = max(peak, cnt);
    t1w += (store && dv) ? t_last - dt : 0u;
    dv ^= store ? 1u : 0u;
    dt = store ? t_last : dt;
    const bool inwin = t_out < wlen;
    disc += (emit && !inwin) ? 1 : 0;
    last_stored = emit ? inwin : last_stored;
    t_last = emit ? t_out : t_last;
    has_last = emit || (has_last && !cancel);
    y = chg ? ny : y;
  }
  if (has_last && last_stored) {
    stage[so + cnt] = t_last;
    ++cnt;
    peak = max(peak, cnt);
    t1w += dv ? t_last - dt : 0u;
    dv ^= 1u;
    dt = t_last;
  }
  if (PCT100) {
    acc.t1 += (long long)(t1w + (dv ? wlen - dt : 0u));
  } else {
    // below 100 % stored edges may be popped: the dwell comes from the final
    // stored waveform (dwell_sweep, _kernels.py:254-295)
    unsigned v = y0, prev = 0;
    long long a1 = 0;
    for (int q = 0; q < cnt; ++q) {
      const unsigned x = stage[so + q];
      if (v) a1 += x - prev;
      v ^= 1u;
      prev = x;
    }
    if (v) a1 += wlen - prev;
    acc.t1 += a1;
  }
  T.cnt[w] = (unsigned)cnt;
  acc.filt += (unsigned)filt;
  acc.icf += (unsigned)icf;
  acc.disc += disc;
  record_arena<MODE, unsigned>(C, g, base_w + w, cnt, peak, filt, icf, disc, y0,
                               [&](int j) -> unsigned & { return stage[so + j]; },
                               (unsigned long long)(stage + so - reinterpret_cast<unsigned *>(C.data)));
}

// One input transition: Algo. 1 with a single event (K:94-203, one
// iteration) -- one LUT lookup, one delay lookup, one window-end test.  Only
// staged tiles classify windows as single.
template <int MODE, int K, bool PCT100, int SLAB>
__device__ __forceinline__ void single_window(const ChunkDev &C, int g, unsigned lut,
                                              const unsigned (&ic)[K], const unsigned *ic_of,
                                              const unsigned *dtab,
                                              LeanWarp<K, SLAB> &T, int w, unsigned i0,
                                              LeanAcc &acc) {
  unsigned *stage = tile_stage<true, MODE, K, SLAB>(T);
  const int base_w = T.t * kTile;
  // the one toggling pin: its bit in the mask of pins with a toggle
  unsigned so = 0, mask = 0;
#pragma unroll
  for (int p = 0; p < K; ++p) {
    const unsigned a = T.offs[p][w];
    so += a;
    if (K > 1) mask |= (T.offs[p][w + 1] != a ? 1u : 0u) << p;
  }
  const unsigned pj = K > 1 ? (unsigned)__ffs(mask) - 1u : 0u;
  const unsigned icp = K > 1 ? ic_of[pj] : ic[0];
  const unsigned tv = T.slab[T.seg[pj] + T.offs[pj][w]];
  const unsigned y0 = (unsigned)(lut >> i0) & 1u;
  const unsigned i1 = i0 ^ (1u << pj);
  const unsigned y1 = (unsigned)(lut >> i1) & 1u;
  const bool chg = y1 != y0;
  const unsigned ot = tv + icp + dtab_pin<K>(dtab, pj, i1, y1 ? 0u : 1u);
  const unsigned wln = __ldg(C.wlen32 + base_w + w);
  const bool inwin = ot < wln;
  const bool st = chg && inwin;
  if (st) stage[so] = ot;
  const int disc = (chg && !inwin) ? 1 : 0;
  acc.disc += disc;
  // dwell at 1: the start value holds until the stored edge (or the window
  // end), the other value after it
  const unsigned e = st ? ot : wln;
  acc.t1 += y0 ? e : wln - e;
  T.cnt[w] = st ? 1u : 0u;
  if (MODE != MODE_STATS)
    record_arena<MODE, unsigned>(C, g, base_w + w, st ? 1 : 0, st ? 1 : 0, 0, 0, disc, y0,
                                 [&](int) -> unsigned & { return stage[so]; },
                                 (unsigned long long)(stage + so - reinterpret_cast<unsigned *>(C.data)));
}

// Two input transitions in closed form.  With no edge pending at the first
// event, Algo. 1's output side (K:136-203) collapses to selects: event 1 (both
// pins when the two transitions coincide) can only emit; event 2 can emit,
// cancel event 1's edge, or leave it pending; no stored edge can be popped.
template <int MODE, int K, bool PCT100, int SLAB>
__device__ __forceinline__ void two_window(const ChunkDev &C, int g, unsigned lut,
                                           const unsigned (&ic)[K], const unsigned *ic_of,
                                           int pct, const unsigned *dtab, LeanWarp<K, SLAB> &T,
                                           int w, unsigned i0, LeanAcc &acc) {
  // two-transition windows come from staged tiles
  unsigned *stage = tile_stage<true, MODE, K, SLAB>(T);
  const int base_w = T.t * kTile;
  // the toggling pins: both toggles on one pin (dbl), or the two lowest pins
  // of the mask of pins with a toggle
  unsigned so = 0, mask = 0, dbl = 0;
#pragma unroll
  for (int p = 0; p < K; ++p) {
    const unsigned a = T.offs[p][w], m = T.offs[p][w + 1] - a;
    so += a;
    mask |= (m != 0 ? 1u : 0u) << p;
    dbl |= (m >= 2 ? 1u : 0u) << p;
  }
  unsigned pa = (unsigned)__ffs(dbl ? dbl : mask) - 1u;
  unsigned pb = dbl ? pa : (unsigned)__ffs(mask & (mask - 1u)) - 1u;
  if (K == 1) pa = pb = 0;
  const unsigned xa = T.seg[pa] + T.offs[pa][w];
  const unsigned xb = dbl ? xa + 1u : T.seg[pb] + T.offs[pb][w];
  const unsigned ica = K > 1 ? ic_of[pa] : ic[0], icb = K > 1 ? ic_of[pb] : ic[0];
  const unsigned va = T.slab[xa], vb = T.slab[xb];
  // a same-pin pair narrower than the pin's interconnect delay is filtered
  // out whole (_kernels.py:96-117): no event remains
  const bool pairf = pa == pb && ica > 0 && vb - va < ica;
  unsigned ta = va + ica, tb2 = vb + icb;
  const bool sw2 = tb2 < ta;
  { const unsigned tt = sw2 ? tb2 : ta; tb2 = sw2 ? ta : tb2; ta = tt; }
  { const unsigned pp = sw2 ? pb : pa; pb = sw2 ? pa : pb; pa = pp; }
  const bool both = ta == tb2 && pa != pb;  // two pins at one instant: one event
  const bool n1 = !pairf, n2 = !pairf && !both;
  const unsigned s1 = (1u << pa) | (both ? (1u << pb) : 0u), s2 = 1u << pb;
  const unsigned i1 = i0 ^ (n1 ? s1 : 0u), i2 = i1 ^ (n2 ? s2 : 0u);
  const unsigned yy0 = (unsigned)(lut >> i0) & 1u;
  const unsigned y1 = (unsigned)(lut >> i1) & 1u;
  const unsigned y2 = (unsigned)(lut >> i2) & 1u;
  const bool c1 = y1 != yy0, c2 = y2 != y1;
  const unsigned d2 = dtab_delay<K>(dtab, s2, i2, y2 ? 0 : 1);
  const unsigned o1 = ta + dtab_delay<K>(dtab, s1, i1, y1 ? 0 : 1);
  const unsigned o2 = tb2 + d2;
  const unsigned thr = PCT100 ? d2 : (unsigned)((unsigned long long)d2 * (unsigned)pct / 100u);
  const unsigned wlw = __ldg(C.wlen32 + base_w + w);
  const bool x2 = c2 && c1 && (o2 <= o1 || o2 - o1 < thr);   // edge 1 cancelled
  const bool e2 = c2 && !x2;                                 // edge 2 emitted
  const bool in1 = o1 < wlw, in2 = o2 < wlw;
  const bool st1 = e2 && c1 && in1;                          // edge 1 stored at event 2
  const unsigned tp = e2 ? o2 : o1;                          // pending at the end
  const bool fl = e2 ? in2 : (c1 && !x2 && in1);             // ... and flushed
  const unsigned cnt = (st1 ? 1u : 0u) + (fl ? 1u : 0u);
  const unsigned f0 = st1 ? o1 : tp;
  unsigned *st = stage + so;
  if (cnt >= 1) st[0] = f0;
  if (cnt == 2) st[1] = tp;
  const int disc = (c1 && !in1 ? 1 : 0) + (e2 && !in2 ? 1 : 0) - (x2 && !in1 ? 1 : 0);
  // dwell at 1: +-edge times by the value before each edge, plus the window
  // end when the final value is 1 (wrapping arithmetic, exact since the
  // result lies in [0, wlen])
  const unsigned e0 = cnt >= 1 ? f0 : 0u, e1 = cnt == 2 ? tp : 0u;
  const unsigned wf = (cnt & 1u) ? (yy0 ? 0u : wlw) : (yy0 ? wlw : 0u);
  acc.t1 += (long long)(yy0 ? e0 - e1 + wf : e1 - e0 + wf);
  T.cnt[w] = cnt;
  acc.filt += x2 ? 1u : 0u;
  acc.icf += pairf ? 1u : 0u;
  acc.disc += disc;
  if (MODE != MODE_STATS)
    record_arena<MODE, unsigned>(C, g, base_w + w, (int)cnt, (int)cnt, x2 ? 1 : 0,
                                 pairf ? 1 : 0, disc, yy0,
                                 [&](int q) -> unsigned & { return st[q]; },
                                 (unsigned long long)(st - reinterpret_cast<unsigned *>(C.data)));
}

// ------------------------------------------------------------------ kernel
// One launch per (logic level, fanin-count group), as gate_eval: persistent
// grid; work items (gate, run of super-tiles) fetched by the CTA from a
// per-launch counter in super-tile-group-major order (the CTAs in flight share
// fanin tiles while they are in L2), head items of tpi super-tiles then tail
// items of tpi2.
template <int MODE, int K, bool PCT100>
__global__ void __launch_bounds__(kLeanThreads, lean_ctas<K>())
gate_eval_lean(DesignDev D, ChunkDev C, LevelArgs A) {
  constexpr int SLAB = lean_slab_words<K>();
  using SM = LeanSmem<K>;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  SM &S = *reinterpret_cast<SM *>(smem_raw);
  // the thread index through a shuffle, so that register allocation keeps it
  // (and the warp's slice of shared memory derived from it) in registers
  // instead of re-reading the special register at every use
  const int tid = (int)__shfl_sync(0xffffffffu, threadIdx.x, threadIdx.x & (kWarp - 1));
  const int warp = tid / kWarp;
  const unsigned lane = (unsigned)tid & (kWarp - 1);
  LeanWarp<K, SLAB> &T = S.w[warp];
  Region R = region_open(C, (unsigned long long)blockIdx.x * kLeanWarps + warp);
  if (lane == 0) mbar_init(&T.mbar, 1);
  if (tid < 2) S.s.nlist[tid] = 0;
  unsigned phase = 0, par = 0;
  unsigned *data = reinterpret_cast<unsigned *>(C.data);
  const int Tw = C.Wpad / 32;
  const int STc = (C.Tc + kSuper - 1) / kSuper;
  const unsigned head = (unsigned)A.n * (unsigned)A.ntg;
  const unsigned items = head + (unsigned)A.n * (unsigned)A.ntg2;
  while (true) {
    if (tid == 0) S.s.item = atomicAdd(C.work + A.counter, 1u);
    __syncthreads();
    const unsigned it = S.s.item;
    if (it >= items) break;
    const bool in_head = it < head;
    const unsigned iq = in_head ? it : it - head;
    const int jg = (int)(iq % (unsigned)A.n);
    const int tg = (int)(iq / (unsigned)A.n);
    const int g = __ldg(D.order + A.lo + jg);
    const int gnet = D.P + g;
    const int pin0 = __ldg(D.gate_pin + g);
    // the truth table of a k <= 4 cell fits 16 bits: 32-bit shifts
    const unsigned lut = (unsigned)__ldg(D.gate_lut + g);
    const int u_lo = in_head ? tg * A.tpi : A.ntg * A.tpi + tg * A.tpi2;
    const int u_hi = min(u_lo + (in_head ? A.tpi : A.tpi2), STc);
    int net[K], arc[K];
    unsigned ic[K];
#pragma unroll
    for (int p = 0; p < K; ++p) {
      net[p] = __ldg(D.pin_net + pin0 + p);
      ic[p] = (unsigned)__ldg(D.pin_ic + pin0 + p);
      arc[p] = __ldg(D.pin_arc + pin0 + p);
    }
    if (warp == 0) build_dtab<K>(S.s.arcs, S.s.dtab, D.arc32, arc);
    if (tid < K) {
      unsigned v = ic[0];
#pragma unroll
      for (int p = 1; p < K; ++p) v = tid == p ? ic[p] : v;
      S.s.ic[tid] = v;
    }
    __syncthreads();
    LeanAcc acc;
    const int t_end = min(u_hi * kSuper, C.Tc);
    if (u_lo * kSuper + warp < t_end) prefetch_tile<K, SLAB>(C, net, u_lo * kSuper + warp, T, lane);
    for (int t0 = u_lo * kSuper; t0 < t_end; t0 += kSuper, par ^= 1u) {
      const int t = t0 + warp;
      const bool tile = t < t_end;
      const int base_w = t * kTile;
      const int nact = tile ? min(kTile, C.Wc - base_w) : 0;
      const int wl = (int)lane * kWPL;
      unsigned nib = 0;
      bool ok = true;
      // ---- (A) this warp's tile
      GS_PROF_T(pt0);
      if (tile) {
        GS_PROF_ADD(PF_TILES, 1);
        unsigned c[K][kWPL];
        unsigned long long tb[K];
        unsigned bits[K];
        __pipeline_wait_prior(0);
        __syncwarp();
#pragma unroll
        for (int p = 0; p < K; ++p) {
          ld4(&T.pcnt[p][wl], c[p]);
          tb[p] = T.ptb[p];
          bits[p] = (T.pinit[p][(lane * kWPL) / 32] >> ((lane * kWPL) % 32)) & ((1u << kWPL) - 1u);
        }
        __syncwarp();
        // the next tile of this warp in the item: its rows fly during this one
        if (t + kSuper < t_end) prefetch_tile<K, SLAB>(C, net, t + kSuper, T, lane);
        // window-start input vectors: the (pin x window) bit matrix transposed
        unsigned n[kWPL], ix[kWPL];
        {
          unsigned B = 0;
#pragma unroll
          for (int p = 0; p < K; ++p) B |= bits[p] << (4 * p);
          if (K > 1) {
            unsigned x = (B ^ (B >> 3)) & 0x0A0Au;
            B ^= x ^ (x << 3);
            x = (B ^ (B >> 6)) & 0x00CCu;
            B ^= x ^ (x << 6);
          }
#pragma unroll
          for (int j = 0; j < kWPL; ++j) {
            ix[j] = K > 1 ? (B >> (4 * j)) & 15u : (B >> j) & 1u;
            n[j] = 0;
          }
        }
        // per-pin window offsets: warp scans of the lane sums, two pins per
        // scan (16-bit halves) unless some lane's sum could overflow a half
        unsigned s4[K], ex0[K], tot[K];
#pragma unroll
        for (int p = 0; p < K; ++p) {
          s4[p] = 0;
#pragma unroll
          for (int j = 0; j < kWPL; ++j) s4[p] += c[p][j];
        }
        bool pair = false;
        if constexpr (K > 1) {
          unsigned big = 0;
#pragma unroll
          for (int p = 0; p < K; ++p) big |= s4[p];
          pair = !__any_sync(0xffffffffu, big >= 2048u);
        }
        if (pair) {
#pragma unroll
          for (int p = 0; p + 1 < K; p += 2) {
            unsigned t2;
            const unsigned e = warp_excl_scan(s4[p] | (s4[p + 1] << 16), &t2);
            ex0[p] = e & 0xFFFFu;
            ex0[p + 1] = e >> 16;
            tot[p] = t2 & 0xFFFFu;
            tot[p + 1] = t2 >> 16;
          }
          if (K & 1) ex0[K - 1] = warp_excl_scan(s4[K - 1], &tot[K - 1]);
        } else {
#pragma unroll
          for (int p = 0; p < K; ++p) ex0[p] = warp_excl_scan(s4[p], &tot[p]);
        }
        unsigned seg[K], inw = 0, UB = 0;
#pragma unroll
        for (int p = 0; p < K; ++p) {
          unsigned ex = ex0[p];
          const unsigned sh = (unsigned)tb[p] & 3u;
          seg[p] = inw + sh;
          inw += tot[p] ? (sh + tot[p] + 3u) & ~3u : 0u;
          UB += tot[p];
          unsigned o4[kWPL];
#pragma unroll
          for (int j = 0; j < kWPL; ++j) {
            o4[j] = ex;
            n[j] += c[p][j];
            ex += c[p][j];
          }
          st4(&T.offs[p][wl], o4);
          if (lane == kWarp - 1) T.offs[p][kTile] = tot[p];
        }
        // inputs (aligned per pin) and outputs (UB words) in the slab, or both
        // in global memory
        const bool in_smem = inw + UB <= (unsigned)SLAB;
        unsigned *stage;
        if (in_smem) {
          if (inw && lane < (unsigned)K) {
            // lane p issues pin p's copy (the mbarrier's transaction count
            // may run ahead of lane 0's expect, PTX: -(2^20-1) .. 2^20-1)
            unsigned tp = tot[0], sp = seg[0];
            unsigned long long bp = tb[0];
#pragma unroll
            for (int p = 1; p < K; ++p) {
              tp = lane == (unsigned)p ? tot[p] : tp;
              sp = lane == (unsigned)p ? seg[p] : sp;
              bp = lane == (unsigned)p ? tb[p] : bp;
            }
            fence_proxy_async();  // the slab's earlier generic accesses before the async writes
            if (lane == 0) mbar_expect_tx(&T.mbar, inw * 4u);
            if (tp) {
              const unsigned sh = (unsigned)bp & 3u;
              bulk_g2s(&T.slab[sp - sh], data + (bp - sh), ((sh + tp + 3u) & ~3u) * 4u, &T.mbar);
            }
          }
          // staged statistics runs address the slab by offset (stage_at);
          // no generic pointer is formed
          stage = nullptr;
          if (MODE != MODE_STATS) {
            // arena runs: outputs stay in the pool until the chunk's arena is
            // packed (K5)
            const unsigned long long sb = region_alloc(C, R, UB);
            ok = sb != ~0ull;
            stage = data + (ok ? sb : 0ull);
          }
        } else {
          const unsigned long long sb = region_alloc(C, R, UB);
          ok = sb != ~0ull;
          stage = data + (ok ? sb : 0ull);
        }
        if (lane == 0) {
          T.in_smem = in_smem ? 1 : 0;
          T.t = t;
          T.stage = reinterpret_cast<unsigned long long>(stage);
          T.stage_at = inw;
#pragma unroll
          for (int p = 0; p < K; ++p) {
            T.seg[p] = seg[p];
            T.tb[p] = tb[p];
          }
        }
        // worklists by class: staged tiles send windows with one, two, or
        // three and more transitions to the single / two / loop lists; tiles
        // read in place send every window with a transition to the loop list.
        // Positions: one warp scan of the lane's packed class counts, one
        // shared-memory atomic for all three lists of the warp.
        // the lane's windows inside the chunk: j < nv
        const int nv = ok ? min(max(nact - wl, 0), kWPL) : 0;
        unsigned cls[kWPL], V = 0;
        const unsigned mul = in_smem ? 1u : 3u;  // in place: every active window loops
#pragma unroll
        for (int j = 0; j < kWPL; ++j) {
          const bool a = j < nv;
          const unsigned m = min(n[j] * mul, 3u);
          cls[j] = a ? m : 0u;
          V += (1u << (kListBits * cls[j])) >> kListBits;
        }
        unsigned VT;
        unsigned P = warp_excl_scan(V, &VT);
        // lane 0's shared-memory atomic as a predicated instruction (no
        // branch); the other lanes' result register is never read
        unsigned base;
        asm volatile(
            "{\n\t.reg .pred p;\n\tsetp.eq.u32 p, %1, 0;\n\t"
            "@p atom.shared.add.u32 %0, [%2], %3;\n\t}"
            : "=r"(base)
            : "r"(lane), "r"(smem_addr(&S.s.nlist[par])), "r"(VT)
            : "memory");
        P += __shfl_sync(0xffffffffu, base, 0);
        // every window stores (no branch): quiet ones into the thread's sink slot
        unsigned short *lists = S.s.list;
        const unsigned sink = 3 * kPool + (unsigned)tid;
#pragma unroll
        for (int j = 0; j < kWPL; ++j) {
          const unsigned c1 = cls[j] ? cls[j] - 1u : 0u;
          const unsigned at = cls[j] ? (2u - c1) * kPool + ((P >> (kListBits * c1)) & kListMask)
                                     : sink;
          lists[at] = wl_entry(wl + j, ix[j], warp);
          P += (1u << (kListBits * cls[j])) >> kListBits;
        }
        // the staged segments have landed (all lanes observe the barrier)
        if (in_smem && inw) {
          mbar_wait(&T.mbar, phase);
          phase ^= 1u;
        }
        // windows with no transition: the output keeps its start value
        unsigned wl4[kWPL];
        load_counts(C.wlen32 + base_w + wl, wl4);
#pragma unroll
        for (int j = 0; j < kWPL; ++j) {
          const bool act = j < nv;
          const unsigned y0 = (unsigned)(lut >> ix[j]) & 1u;
          const bool quiet = act && n[j] == 0;
          acc.t1 += (quiet && y0) ? wl4[j] : 0u;
          nib |= (act ? y0 : 0u) << j;
          if (MODE != MODE_STATS && quiet)
            record_arena<MODE, unsigned>(C, g, base_w + wl + j, 0, 0, 0, 0, 0, y0,
                                         [&](int) -> unsigned & { return stage[0]; },
                                         (unsigned long long)(stage - data));
        }
        // counts of the quiet windows (list windows overwrite theirs)
        const unsigned z4[kWPL] = {0u, 0u, 0u, 0u};
        st4(&T.cnt[wl], z4);
      }
      GS_PROF_T(pt1);
      GS_PROF_ADD(PF_PHASE1, pt1 - pt0);
      __syncthreads();
      // ---- (M) the pooled worklists of the CTA's tiles: loop windows first
      // (the longest), then two-transition, then single-transition windows,
      // each list starting on a warp boundary
      {
        const unsigned pk = S.s.nlist[par];
        if (tid == 0) S.s.nlist[par ^ 1u] = 0;  // the next step's lists
        const unsigned nS = pk & kListMask, nT = (pk >> kListBits) & kListMask,
                       nL = pk >> (2 * kListBits);
        const unsigned aL = (nL + kWarp - 1) & ~(unsigned)(kWarp - 1);
        const unsigned aT = aL + ((nT + kWarp - 1) & ~(unsigned)(kWarp - 1));
        GS_PROF_ADD(PF_LOOP_WINDOWS, warp == 0 ? nL : 0);
        GS_PROF_ADD(PF_TRIVIAL, warp == 0 ? nT : 0);
        // loop windows: one per thread from warp 0 up (the whole CTA round
        // robin when there are more than its threads); two- and single-
        // transition windows (one index space, the singles after the
        // warp-aligned twos) dealt round robin over the warps left without
        // loop windows, so the long event loops and the short windows finish
        // together at the barrier
        const unsigned ut = (unsigned)tid;
        for (unsigned i = ut; i < nL; i += kLeanThreads) {
          const unsigned e = S.s.list[i];
          LeanWarp<K, SLAB> &Tw = S.w[e >> 11];
          if (Tw.in_smem)
            loop_window<MODE, K, PCT100, true, SLAB>(C, g, lut, ic, A.pct, S.s.dtab, Tw,
                                                     (int)(e & 127u), (e >> 7) & 15u, acc);
          else
            loop_window<MODE, K, PCT100, false, SLAB>(C, g, lut, ic, A.pct, S.s.dtab, Tw,
                                                      (int)(e & 127u), (e >> 7) & 15u, acc);
        }
        const unsigned loop_warps = aL / kWarp;
        const bool spare = loop_warps < (unsigned)kLeanWarps;
        const unsigned first = spare ? loop_warps * kWarp : 0u;  // first thread of the deal
        const unsigned nth = kLeanThreads - first;
        const unsigned aT2 = (nT + kWarp - 1) & ~(unsigned)(kWarp - 1);
        if (ut >= first) {
          for (unsigned i = ut - first; i < aT2 + nS; i += nth) {
            if (i < aT2) {
              if (i < nT) {
                const unsigned e = S.s.list[kPool + i];
                two_window<MODE, K, PCT100, SLAB>(C, g, lut, ic, S.s.ic, A.pct, S.s.dtab,
                                                  S.w[e >> 11], (int)(e & 127u), (e >> 7) & 15u,
                                                  acc);
              }
            } else {
              const unsigned e = S.s.list[2 * kPool + i - aT2];
              single_window<MODE, K, PCT100, SLAB>(C, g, lut, ic, S.s.ic, S.s.dtab, S.w[e >> 11],
                                                   (int)(e & 127u), (e >> 7) & 15u, acc);
            }
          }
        }
      }
      GS_PROF_T(pt2);
      GS_PROF_ADD(PF_LOOP, pt2 - pt1);
      __syncthreads();
      // ---- (C) compaction of this warp's tile and the per-net sums
      if (tile) {
        unsigned co[kWPL], so[kWPL], s = 0;
        const unsigned amask = (1u << (ok ? min(max(nact - wl, 0), kWPL) : 0)) - 1u;
        ld4(&T.cnt[wl], co);
        ld4(&T.offs[0][wl], so);
#pragma unroll
        for (int p = 1; p < K; ++p) {
          unsigned o4[kWPL];
          ld4(&T.offs[p][wl], o4);
#pragma unroll
          for (int j = 0; j < kWPL; ++j) so[j] += o4[j];
        }
#pragma unroll
        for (int j = 0; j < kWPL; ++j) {
          co[j] = (amask >> j) & 1u ? co[j] : 0u;
          s += co[j];
        }
        unsigned CNT;
        const unsigned cx = warp_excl_scan(s, &CNT);
        const unsigned long long ob = CNT ? region_alloc(C, R, CNT) : 0ull;
        const bool wrote = ob != ~0ull;  // else the chunk is re-run; keep readers in bounds
        // up to two outputs per window as predicated copies; the rare windows
        // with more take a loop.  Staged statistics tiles read the slab with
        // shared-memory addressing, the others the generic staging pointer.
        auto copy_out = [&](const unsigned *stage) {
          // the lane's outputs as one flat run: output q of the lane comes
          // from window j (the last with cum[j] <= q) at so[j] + q - cum[j]
          unsigned *dst = data + ob + cx;
          const unsigned c1 = co[0], c2 = c1 + co[1], c3 = c2 + co[2];
          const unsigned d0 = so[0], d1 = so[1] - c1, d2 = so[2] - c2, d3 = so[3] - c3;
#pragma unroll 2
          for (unsigned q = 0; q < s; ++q) {
            const unsigned d = q >= c3 ? d3 : q >= c2 ? d2 : q >= c1 ? d1 : d0;
            dst[q] = stage[d + q];
          }
        };
        if (wrote) {
          if (MODE == MODE_STATS && T.in_smem)
            copy_out(&T.slab[T.stage_at]);
          else
            copy_out(reinterpret_cast<const unsigned *>(T.stage));
        }
        acc.tc += s;
        if (lane == 0) C.tbase[(size_t)gnet * C.Tc + t] = wrote ? ob : 0ull;
        store_counts(C.cnt + (size_t)gnet * C.Wpad + base_w + wl, co, wrote);
        store_init_words(C.init + (size_t)gnet * Tw, t, nib);
      }
      GS_PROF_T(pt3);
      GS_PROF_ADD(PF_PHASE3, pt3 - pt2);
    }
    acc_flush(C, gnet, acc.t1, acc.tc, (long long)acc.filt, (long long)acc.icf,
              (long long)acc.disc);
  }
  region_close(C, R);
}

}  // namespace gs
