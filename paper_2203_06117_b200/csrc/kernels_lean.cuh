// kernels_lean.cuh -- K4 gate_eval for the hot instances: fanin count K = 1..4
// and 32-bit window-relative time (every window length plus the largest
// interconnect and arc delay stays below 2^32 - 1).  Same chunk layout and
// same results as the generic kernel in kernels.cuh; built around what the
// benchmark activities look like (0.2 - 1.7 fanin toggles and
// 0.2 - 0.8 output toggles per gate-window), where most windows of a gate see
// no input transition at all or exactly one.
//
// One warp = one gate x one 128-window tile; lane l owns windows 4l .. 4l+3.
//   (1) per pin: the tile's count row (one 16-byte load per lane), a warp scan
//       -> the lane's window offsets in the pin's segment; the pins' segments
//       are staged into the warp's shared-memory slab by one TMA bulk copy
//       (cp.async.bulk, completion on an mbarrier) per pin, issued by one lane
//       and overlapped with the classification below;
//   (2) classification in registers: windows with no input transition (the
//       output keeps its window-start value) and with exactly one are
//       finished by the lane that owns them, in registers -- Algo. 1 with a
//       single event is one LUT lookup, one delay lookup and one window-end
//       test (_kernels.py:94-203 with one iteration);
//   (3) windows with two transitions (worklist, one window per lane): the
//       closed form of two events, with the interconnect pair filter of a
//       same-pin pair (_kernels.py:96-117);
//   (4) windows with three or more (worklist): the lockstep event loop of
//       sim_span, interconnect filter applied lazily as sim_span does;
//   (5) compaction: warp scan of the output counts, one pool allocation,
//       stores straight from registers (windows of (2)) or from the staging
//       area (windows of (3), (4)); per-net dwell / toggle / filter sums.
// Tiles whose fanin toggles do not fit the slab read their segments in place
// (generic pointers) and stage outputs in the pool; every active window then
// goes through (3) / (4).
#pragma once
#include "kernels.cuh"

namespace gs {

// CTAs of 4 warps per SM each fixed-K instance is built for (launch bounds),
// and the staged words per warp that this occupancy leaves in 228 KB of
// shared memory (1 KB per CTA reserved)
template <int K>
__host__ __device__ constexpr int lean_ctas() { return K <= 2 ? 8 : K == 3 ? 7 : 6; }

template <int K>
struct LeanFixed {
  unsigned offs[K][kTile + 4];
  unsigned cnt[kTile];
  unsigned list[kTile];
  unsigned arcs[K * (1 << (K - 1)) * 2];
  unsigned dtab[K <= 2 ? (1 << (2 * K)) * 2 : K * (1 << K) * 2];
  unsigned long long mbar;
  unsigned next;
};

template <int K>
__host__ __device__ constexpr int lean_slab_words() {
  return (int)((((233472 / lean_ctas<K>() - 1024) / kEvalWarps) - sizeof(LeanFixed<K>) - 16) / 16 * 4);
}

template <int K>
struct alignas(16) LeanSmem {
  unsigned slab[lean_slab_words<K>()];       // staged fanin segments, then multi-window outputs
  alignas(16) unsigned offs[K][kTile + 4];   // pin p: window w's toggles start at offs[p][w]
  alignas(16) unsigned cnt[kTile];           // stored toggles of the worklist windows
  unsigned list[kTile];                      // worklist: w | start input vector << 8
  // the item's condition tables and the delay table built from them
  unsigned arcs[K * (1 << (K - 1)) * 2];
  unsigned dtab[K <= 2 ? (1 << (2 * K)) * 2 : K * (1 << K) * 2];
  unsigned long long mbar;                   // bulk-copy completion
  unsigned next;                             // dynamic worklist counter (event loop)
};

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

// ------------------------------------------------------- (4) event loop
// sim_span's event loop (_kernels.py:94-203) for the worklist windows with
// three or more input transitions; a lane whose window is finished takes the
// next one from the shared counter.  Inputs come from `src` (staged or in
// place); the interconnect pair filter runs lazily exactly as sim_span's
// refresh (_kernels.py:96-117).
template <int MODE, int K, bool PCT100>
__device__ __forceinline__ void lean_loop(const ChunkDev &C, int g, unsigned long long lut,
                                          const unsigned (&ic)[K], int pct, LeanSmem<K> &S,
                                          const unsigned *const (&src)[K], unsigned *stage,
                                          int base_w, unsigned nwork, LeanAcc &acc) {
  constexpr unsigned INF = 0xffffffffu;
  unsigned cur[K], end[K], nxt[K];
  unsigned idx = 0, y = 0, y0 = 0, so = 0, wlen = 0, t_last = 0, t_stored = 0, dt = 0, t1w = 0,
           dv = 0;
  int w = -1, cnt = 0, peak = 0, filt = 0, icf = 0, disc = 0;
  bool has = false, has_last = false, last_stored = false;
  auto refresh = [&](int p) {
    unsigned q = cur[p];
    const unsigned d = ic[p];
    if (d > 0) {
      while (q + 1 < end[p] && src[p][q + 1] - src[p][q] < d) {
        q += 2;
        ++icf;
      }
      cur[p] = q;
    }
    nxt[p] = q < end[p] ? src[p][q] + d : INF;
  };
  auto start = [&](unsigned i) {
    const unsigned e = S.list[i];
    w = (int)(e & 0xFFu);
    idx = e >> 8;
    has = true;
    cnt = peak = filt = icf = disc = 0;
    so = 0;
#pragma unroll
    for (int p = 0; p < K; ++p) {
      cur[p] = S.offs[p][w];
      end[p] = S.offs[p][w + 1];
      so += cur[p];
      refresh(p);
    }
    y0 = y = (unsigned)(lut >> idx) & 1u;
    wlen = __ldg(C.wlen32 + base_w + w);
    has_last = last_stored = false;
    dv = y0;
    dt = t1w = 0;
  };
  auto finish = [&]() {
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
      // below 100 % stored edges may be popped: the dwell comes from the
      // final stored waveform (dwell_sweep, _kernels.py:254-295)
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
    S.cnt[w] = (unsigned)cnt;
    acc.filt += (unsigned)filt;
    acc.icf += (unsigned)icf;
    acc.disc += disc;
    record_arena<MODE, unsigned>(C, g, base_w + w, cnt, peak, filt, icf, disc, y0,
                                 [&](int j) -> unsigned & { return stage[so + j]; });
    has = false;
  };
  auto first_event = [&]() {
    unsigned t = nxt[0];
#pragma unroll
    for (int p = 1; p < K; ++p) t = min(t, nxt[p]);
    return t;
  };
  volatile unsigned *next = &S.next;
  unsigned tmin = INF;
  auto refill = [&]() {
    while (*next < nwork) {
      if (has) finish();
      const unsigned nw = atomicAdd(&S.next, 1u);
      if (nw >= nwork) break;
      start(nw);
      tmin = first_event();
      if (tmin != INF) break;
    }
  };
  if (lane_id() < nwork) {
    start(lane_id());
    tmin = first_event();
    if (tmin == INF) refill();
  }
  while (true) {
    const bool live = has && tmin != INF;
    if (!__any_sync(0xffffffffu, live)) break;
    if (live) {
      unsigned sw = 0;
#pragma unroll
      for (int p = 0; p < K; ++p) sw |= (nxt[p] == tmin ? 1u : 0u) << p;
      idx ^= sw;
#pragma unroll
      for (int p = 0; p < K; ++p)
        if ((sw >> p) & 1u) {
          cur[p] += 1;
          refresh(p);
        }
      // output side (K:136-193), as selects so the lanes stay converged
      const unsigned ny = (unsigned)(lut >> idx) & 1u;
      const bool chg = ny != y;
      const int col = ny ? 0 : 1;
      const unsigned dly = dtab_delay<K>(S.dtab, sw, idx, col);
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
      tmin = first_event();
      if (tmin == INF) refill();
    }
  }
  if (has) finish();
}

// ------------------------------------------------------------ one tile
// Per-lane window metadata, 8 bits per window j of the lane: start input
// vector (bits 0-3), the pin of a single transition (4-5), class (6-7).
enum LeanClass : unsigned { CL_QUIET = 0, CL_ONE = 1, CL_TWO = 2, CL_LOOP = 3 };
__device__ __forceinline__ unsigned meta_ix(unsigned m, int j) { return (m >> (8 * j)) & 15u; }
__device__ __forceinline__ unsigned meta_pin(unsigned m, int j) { return (m >> (8 * j + 4)) & 3u; }
__device__ __forceinline__ unsigned meta_cls(unsigned m, int j) { return (m >> (8 * j + 6)) & 3u; }

template <int MODE, int K, bool PCT100>
__device__ __forceinline__ void lean_tile(const ChunkDev &C, int g, int gnet,
                                          unsigned long long lut, const int (&net)[K],
                                          const unsigned (&ic)[K], int t, int pct, LeanSmem<K> &S,
                                          Region &R, unsigned &phase, LeanAcc &acc) {
  constexpr int SLAB = lean_slab_words<K>();
  const unsigned lane = lane_id();
  const int base_w = t * kTile;
  const int nact = min(kTile, C.Wc - base_w);
  const int wl = (int)lane * kWPL;
  const int Tw = C.Wpad / 32;
  unsigned *data = reinterpret_cast<unsigned *>(C.data);

  GS_PROF_T(pt0);
  GS_PROF_ADD(PF_TILES, 1);
  // ---- (1) fanin count rows -> window offsets; staging plan
  unsigned c[K][kWPL];
  unsigned long long tb[K];
  unsigned bits[K];
#pragma unroll
  for (int p = 0; p < K; ++p) {
    load_counts(C.cnt + (size_t)net[p] * C.Wpad + base_w + wl, c[p]);
    tb[p] = __ldg(C.tbase + (size_t)net[p] * C.Tc + t);
    bits[p] = load_init_bits(C.init + (size_t)net[p] * Tw, t);
  }
  unsigned n[kWPL], sidx[kWPL], meta = 0;
#pragma unroll
  for (int j = 0; j < kWPL; ++j) n[j] = sidx[j] = 0;
  unsigned tot[K], seg[K], inw = 0, UB = 0;
#pragma unroll
  for (int p = 0; p < K; ++p) {
    unsigned s4 = 0;
#pragma unroll
    for (int j = 0; j < kWPL; ++j) s4 += c[p][j];
    unsigned ex = warp_excl_scan(s4, &tot[p]);
    const unsigned sh = (unsigned)tb[p] & 3u;
    seg[p] = inw + sh;
    inw += tot[p] ? (sh + tot[p] + 3u) & ~3u : 0u;
    UB += tot[p];
    unsigned o4[kWPL];
#pragma unroll
    for (int j = 0; j < kWPL; ++j) {
      o4[j] = ex;
      // the single transition of a one-transition window: its slab position
      if (c[p][j]) {
        sidx[j] = seg[p] + ex;
        meta = (meta & ~(3u << (8 * j + 4))) | ((unsigned)p << (8 * j + 4));
      }
      n[j] += c[p][j];
      meta |= ((bits[p] >> j) & 1u) << (8 * j + p);
      ex += c[p][j];
    }
    st4(&S.offs[p][wl], o4);
    if (lane == kWarp - 1) S.offs[p][kTile] = tot[p];
  }
  // inputs (aligned per pin) and worklist outputs (UB words) in the slab, or
  // both in global memory
  const bool in_smem = inw + UB <= (unsigned)SLAB;
  const unsigned *src[K];
  unsigned *stage;
  bool ok = true;
  if (in_smem) {
    if (inw) {
      __syncwarp();
      if (lane == 0) {
        fence_proxy_async();  // the slab's previous generic accesses before the async writes
        mbar_expect_tx(&S.mbar, inw * 4u);
#pragma unroll
        for (int p = 0; p < K; ++p)
          if (tot[p]) {
            const unsigned sh = (unsigned)tb[p] & 3u;
            bulk_g2s(&S.slab[seg[p] - sh], data + (tb[p] - sh), ((sh + tot[p] + 3u) & ~3u) * 4u,
                     &S.mbar);
          }
      }
    }
#pragma unroll
    for (int p = 0; p < K; ++p) src[p] = &S.slab[seg[p]];
    stage = &S.slab[inw];
  } else {
#pragma unroll
    for (int p = 0; p < K; ++p) src[p] = data + tb[p];
    const unsigned long long sb = region_alloc(C, R, UB);
    ok = sb != ~0ull;
    stage = data + (ok ? sb : 0ull);
  }

  // ---- (2) classes; worklist of the windows with >= 2 transitions (>= 1
  // when reading in place), loop windows (>= 3) at the front.  A single
  // transition's slab position waits in S.cnt until the inline pass.
  unsigned cl = 0;
#pragma unroll
  for (int j = 0; j < kWPL; ++j) {
    const bool act = ok && wl + j < nact;
    const unsigned k = !act || n[j] == 0 ? CL_QUIET
                       : !in_smem || n[j] > 2 ? CL_LOOP
                       : n[j] == 2 ? CL_TWO : CL_ONE;
    meta |= k << (8 * j + 6);
    cl += k == CL_LOOP ? 1u : k == CL_TWO ? 1u << 16 : 0u;
  }
  st4(&S.cnt[wl], sidx);
  unsigned tot2;
  {
    const unsigned x = warp_excl_scan(cl, &tot2);
    unsigned xl = x & 0xFFFFu, xt = (tot2 & 0xFFFFu) + (x >> 16);
#pragma unroll
    for (int j = 0; j < kWPL; ++j) {
      const unsigned k = meta_cls(meta, j);
      if (k >= CL_TWO) S.list[k == CL_LOOP ? xl++ : xt++] = (unsigned)(wl + j) | (meta_ix(meta, j) << 8);
    }
  }
  if (lane == 0) S.next = kWarp;
  // wait for the staged segments (all lanes observe the barrier phase)
  if (in_smem && inw) {
    mbar_wait(&S.mbar, phase);
    phase ^= 1u;
  }
  __syncwarp();
  GS_PROF_T(pt1);
  GS_PROF_ADD(PF_PHASE1, pt1 - pt0);

  // ---- (3) two transitions, closed form (one window per lane per round).
  // With no edge pending at the first event, Algo. 1's output side
  // (K:136-203) collapses to selects: event 1 (both pins when the two
  // transitions coincide) can only emit; event 2 can emit, cancel event 1's
  // edge, or leave it pending; no stored edge can be popped.
  const unsigned nloop = tot2 & 0xFFFFu, nlist = nloop + (tot2 >> 16);
  for (unsigned i = nloop + lane; i < nlist; i += kWarp) {
    const unsigned e = S.list[i];
    const int w = (int)(e & 0xFFu);
    const unsigned i0 = e >> 8;
    unsigned nt = 0, pa = 0, pb = 0, so = 0;
    const unsigned *qa = src[0], *qb = src[0];
#pragma unroll
    for (int p = 0; p < K; ++p) {
      const unsigned a = S.offs[p][w], m = S.offs[p][w + 1] - a;
      so += a;
      pa = (m >= 1 && nt == 0) ? (unsigned)p : pa;
      qa = (m >= 1 && nt == 0) ? src[p] + a : qa;
      pb = ((m >= 1 && nt == 1) || (m >= 2 && nt == 0)) ? (unsigned)p : pb;
      qb = (m >= 1 && nt == 1) ? src[p] + a : (m >= 2 && nt == 0) ? src[p] + a + 1 : qb;
      nt += m;
    }
    unsigned ica = ic[0], icb = ic[0];
#pragma unroll
    for (int p = 1; p < K; ++p) {
      ica = pa == (unsigned)p ? ic[p] : ica;
      icb = pb == (unsigned)p ? ic[p] : icb;
    }
    const unsigned va = *qa, vb = *qb;
    // a same-pin pair narrower than the pin's interconnect delay is
    // filtered out whole (_kernels.py:96-117): no event remains
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
    const unsigned d2 = dtab_delay<K>(S.dtab, s2, i2, y2 ? 0 : 1);
    const unsigned o1 = ta + dtab_delay<K>(S.dtab, s1, i1, y1 ? 0 : 1);
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
    // dwell at 1: +-edge times by the value before each edge, plus the
    // window end when the final value is 1 (wrapping arithmetic, exact
    // since the result lies in [0, wlen])
    const unsigned e0 = cnt >= 1 ? f0 : 0u, e1 = cnt == 2 ? tp : 0u;
    const unsigned wf = (cnt & 1u) ? (yy0 ? 0u : wlw) : (yy0 ? wlw : 0u);
    acc.t1 += (long long)(yy0 ? e0 - e1 + wf : e1 - e0 + wf);
    S.cnt[w] = cnt;
    acc.filt += x2 ? 1u : 0u;
    acc.icf += pairf ? 1u : 0u;
    acc.disc += disc;
    if (MODE != MODE_STATS)
      record_arena<MODE, unsigned>(C, g, base_w + w, (int)cnt, (int)cnt, x2 ? 1 : 0,
                                   pairf ? 1 : 0, disc, yy0,
                                   [&](int q) -> unsigned & { return st[q]; });
  }
  GS_PROF_T(pt2);
  GS_PROF_ADD(PF_CLOSED, pt2 - pt1);
  GS_PROF_ADD(PF_LOOP_WINDOWS, nloop);
  GS_PROF_ADD(PF_TRIVIAL, nlist - nloop);
  // ---- (4) three or more transitions: the event loop
  if (nloop) lean_loop<MODE, K, PCT100>(C, g, lut, ic, pct, S, src, stage, base_w, nloop, acc);
  __syncwarp();
  GS_PROF_T(pt3);
  GS_PROF_ADD(PF_LOOP, pt3 - pt2);

  // ---- (5) the lane's own windows: quiet and single-transition windows in
  // registers, then compaction and the per-net sums
  unsigned cm[kWPL], wlen[kWPL], ot[kWPL], co[kWPL], nib = 0, s = 0;
  ld4(&S.cnt[wl], cm);   // worklist windows: stored count; one-transition: slab position
  load_counts(C.wlen32 + base_w + wl, wlen);
#pragma unroll
  for (int j = 0; j < kWPL; ++j) {
    const unsigned k = meta_cls(meta, j), ix = meta_ix(meta, j), p1 = meta_pin(meta, j);
    const bool act = ok && wl + j < nact;
    const bool one = k == CL_ONE;
    unsigned icp = ic[0];
#pragma unroll
    for (int p = 1; p < K; ++p) icp = p1 == (unsigned)p ? ic[p] : icp;
    const unsigned tv = one ? S.slab[one ? cm[j] : 0u] + icp : 0u;
    const unsigned y0 = (unsigned)(lut >> ix) & 1u;
    const unsigned i1 = ix ^ (1u << p1);
    const unsigned y1 = (unsigned)(lut >> i1) & 1u;
    const bool chg = one && y1 != y0;
    ot[j] = tv + dtab_pin<K>(S.dtab, p1, i1, y1 ? 0u : 1u);
    const bool inwin = ot[j] < wlen[j];
    const bool st = chg && inwin;
    const bool inl = act && k <= CL_ONE;
    acc.disc += (chg && !inwin) ? 1 : 0;
    acc.t1 += inl ? (y0 ? (st ? ot[j] : wlen[j]) : (st ? wlen[j] - ot[j] : 0u)) : 0u;
    co[j] = !act ? 0u : k >= CL_TWO ? cm[j] : st ? 1u : 0u;
    nib |= (act ? y0 : 0u) << j;
    s += co[j];
    if (MODE != MODE_STATS && inl)
      record_arena<MODE, unsigned>(C, g, base_w + wl + j, (int)co[j], (int)co[j], 0, 0,
                                   (chg && !inwin) ? 1 : 0, y0,
                                   [&](int) -> unsigned & { return ot[j]; });
  }
  unsigned CNT;
  const unsigned cx = warp_excl_scan(s, &CNT);
  const unsigned long long ob = CNT ? region_alloc(C, R, CNT) : 0ull;
  const bool wrote = ob != ~0ull;  // else the chunk is re-run; keep readers in bounds
  if (wrote) {
    unsigned *dst = data + ob + cx;
#pragma unroll
    for (int j = 0; j < kWPL; ++j) {
      if (meta_cls(meta, j) <= CL_ONE) {
        if (co[j]) dst[0] = ot[j];
      } else if (co[j]) {
        unsigned so = 0;
#pragma unroll
        for (int p = 0; p < K; ++p) so += S.offs[p][wl + j];
        for (unsigned q = 0; q < co[j]; ++q) dst[q] = stage[so + q];
      }
      dst += co[j];
    }
  }
  acc.tc += s;
  // the gate's own net: tile base, counts, window-start bits
  if (lane == 0) C.tbase[(size_t)gnet * C.Tc + t] = wrote ? ob : 0ull;
  store_counts(C.cnt + (size_t)gnet * C.Wpad + base_w + wl, co, wrote);
  store_init_words(C.init + (size_t)gnet * Tw, t, nib);
  __syncwarp();
  GS_PROF_T(pt4);
  GS_PROF_ADD(PF_PHASE3, pt4 - pt3);
}

// condition tables of one gate -> smem: arcs[(p << (K-1) | row) * 2 + col],
// then the delay table of the event step: k <= 2 by (switching pin set,
// post-transition inputs, edge) -- the max over the switching arcs of the
// conditioned delay (K:139-151); k = 3, 4 by (single pin, inputs, edge),
// simultaneous pins taking the max of their entries
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
  __syncwarp();
}

// One launch per (logic level, fanin-count group), as gate_eval: persistent
// grid, work items (gate, run of tiles) fetched from a per-launch counter in
// tile-group-major order, head items of tpi tiles then tail items of tpi2.
template <int MODE, int K, bool PCT100>
__global__ void __launch_bounds__(kEvalThreads, lean_ctas<K>())
gate_eval_lean(DesignDev D, ChunkDev C, LevelArgs A) {
  using SM = LeanSmem<K>;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int warp = threadIdx.x / kWarp;
  SM &S = reinterpret_cast<SM *>(smem_raw)[warp];
  const unsigned lane = lane_id();
  Region R = region_open(C, (unsigned long long)blockIdx.x * kEvalWarps + warp);
  if (lane == 0) mbar_init(&S.mbar, 1);
  __syncwarp();
  unsigned phase = 0;
  const unsigned head = (unsigned)A.n * (unsigned)A.ntg;
  const unsigned items = head + (unsigned)A.n * (unsigned)A.ntg2;
  while (true) {
    unsigned it = 0;
    if (lane == 0) it = atomicAdd(C.work + A.counter, 1u);
    it = __shfl_sync(0xffffffffu, it, 0);
    if (it >= items) break;
    const bool in_head = it < head;
    const unsigned iq = in_head ? it : it - head;
    const int j = (int)(iq % (unsigned)A.n);
    const int tg = (int)(iq / (unsigned)A.n);
    const int g = __ldg(D.order + A.lo + j);
    const int pin0 = __ldg(D.gate_pin + g);
    const unsigned long long lut = __ldg(D.gate_lut + g);
    const int t_lo = in_head ? tg * A.tpi : A.ntg * A.tpi + tg * A.tpi2;
    const int t_hi = min(t_lo + (in_head ? A.tpi : A.tpi2), C.Tc);
    int net[K], arc[K];
    unsigned ic[K];
#pragma unroll
    for (int p = 0; p < K; ++p) {
      net[p] = __ldg(D.pin_net + pin0 + p);
      ic[p] = (unsigned)__ldg(D.pin_ic + pin0 + p);
      arc[p] = __ldg(D.pin_arc + pin0 + p);
    }
    build_dtab<K>(S.arcs, S.dtab, D.arc32, arc);
    LeanAcc acc;
    for (int t = t_lo; t < t_hi; ++t)
      lean_tile<MODE, K, PCT100>(C, g, D.P + g, lut, net, ic, t, A.pct, S, R, phase, acc);
    acc_flush(C, D.P + g, acc.t1, acc.tc, (long long)acc.filt, (long long)acc.icf,
              (long long)acc.disc);
  }
  region_close(C, R);
}

template <int K>
constexpr size_t lean_smem_bytes() {
  return sizeof(LeanSmem<K>) * kEvalWarps;
}

}  // namespace gs
