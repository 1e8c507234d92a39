/*
 * glsim_oracle.c -- CPU restatement of the reference hot-path kernels.
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the parity checker for the CUDA
 * engine and the CPU baseline of bench.py.  Nothing in the product package
 * (paper_2203_06117_b200/) may import, link or call it.
 *
 * Each function restates one numba kernel of the reference, statement for
 * statement, over the same flat int64/uint8 arrays:
 *   or_sim_span     <- pkg/src/glsim/_kernels.py:17-210   (sim_span, Algo. 1)
 *   or_init_values  <- pkg/src/glsim/_kernels.py:213-231  (init_values)
 *   or_level_ub     <- pkg/src/glsim/_kernels.py:234-251  (level_ub)
 *   or_dwell_sweep  <- pkg/src/glsim/_kernels.py:254-295  (dwell_sweep)
 * Two-dimensional numpy arrays are passed row-major with their column count.
 * or_sim_span_mt splits the gate range over OpenMP threads exactly like the
 * reference's _run_level splits it over its thread pool (simcore.py:295-325):
 * tasks touch disjoint (gate, window) regions, so the result is independent
 * of the thread count.
 */
#include <stdint.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define I64MAX INT64_MAX
#define MAXK 16

typedef int64_t i64;
typedef uint8_t u8;

/* _kernels.py:17-210 */
void or_sim_span(i64 oi_lo, i64 oi_hi, i64 w_lo, i64 w_hi, i64 w_off,
                 const i64 *order, const i64 *pin_off, const i64 *pin_net, const i64 *pin_ic,
                 const i64 *pin_arc, const i64 *arc_rows, const i64 *lut_off, const u8 *lut_bits,
                 const i64 *out_net, const u8 *net_kind, const i64 *net_slot,
                 const i64 *stim_buf, const i64 *stim_off, const i64 *stim_cnt, i64 stim_cols,
                 const u8 *init_vals, i64 init_cols, const i64 *boundaries,
                 i64 *gbuf, const i64 *g_off, const i64 *g_cap, i64 *g_cnt, i64 g_cols,
                 i64 *out_filt, i64 *out_icf, i64 *out_disc, i64 *out_err, i64 *out_peak,
                 i64 pct) {
  i64 pos[MAXK], nxt[MAXK], sof[MAXK], scn[MAXK];
  u8 val[MAXK], sst[MAXK];
  (void)out_net;
  for (i64 oi = oi_lo; oi < oi_hi; ++oi) {
    const i64 g = order[oi];
    const i64 p0 = pin_off[g];
    const i64 k = pin_off[g + 1] - p0;
    const i64 lidx = lut_off[g];
    for (i64 w = w_lo; w < w_hi; ++w) {
      const i64 wj = w - w_off;
      const i64 wend = boundaries[w + 1];
      i64 idx = 0;
      for (i64 p = 0; p < k; ++p) {
        const i64 n = pin_net[p0 + p];
        const i64 s = net_slot[n];
        if (net_kind[n] == 0) {
          sof[p] = stim_off[s * stim_cols + w];
          scn[p] = stim_cnt[s * stim_cols + w];
          sst[p] = 1;
        } else {
          sof[p] = g_off[s * g_cols + wj];
          scn[p] = g_cnt[s * g_cols + wj];
          sst[p] = 0;
        }
        pos[p] = 0;
        nxt[p] = -1; /* needs refresh */
        const u8 v = init_vals[n * init_cols + w];
        val[p] = v;
        if (v) idx |= (i64)1 << p;
      }
      u8 y = lut_bits[lidx + idx];
      i64 cnt = 0, peak = 0, filt = 0, icf = 0, disc = 0;
      int has_last = 0, last_stored = 0;
      i64 t_last = 0;
      const i64 roff = g_off[g * g_cols + wj];
      const i64 rcap = g_cap[g * g_cols + wj];
      int err = 0;
      for (;;) {
        i64 tmin = I64MAX;
        for (i64 p = 0; p < k; ++p) {
          if (nxt[p] == -1) {
            const i64 d = pin_ic[p0 + p];
            const i64 *src = sst[p] ? stim_buf : gbuf;
            while (pos[p] + 1 < scn[p]) {
              const i64 ta = src[sof[p] + pos[p]];
              const i64 tb = src[sof[p] + pos[p] + 1];
              if (tb - ta < d) {
                pos[p] += 2;
                icf += 1;
              } else {
                break;
              }
            }
            nxt[p] = pos[p] < scn[p] ? src[sof[p] + pos[p]] + d : I64MAX;
          }
          if (nxt[p] < tmin) tmin = nxt[p];
        }
        if (tmin == I64MAX) break;
        i64 sw = 0;
        for (i64 p = 0; p < k; ++p) {
          if (nxt[p] == tmin) {
            pos[p] += 1;
            nxt[p] = -1;
            if (val[p]) {
              val[p] = 0;
              idx &= ~((i64)1 << p);
            } else {
              val[p] = 1;
              idx |= (i64)1 << p;
            }
            sw |= (i64)1 << p;
          }
        }
        const u8 new_y = lut_bits[lidx + idx];
        if (new_y != y) {
          const i64 col = new_y == 1 ? 0 : 1;
          i64 dly = 0;
          for (i64 p = 0; p < k; ++p) {
            if (sw & ((i64)1 << p)) {
              i64 row = 0, j = 0;
              for (i64 q = 0; q < k; ++q) {
                if (q != p) {
                  if (val[q]) row |= (i64)1 << j;
                  j += 1;
                }
              }
              const i64 a = arc_rows[(pin_arc[p0 + p] + row) * 2 + col];
              if (a > dly) dly = a;
            }
          }
          const i64 t_out = tmin + dly;
          const i64 thr = dly * pct / 100; /* operands non-negative: == floor div */
          int have_tgt;
          i64 t_tgt;
          if (has_last) {
            have_tgt = 1;
            t_tgt = t_last;
          } else if (cnt > 0) {
            have_tgt = 1;
            t_tgt = gbuf[roff + cnt - 1];
          } else {
            have_tgt = 0;
            t_tgt = 0;
          }
          if (have_tgt && (t_out <= t_tgt || t_out - t_tgt < thr)) {
            if (has_last) {
              if (!last_stored) disc -= 1;
              has_last = 0;
            } else {
              cnt -= 1;
            }
            filt += 1;
          } else {
            if (has_last && last_stored) {
              if (cnt < rcap) {
                gbuf[roff + cnt] = t_last;
                cnt += 1;
              } else {
                err = 1;
                cnt += 1;
              }
              if (cnt > peak) peak = cnt;
            }
            if (t_out < wend) {
              last_stored = 1;
            } else {
              disc += 1;
              last_stored = 0;
            }
            has_last = 1;
            t_last = t_out;
          }
          y = new_y;
        }
      }
      if (has_last && last_stored) {
        if (cnt < rcap) {
          gbuf[roff + cnt] = t_last;
          cnt += 1;
        } else {
          err = 1;
          cnt += 1;
        }
        if (cnt > peak) peak = cnt;
      }
      g_cnt[g * g_cols + wj] = cnt;
      out_filt[g * g_cols + wj] = filt;
      out_icf[g * g_cols + wj] = icf;
      out_disc[g * g_cols + wj] = disc;
      out_peak[g * g_cols + wj] = peak;
      if (err) out_err[g * g_cols + wj] = 1;
    }
  }
}

/* the reference's _run_level task split (simcore.py:295-325) on OpenMP threads:
 * gate chunks of ceil(n / (4 * threads)) x window batches of cycle_parallelism */
void or_sim_span_mt(int threads, i64 cycle_parallelism, i64 oi_lo, i64 oi_hi, i64 w_lo, i64 w_hi,
                    i64 w_off, const i64 *order, const i64 *pin_off, const i64 *pin_net,
                    const i64 *pin_ic, const i64 *pin_arc, const i64 *arc_rows,
                    const i64 *lut_off, const u8 *lut_bits, const i64 *out_net,
                    const u8 *net_kind, const i64 *net_slot, const i64 *stim_buf,
                    const i64 *stim_off, const i64 *stim_cnt, i64 stim_cols, const u8 *init_vals,
                    i64 init_cols, const i64 *boundaries, i64 *gbuf, const i64 *g_off,
                    const i64 *g_cap, i64 *g_cnt, i64 g_cols, i64 *out_filt, i64 *out_icf,
                    i64 *out_disc, i64 *out_err, i64 *out_peak, i64 pct) {
  const i64 n = oi_hi - oi_lo;
  if (threads < 1) threads = 1;
  i64 chunk = (n + 4 * threads - 1) / (4 * threads);
  if (chunk < 1) chunk = 1;
  const i64 ng = (n + chunk - 1) / chunk;
  const i64 nb = (w_hi - w_lo + cycle_parallelism - 1) / cycle_parallelism;
  const i64 tasks = ng * nb;
#pragma omp parallel for schedule(dynamic, 1) num_threads(threads)
  for (i64 t = 0; t < tasks; ++t) {
    const i64 s = oi_lo + (t / nb) * chunk;
    const i64 e = s + chunk < oi_hi ? s + chunk : oi_hi;
    const i64 wb = w_lo + (t % nb) * cycle_parallelism;
    const i64 we = wb + cycle_parallelism < w_hi ? wb + cycle_parallelism : w_hi;
    or_sim_span(s, e, wb, we, w_off, order, pin_off, pin_net, pin_ic, pin_arc, arc_rows, lut_off,
                lut_bits, out_net, net_kind, net_slot, stim_buf, stim_off, stim_cnt, stim_cols,
                init_vals, init_cols, boundaries, gbuf, g_off, g_cap, g_cnt, g_cols, out_filt,
                out_icf, out_disc, out_err, out_peak, pct);
  }
}

/* _kernels.py:213-231 ; vals is [num_nets][W], rows < P preset by the caller */
void or_init_values(i64 num_gates, const i64 *order, const i64 *pin_off, const i64 *pin_net,
                    const i64 *lut_off, const u8 *lut_bits, const i64 *out_net, u8 *vals, i64 W) {
  for (i64 oi = 0; oi < num_gates; ++oi) {
    const i64 g = order[oi];
    const i64 p0 = pin_off[g];
    const i64 k = pin_off[g + 1] - p0;
    const i64 lidx = lut_off[g];
    for (i64 w = 0; w < W; ++w) {
      i64 idx = 0;
      for (i64 p = 0; p < k; ++p)
        if (vals[pin_net[p0 + p] * W + w]) idx |= (i64)1 << p;
      vals[out_net[g] * W + w] = lut_bits[lidx + idx];
    }
  }
}

/* _kernels.py:234-251 ; ub is [oi_hi-oi_lo][w_hi-w_lo] */
void or_level_ub(const i64 *order, i64 oi_lo, i64 oi_hi, const i64 *pin_off, const i64 *pin_net,
                 const u8 *net_kind, const i64 *net_slot, const i64 *stim_cnt, i64 stim_cols,
                 const i64 *g_cnt, i64 g_cols, i64 w_lo, i64 w_hi, i64 w_off, i64 *ub) {
  const i64 ws = w_hi - w_lo;
  for (i64 i = 0; i < oi_hi - oi_lo; ++i) {
    const i64 g = order[oi_lo + i];
    const i64 p0 = pin_off[g];
    const i64 k = pin_off[g + 1] - p0;
    for (i64 w = w_lo; w < w_hi; ++w) {
      i64 total = 0;
      for (i64 p = 0; p < k; ++p) {
        const i64 n = pin_net[p0 + p];
        const i64 s = net_slot[n];
        if (net_kind[n] == 0) total += stim_cnt[s * stim_cols + w];
        else total += g_cnt[s * g_cols + (w - w_off)];
      }
      ub[i * ws + (w - w_lo)] = total;
    }
  }
}

/* _kernels.py:254-295 ; adds into t0/t1/tc [num_nets] */
void or_dwell_sweep(i64 num_nets, const u8 *net_kind, const i64 *net_slot, const i64 *stim_buf,
                    const i64 *stim_off, const i64 *stim_cnt, const u8 *stim_init, i64 stim_cols,
                    const i64 *gbuf, const i64 *g_off, const i64 *g_cnt, const u8 *g_init,
                    i64 g_cols, const i64 *boundaries, i64 w_lo, i64 w_hi, i64 w_off,
                    i64 *t0_out, i64 *t1_out, i64 *tc_out, int threads) {
#pragma omp parallel for schedule(static) num_threads(threads > 0 ? threads : 1)
  for (i64 n = 0; n < num_nets; ++n) {
    const i64 s = net_slot[n];
    i64 acc0 = 0, acc1 = 0, tcn = 0;
    for (i64 w = w_lo; w < w_hi; ++w) {
      i64 off, cnt;
      u8 v;
      if (net_kind[n] == 0) {
        off = stim_off[s * stim_cols + w];
        cnt = stim_cnt[s * stim_cols + w];
        v = stim_init[s * stim_cols + w];
      } else {
        off = g_off[s * g_cols + (w - w_off)];
        cnt = g_cnt[s * g_cols + (w - w_off)];
        v = g_init[s * g_cols + (w - w_off)];
      }
      i64 prev = boundaries[w];
      for (i64 i = 0; i < cnt; ++i) {
        const i64 t = net_kind[n] == 0 ? stim_buf[off + i] : gbuf[off + i];
        if (v) acc1 += t - prev;
        else acc0 += t - prev;
        v ^= 1;
        prev = t;
      }
      const i64 endt = boundaries[w + 1];
      if (v) acc1 += endt - prev;
      else acc0 += endt - prev;
      tcn += cnt;
    }
    t0_out[n] += acc0;
    t1_out[n] += acc1;
    tc_out[n] += tcn;
  }
}

int or_max_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}
