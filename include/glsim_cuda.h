/*
 * glsim_cuda.h -- C ABI of libglsim_cuda.so, the B200 (sm_100a) engine for the
 * windowed gate-level re-simulation hot path of GATSPI (arXiv 2203.06117).
 *
 * The reference package calls its hot path through four numba kernels in
 * pkg/src/glsim/_kernels.py, orchestrated by pkg/src/glsim/simcore.py and
 * report.py.  This library replaces that seam.  Every entry point below names
 * the reference interface it stands in for (file:line, 1-based).
 *
 * Conventions
 *   - plain pointers and sizes only; all pointers are HOST pointers unless a
 *     parameter name ends in _dev;
 *   - integers are the reference's int64 femtoseconds / counts (numpy int64),
 *     value bits are uint8 (numpy uint8);
 *   - every function returns a gs_status (0 = ok); gs_last_error() returns a
 *     thread-local message for the last failure;
 *   - the caller owns all host memory; handles own their device memory;
 *   - one engine per device; calls on one engine are not thread-safe.
 */
#ifndef GLSIM_CUDA_H
#define GLSIM_CUDA_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum gs_status {
  GS_OK = 0,
  GS_ERR_ARG = 1,         /* bad argument / unsupported input  -> ValueError        */
  GS_ERR_CUDA = 2,        /* CUDA runtime failure              -> RuntimeError      */
  GS_ERR_NODEVICE = 3,    /* no CUDA device visible            -> RuntimeError      */
  GS_ERR_CAPACITY = 4,    /* device memory cannot hold one tile-> CapacityError     */
  GS_ERR_CONSISTENCY = 5, /* device-side invariant violated    -> ConsistencyError  */
  GS_ERR_PARSE = 6,       /* malformed document (line in gs_last_error_line) -> ParseError */
  GS_ERR_SEMANTIC = 7,    /* document breaks a design contract -> SemanticError     */
  GS_ERR_UNSUPPORTED = 8  /* input outside the native reader's byte-exact subset:
                             the caller uses its own (Python) reader            */
} gs_status;

typedef struct gs_design gs_design;
typedef struct gs_stim gs_stim;
typedef struct gs_engine gs_engine;
typedef struct gs_vcd gs_vcd;

/* Flat design, exactly the arrays of reference CompiledDesign
 * (pkg/src/glsim/simcore.py:203-272) plus the levelization
 * (pkg/src/glsim/netlist.py:293-312).  Gate g drives net num_pis + g
 * (netlist.py:144-149). */
typedef struct gs_design_desc {
  int64_t num_pis, num_gates, num_levels;
  const int64_t *order;        /* [G] gates in level order               */
  const int64_t *level_starts; /* [L+1] CSR offsets into order           */
  const int64_t *pin_off;      /* [G+1]                                   */
  const int64_t *pin_net;      /* [sum k] driving net of each input pin   */
  const int64_t *pin_ic;       /* [sum k] interconnect delay (fs)         */
  const int64_t *pin_arc;      /* [sum k] first row of the pin's table    */
  const int64_t *arc_rows;     /* [R*2] (rise, fall) per condition row    */
  int64_t num_arc_rows;
  const int64_t *lut_off;      /* [G] offset of the gate's truth table    */
  const uint8_t *lut_bits;     /* [sum 2^k]                               */
  int64_t num_lut_bits;
} gs_design_desc;

/* Stimulus.  Either the whole-run CSR form (what StimulusSet.build receives,
 * pkg/src/glsim/waveform.py:243-265; kernel K1 cuts the windows on the GPU)
 * or the reference's windowed arrays (StimulusSet.__init__, waveform.py:235-241).
 * Set the pointers of exactly one form; the other form's pointers are NULL. */
typedef struct gs_stim_desc {
  int64_t num_pis, num_windows;
  const int64_t *boundaries;   /* [W+1] strictly ascending window edges    */
  /* CSR form */
  const int64_t *pi_off;       /* [P+1]                                    */
  const int64_t *pi_times;     /* [pi_off[P]] strictly ascending per input  */
  const uint8_t *pi_init;      /* [P]                                      */
  /* windowed form */
  const int64_t *buf;          /* [n_buf] absolute toggle times            */
  int64_t n_buf;
  const int64_t *offsets;      /* [P*W]                                    */
  const int64_t *counts;       /* [P*W]                                    */
  const uint8_t *initials;     /* [P*W]                                    */
} gs_stim_desc;

/* Per-net results of a stats run; host arrays the caller allocates. */
typedef struct gs_stats_out {
  int64_t *t1;    /* [N] fs at 1 (T0 = duration - T1)        (report.py:82-86)  */
  int64_t *tc;    /* [N] stored toggles                       (report.py:82-86)  */
  int64_t *ig;    /* [N] inertially filtered pulses, gates    (report.py:87-89)  */
  int64_t totals[3]; /* filtered, ic_filtered, discarded      (scheduler.py:70-74)*/
} gs_stats_out;

/* Per-(gate, window) arrays of one window range, row-major [G, Ws] (pitch Ws);
 * host arrays the caller allocates; any pointer may be NULL to skip it.
 * These are the fields of reference WaveformArena (waveform.py:280-303) and
 * PassResult (simcore.py:286-292). */
typedef struct gs_arena_out {
  int64_t *counts, *peak, *filtered, *ic_filtered, *discarded;
  uint8_t *initials;
  /* store pass: region offsets [G, Ws] into buf (waveform.py:340-345) and the
   * buffer itself (absolute int64 fs, sum(caps) entries).  buf != NULL makes
   * the run a store pass. */
  const int64_t *offsets;
  int64_t *buf;
  int64_t n_buf;
  /* store pass: region capacities [G, Ws] (pass-1 peak); a region that needs
   * more is GS_ERR_CONSISTENCY (sim_span's cap check).  NULL: not checked. */
  const int64_t *caps;
} gs_arena_out;

/* Timing of the last gs_run (CUDA events on the engine stream). */
typedef struct gs_timing {
  float ms_total;        /* all kernels of the run, device time               */
  float ms_gate_eval;    /* K4 launches only                                  */
  float ms_stim;         /* K1 launches only                                  */
  int64_t launches;      /* kernels launched                                  */
  int64_t gate_eval_launches;
  int64_t chunks;        /* window chunks the run was split into              */
  int64_t data_bytes_peak; /* high-water device waveform pool usage            */
  int64_t input_toggles; /* sum over gate-windows of fanin toggles (n_in)      */
  int64_t output_toggles;/* stored output toggles                              */
  int64_t graph_builds;  /* chunk launch sequences captured as CUDA graphs     */
  int64_t graph_replays; /* chunk graphs replayed from the engine's cache      */
} gs_timing;

/* ---- library ---------------------------------------------------------- */
int gs_version(void);
const char *gs_last_error(void);
int gs_device_count(int *count);

/* ---- design (replaces CompiledDesign, simcore.py:203-276) ------------- */
int gs_design_create(const gs_design_desc *desc, int device, gs_design **out);
int gs_design_destroy(gs_design *d);

/* ---- stimulus (replaces StimulusSet.build / slice_windows,
 *      waveform.py:49-63,243-265; the cutting itself runs in kernel K1) --- */
int gs_stim_create(gs_design *d, const gs_stim_desc *desc, gs_stim **out);
int gs_stim_destroy(gs_stim *s);

/* Synthetic benchmark stimulus, generated on the device (no reference
 * counterpart: the benchmark configs of SURVEY §8(d); bit-identical to the
 * package's synth.stimulus_arrays).  Input p toggles in absolute window w iff
 * (splitmix64(seed<<56 ^ p<<32 ^ w) >> 11) < thr (thr = ceil(alpha * 2^53)),
 * at w*period + lo + splitmix64(h1 ^ 0xD1B54A32D192ED03) % span; inputs
 * [0, num_ppis) use the ppi_* parameters.  The stimulus' window 0 is w_lo
 * (initial values carry the toggle parity of windows [0, w_lo)). */
typedef struct gs_synth_desc {
  int64_t num_pis, num_ppis;
  uint64_t seed;
  int64_t period;
  uint64_t ppi_thr, pi_thr;
  int64_t ppi_lo, ppi_span, pi_lo, pi_span;
  int64_t w_lo, w_hi;
} gs_synth_desc;
int gs_stim_synth(gs_design *d, const gs_synth_desc *desc, gs_stim **out);
/* per-window input toggles of the synthetic stimulus over [w_lo, w_hi) on
 * `device`, into counts [w_hi - w_lo] (the weights window shards are balanced
 * by, without generating the stimulus) */
int gs_synth_window_counts(const gs_synth_desc *desc, int device, int64_t *counts);
/* windows and input toggles of a stimulus */
int gs_stim_sizes(const gs_stim *s, int64_t *num_windows, int64_t *num_toggles);
/* copy a CSR stimulus back to host arrays: boundaries [W+1], pi_off [P+1],
 * pi_times [num_toggles], pi_init [P] (any may be NULL) */
int gs_stim_download(const gs_stim *s, int64_t *boundaries, int64_t *pi_off, int64_t *pi_times,
                     uint8_t *pi_init);

/* ---- engine ------------------------------------------------------------ */
/* mem_budget: bytes of device memory the engine may use for its window-chunk
 * workspace (0 = 75% of free memory).  stream: a cudaStream_t (NULL = the
 * engine's own stream). */
int gs_engine_create(gs_design *d, int64_t mem_budget, void *stream, gs_engine **out);
int gs_engine_destroy(gs_engine *e);
/* K4 work-item sizing (no reference counterpart; tuning and tests): the
 * number of workers items are sized for (0 = the launch's own grid), the
 * divisor the tail items are re-cut by (1 = no tail re-cut) and the largest
 * tail share 1/tail_frac of a launch's columns.  Results never depend on it. */
int gs_engine_set_items(gs_engine *e, int64_t workers, int tail_div, int tail_frac);
/* words per warp of the shared-memory slab that stages a tile's fanin
 * segments and outputs in the K4 instance for k-input gates (narrow != 0:
 * 32-bit window-relative time); tiles that do not fit read in place */
int gs_slab_words(int k, int narrow);

/* Stats run over windows [w_lo, w_hi): K1 stim_segment + per level K4
 * gate_eval with the dwell/toggle reduction fused (replaces count_pass +
 * store_pass + compute_stats: simcore.py:328-410, report.py:57-91,
 * _kernels.py:17-210,254-295).  Results are ADDED into *out (so window shards
 * and segments merge by summation, report.py:46-54).  pct = pathpulse percent
 * (scheduler.py:390). */
int gs_run_stats(gs_engine *e, gs_stim *s, int64_t w_lo, int64_t w_hi, int pct,
                 gs_stats_out *out);

/* Same run writing per-(gate, window) arena arrays for [w_lo, w_hi): a count
 * pass when arena->buf is NULL (count_pass, simcore.py:328-379, incl. peak),
 * a store pass into the reference arena layout otherwise (store_pass,
 * simcore.py:382-410).  stats may be NULL. */
int gs_run_arena(gs_engine *e, gs_stim *s, int64_t w_lo, int64_t w_hi, int pct,
                 gs_arena_out *arena, gs_stats_out *stats);

int gs_last_timing(gs_engine *e, gs_timing *t);

/* The arena buffer of the last count pass (gs_run_arena with buf == NULL) on
 * this engine, without a second simulation: the count pass keeps every
 * gate-window's peak entries (K5 packs them per window chunk, gate-major in
 * level order, absolute int64 times); this scatters them into `buf` at the
 * regions `offsets` [G, cols] (allocate_arena's layout, waveform.py:321-346)
 * -- the contents store_pass (simcore.py:382-410) would write.  *filled = 0
 * (and nothing written) unless the engine's last count pass was this
 * stimulus, window range and pct. */
int gs_arena_fill(gs_engine *e, const gs_stim *s, int64_t w_lo, int64_t w_hi, int pct,
                  int64_t *buf, int64_t n_buf, const int64_t *offsets, int64_t cols,
                  int *filled);

/* Device-side stats accumulation for multi-GPU reduction: like gs_run_stats
 * but ADDS into a caller-owned device buffer acc_dev of 3*N+3 int64
 * ([t1 | tc | ig | filtered, ic_filtered, discarded]), so the caller can
 * all-reduce it with NCCL before one host copy. */
int gs_run_stats_device(gs_engine *e, gs_stim *s, int64_t w_lo, int64_t w_hi, int pct,
                        int64_t *acc_dev);

/* Device-side cross-check of a run against reference waveforms (SURVEY
 * §8(f) item 4; the host compare_waveforms, pkg/src/glsim/oracle.py:201-226):
 * simulates windows [w_lo, w_hi) and compares, on the GPU, every gate's
 * window-start value, toggle count and toggle times with `ref` -- a reference
 * arena in the layout of gs_arena_out ([G][cols] offsets / counts / initials,
 * absolute int64 times in buf, column 0 = window w_lo).  Returns the number
 * of mismatching (gate, window) pairs and the first one (gate, absolute
 * window; -1 when none). */
typedef struct gs_arena_ref {
  const int64_t *buf;
  int64_t n_buf;
  const int64_t *offsets, *counts;
  const uint8_t *initials;
  int64_t cols;
} gs_arena_ref;
int gs_run_compare(gs_engine *e, gs_stim *s, int64_t w_lo, int64_t w_hi, int pct,
                   const gs_arena_ref *ref, int64_t *mismatches, int64_t *first_gate,
                   int64_t *first_window);

/* ---- kernel-seam entry points: same arguments as the reference's numba
 * kernels, host arrays in and out, executed on the GPU ------------------- */

/* dwell_sweep (_kernels.py:254-295): per-net T0/T1/TC over windows
 * [w_lo, w_hi) of windowed stimulus + arena arrays; ADDS into t0/t1/tc [N].
 * g_* arrays are [G, Wg] with column = window - w_off. */
int gs_dwell_sweep(int64_t num_nets, const uint8_t *net_kind, const int64_t *net_slot,
                   const int64_t *stim_buf, int64_t n_stim_buf,
                   const int64_t *stim_off, const int64_t *stim_cnt, const uint8_t *stim_init,
                   int64_t num_pis, int64_t num_windows,
                   const int64_t *gbuf, int64_t n_gbuf,
                   const int64_t *g_off, const int64_t *g_cnt, const uint8_t *g_init,
                   int64_t num_gates, int64_t g_cols,
                   const int64_t *boundaries, int64_t w_lo, int64_t w_hi, int64_t w_off,
                   int64_t *t0_out, int64_t *t1_out, int64_t *tc_out);

/* sim_span (_kernels.py:17-210): Algo. 1 for gates order[oi_lo:oi_hi] over
 * windows [w_lo, w_hi) on the reference's own layout and argument list --
 * host arrays in and out, executed on the GPU (one thread per gate-window),
 * for code that drives the reference's per-level loop (simcore.py:295-325)
 * itself.  2-D arrays are row-major with the given column counts: stim_off /
 * stim_cnt [stim_rows, stim_cols], init_vals [num_nets, init_cols], g_* and
 * out_* [num_gates, g_cols] (column = window - w_off).  gbuf / g_cnt / out_*
 * are read and written back whole; out_err is only set (to 1).  Every index
 * the span follows is checked on the host first (GS_ERR_ARG). */
int gs_sim_span(int64_t oi_lo, int64_t oi_hi, int64_t w_lo, int64_t w_hi, int64_t w_off,
                const int64_t *order, int64_t num_gates, const int64_t *pin_off,
                const int64_t *pin_net, const int64_t *pin_ic, const int64_t *pin_arc,
                const int64_t *arc_rows, int64_t num_arc_rows, const int64_t *lut_off,
                const uint8_t *lut_bits, int64_t num_lut_bits, const int64_t *out_net,
                const uint8_t *net_kind, const int64_t *net_slot, int64_t num_nets,
                const int64_t *stim_buf, int64_t n_stim_buf, const int64_t *stim_off,
                const int64_t *stim_cnt, int64_t stim_rows, int64_t stim_cols,
                const uint8_t *init_vals, int64_t init_cols, const int64_t *boundaries,
                int64_t *gbuf, int64_t n_gbuf, const int64_t *g_off, const int64_t *g_cap,
                int64_t *g_cnt, int64_t g_cols, int64_t *out_filt, int64_t *out_icf,
                int64_t *out_disc, int64_t *out_err, int64_t *out_peak, int64_t pct);

/* init_values (_kernels.py:213-231): zero-delay window-start value of every
 * net; vals_out is [num_nets, W] uint8, rows < P copied from stim_init [P, W]. */
int gs_init_values(const gs_design_desc *desc, const uint8_t *stim_init, int64_t num_windows,
                   uint8_t *vals_out);

/* ---- stimulus document reader (host): the format immediately upstream of
 * the path ------------------------------------------------ */

/* parse_vcd (pkg/src/glsim/waveform.py:101-198): read a VCD document into
 * per-input CSR waveforms for the inputs named pi_names[0..num_pis) (the
 * netlist's primary inputs, in order) -- the form gs_stim_create takes.  On
 * GS_ERR_PARSE / GS_ERR_SEMANTIC gs_last_error() holds the reference's
 * message and gs_last_error_line() the 1-based line of a parse error.
 * GS_ERR_UNSUPPORTED (non-ASCII text, Unicode separators, time values beyond
 * int64): nothing was read; use the reference-semantics reader. */
int gs_vcd_parse(const char *text, int64_t len, const char *const *pi_names, int64_t num_pis,
                 gs_vcd **out);
/* sizes of a parsed document: total toggles and the last time mark (fs) */
int gs_vcd_sizes(const gs_vcd *v, int64_t *num_toggles, int64_t *duration);
/* copy out pi_off [num_pis+1], pi_times [num_toggles], pi_init [num_pis] */
int gs_vcd_copy(const gs_vcd *v, int64_t *pi_off, int64_t *pi_times, uint8_t *pi_init);
int gs_vcd_destroy(gs_vcd *v);
/* 1-based line of the last GS_ERR_PARSE (0 if none) */
int64_t gs_last_error_line(void);

/* parse_sdf (pkg/src/glsim/sdf.py:229-503): read an SDF document into the
 * flat delay arrays of the design -- arc_rows [R][2] (rise, fall per
 * condition row; gates in order, each gate's pins in order, 2^(k-1) rows per
 * pin: exactly gs_design_desc.arc_rows) and pin_ic [sum k] -- for the netlist
 * described below.  corner: 0 min, 1 typ, 2 max.  Skipped constructs produce
 * the reference's warnings (gs_sdf_warning).  Errors as gs_vcd_parse
 * (gs_last_error_line / gs_last_error_col for GS_ERR_PARSE). */
typedef struct gs_sdf_design {
  int64_t num_gates, num_nets, num_cells;
  const char *gate_names;  const int64_t *gate_name_off;   /* [G+1] byte offsets */
  const char *net_names;   const int64_t *net_name_off;    /* [N+1] */
  const char *pin_names;   const int64_t *pin_name_off;    /* all cells' input pin names */
  const int64_t *cell_pin_first;                           /* [C+1] into the pin names */
  const char *cell_outputs; const int64_t *cell_output_off; /* [C+1] */
  const int64_t *gate_cell;                                /* [G] */
  const int64_t *pin_off;                                  /* [G+1] */
  const int64_t *pin_net;                                  /* [sum k] */
  const int64_t *out_net;                                  /* [G] */
} gs_sdf_design;
typedef struct gs_sdf gs_sdf;
int gs_sdf_parse(const char *text, int64_t len, const gs_sdf_design *design, int corner,
                 const char *path, gs_sdf **out);
/* sizes: condition rows R, pins, the document's timescale (fs), warnings */
int gs_sdf_sizes(const gs_sdf *h, int64_t *num_rows, int64_t *num_pins, int64_t *timescale_fs,
                 int64_t *num_warnings);
int gs_sdf_copy(const gs_sdf *h, int64_t *arc_rows, int64_t *pin_ic);
const char *gs_sdf_warning(const gs_sdf *h, int64_t i);
int gs_sdf_destroy(gs_sdf *h);
/* 1-based column of the last GS_ERR_PARSE (0 if none) */
int64_t gs_last_error_col(void);

/* ---- activity report writer (host): the format immediately downstream of
 * the path ------------------------------------------------ */

/* write_saif (pkg/src/glsim/report.py:94-131): the byte-exact flat SAIF text
 * for num_nets nets.  Net names are UTF-8, concatenated in `names` with
 * name_off [num_nets+1] byte offsets; '[', ']', '/' and '\' are escaped with
 * a backslash.  t0/t1/tc/ig [num_nets] (ig only if include_ig).  Writes at
 * most out_cap bytes to `out` and the text length to *out_len; GS_ERR_ARG if
 * out_cap is too small (*out_len then holds the size needed). */
int gs_saif_format(const char *names, const int64_t *name_off, int64_t num_nets,
                   const int64_t *t0, const int64_t *t1, const int64_t *tc, const int64_t *ig,
                   int64_t duration, const char *design_name, const char *saif_version,
                   int include_ig, char *out, int64_t out_cap, int64_t *out_len);

/* VcdWriter / write_vcd (pkg/src/glsim/report.py:144-214): the byte-exact VCD
 * dump of simulated waveforms.  gs_vcdw_create writes the header for the
 * listed net names (UTF-8 in `names`, byte offsets name_off [num_names+1]);
 * each gs_vcdw_feed appends windows [w_lo, w_hi) of every listed net -- net i
 * is row net_row[i] of waveform source src[net_src[i]] (0: primary inputs,
 * 1: gates; windowed int64 arrays, absolute times) -- keeping each name's
 * last value across feeds; gs_vcdw_finish appends the end time.  The text
 * accumulates in the handle: gs_vcdw_take copies it out (buf NULL: size only)
 * and clears it. */
typedef struct gs_wave_src {
  const int64_t *buf;
  int64_t n_buf;
  const int64_t *offsets, *counts;  /* [rows, cols] */
  const uint8_t *initials;          /* [rows, cols] */
  int64_t cols;                     /* row pitch (windows) */
  int64_t col0;                     /* column of window w_lo */
} gs_wave_src;
typedef struct gs_vcdw gs_vcdw;
int gs_vcdw_create(const char *names, const int64_t *name_off, int64_t num_names,
                   const char *design_name, gs_vcdw **out);
int gs_vcdw_feed(gs_vcdw *w, const uint8_t *net_src, const int64_t *net_row,
                 const gs_wave_src *src, const int64_t *boundaries, int64_t w_lo, int64_t w_hi);
int gs_vcdw_finish(gs_vcdw *w, int64_t end_time);
int gs_vcdw_take(gs_vcdw *w, char *buf, int64_t cap, int64_t *len);
int gs_vcdw_destroy(gs_vcdw *w);

/* ---- netlist document reader (host): the format upstream of the design
 * upload ------------------------------------------- */

/* parse_netlist (pkg/src/glsim/netlist.py:190-275): the netlist JSON read
 * straight into flat arrays for the cell library given as flat names (cell
 * c: name, input pins pin_names[cell_pin_first[c] .. cell_pin_first[c+1]),
 * output pin).  Nets are interned as the reference does (inputs, then gate
 * i's output as net P + i).  GS_ERR_UNSUPPORTED for any document the
 * reference would reject (its own reader then raises the exact error). */
typedef struct gs_netlist gs_netlist;
int gs_netlist_parse(const char *text, int64_t len, const char *cell_names,
                     const int64_t *cell_name_off, int64_t num_cells, const char *pin_names,
                     const int64_t *pin_name_off, const int64_t *cell_pin_first,
                     const char *cell_outputs, const int64_t *cell_output_off, gs_netlist **out);
/* counts[4] = inputs, outputs, gates, pins; bytes[5] = UTF-8 bytes of the
 * design name, input names, output names, gate names, gate output net names */
int gs_netlist_sizes(const gs_netlist *h, int64_t *counts, int64_t *bytes);
/* names as byte blobs with [n+1] offsets; gate_cell [G], pin_off [G+1],
 * pin_net [pins] (any pointer may be NULL) */
int gs_netlist_copy(const gs_netlist *h, char *name, char *pis, int64_t *pis_off, char *pos,
                    int64_t *pos_off, char *gates, int64_t *gates_off, char *outs,
                    int64_t *outs_off, int64_t *gate_cell, int64_t *pin_off, int64_t *pin_net);
int gs_netlist_destroy(gs_netlist *h);

/* ---- multi-GPU: the merge of the per-net sums across window shards ----- */

/* The cross-GPU reduction of gs_run_stats_device accumulators (
 * ActivityStats.merge, pkg/src/glsim/report.py:46-54): an in-place NCCL
 * all-reduce (int64 sum) of acc_dev [n] on `stream` over `comm`, NVLink /
 * NVSwitch between the GPUs of a box.  Integer addition is associative, so
 * the merged sums -- and the SAIF -- are identical for any number of ranks.
 * libnccl.so.2 is bound at run time; the communicator comes from
 * gs_nccl_comm_create with an id made by gs_nccl_unique_id on one rank and
 * broadcast to the others (e.g. over torch.distributed). */
#define GS_NCCL_ID_BYTES 128
int gs_nccl_unique_id(uint8_t *id);
int gs_nccl_comm_create(const uint8_t *id, int nranks, int rank, int device, void **comm);
int gs_nccl_comm_destroy(void *comm);
int gs_allreduce_stats(int64_t *acc_dev, int64_t n, void *comm, void *stream);

#ifdef __cplusplus
}
#endif
#endif /* GLSIM_CUDA_H */
