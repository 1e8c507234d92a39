// glsim_cuda.cu -- host engine and C ABI of libglsim_cuda.so (see include/glsim_cuda.h).
//
// One engine per device.  A run walks its window range in chunks sized to the
// device memory budget; per chunk it launches K1 (stimulus segmentation) and
// then one K4 launch per logic level (the level barrier), all on one stream,
// and synchronizes once at the chunk end to check the device-side flags.
#include <algorithm>
#include <dlfcn.h>
#include <nccl.h>
#include <charconv>
#include <map>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "glsim_cuda.h"
#include "kernels.cuh"
#include "kernels_lean.cuh"
#include "synth.cuh"
#include "arena.cuh"
#include "vcd_reader.h"
#include "vcd_writer.h"
#include "netlist_reader.h"
#include "sdf_reader.h"

using namespace gs;

namespace {

thread_local std::string g_err;
thread_local int64_t g_err_line = 0, g_err_col = 0;

int fail(int code, const std::string &msg) {
  g_err = msg;
  g_err_line = g_err_col = 0;
  return code;
}

#define CK(call)                                                                        \
  do {                                                                                  \
    cudaError_t e_ = (call);                                                            \
    if (e_ != cudaSuccess) {                                                            \
      (void)cudaGetLastError();                                                         \
      return fail(e_ == cudaErrorMemoryAllocation ? GS_ERR_CAPACITY : GS_ERR_CUDA,      \
                  std::string(#call) + ": " + cudaGetErrorString(e_));                  \
    }                                                                                   \
  } while (0)

#define TRY(call)               \
  do {                                     \
    int rc_ = (call);                      \
    if (rc_ != GS_OK) return rc_;          \
  } while (0)

template <typename T>
int dalloc(T **p, size_t n) {
  *p = nullptr;
  if (n == 0) n = 1;
  const cudaError_t e = cudaMalloc((void **)p, n * sizeof(T));
  if (e != cudaSuccess) {
    (void)cudaGetLastError();
    size_t fr = 0, tot = 0;
    cudaMemGetInfo(&fr, &tot);
    return fail(e == cudaErrorMemoryAllocation ? GS_ERR_CAPACITY : GS_ERR_CUDA,
                std::string(cudaGetErrorString(e)) + " allocating " +
                    std::to_string(n * sizeof(T)) + " bytes (" + std::to_string(fr) +
                    " of " + std::to_string(tot) + " free)");
  }
  return GS_OK;
}

template <typename T>
void dfree(T *&p) {
  if (p) cudaFree((void *)p);
  p = nullptr;
}

template <typename T>
int upload(T **p, const T *src, size_t n) {
  TRY(dalloc(p, n));
  if (n) CK(cudaMemcpy(*p, src, n * sizeof(T), cudaMemcpyHostToDevice));
  return GS_OK;
}

// Stimulus buffers come from the device's stream-ordered pool, kept warm (no
// release to the OS at synchronisation), so a stimulus uploaded every step --
// the end-to-end path -- does not pay cudaMalloc / cudaFree each time.
int pool_ready(int dev) {
  static bool done[64] = {};
  if (dev < 0 || dev >= 64 || done[dev]) return GS_OK;
  cudaMemPool_t pool;
  CK(cudaDeviceGetDefaultMemPool(&pool, dev));
  unsigned long long thr = ~0ull;
  CK(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr));
  done[dev] = true;
  return GS_OK;
}

// The stimulus is uploaded, validated and freed on a per-device stream of
// its own (non-blocking), so a stimulus for the next step can be created from
// another host thread while an engine simulates the current one.
int upload_stream(int dev, cudaStream_t *us) {
  static cudaStream_t streams[64] = {};
  if (dev < 0 || dev >= 64) return fail(GS_ERR_ARG, "device index out of range");
  if (!streams[dev]) CK(cudaStreamCreateWithFlags(&streams[dev], cudaStreamNonBlocking));
  *us = streams[dev];
  return GS_OK;
}

template <typename T>
int upload_pooled(T **p, const T *src, size_t n, cudaStream_t us) {
  *p = nullptr;
  CK(cudaMallocAsync((void **)p, (n ? n : 1) * sizeof(T), us));
  if (n) CK(cudaMemcpyAsync(*p, src, n * sizeof(T), cudaMemcpyHostToDevice, us));
  return GS_OK;
}

template <typename T>
void dfree_pooled(T *&p, cudaStream_t us) {
  if (p) cudaFreeAsync((void *)p, us);
  p = nullptr;
}

// run a validation kernel that ORs flags into a device int; return the flags
// (synchronises the upload stream: the stimulus is complete on return)
template <typename F>
int device_check(int *flags, cudaStream_t us, F launch) {
  int *f = nullptr;
  CK(cudaMallocAsync((void **)&f, sizeof(int), us));
  cudaError_t e = cudaMemsetAsync(f, 0, sizeof(int), us);
  if (e == cudaSuccess) {
    launch(f);
    e = cudaGetLastError();
  }
  if (e == cudaSuccess) e = cudaMemcpyAsync(flags, f, sizeof(int), cudaMemcpyDeviceToHost, us);
  cudaFreeAsync(f, us);
  if (e == cudaSuccess) e = cudaStreamSynchronize(us);
  if (e != cudaSuccess) return fail(GS_ERR_CUDA, cudaGetErrorString(e));
  return GS_OK;
}

int use_device(int dev) {
  int n = 0;
  cudaError_t e = cudaGetDeviceCount(&n);
  if (e != cudaSuccess || n == 0) {
    (void)cudaGetLastError();
    return fail(GS_ERR_NODEVICE, "no CUDA device visible");
  }
  if (dev < 0 || dev >= n) return fail(GS_ERR_ARG, "device index out of range");
  CK(cudaSetDevice(dev));
  return GS_OK;
}

inline int64_t round_up(int64_t x, int64_t m) { return (x + m - 1) / m * m; }

}  // namespace

// =========================================================================
// design

struct gs_design {
  int device = 0;
  int P = 0, G = 0, N = 0, L = 0;
  std::vector<int64_t> level_starts;
  // per level, gates grouped by fanin count: group g in 0..3 holds k = g+1,
  // group 4 holds k > 4; grp[l*6 + g] .. grp[l*6 + g + 1] in device order
  std::vector<int64_t> grp;
  int64_t max_arc = 0, max_ic = 0;
  std::vector<int64_t> fanout;       // per net: input pins it drives
  std::vector<int> k_of;             // per gate
  int64_t sum_k = 0;
  int *order = nullptr, *gate_k = nullptr, *gate_pin = nullptr, *pin_net = nullptr,
      *pin_arc = nullptr;
  long long *pin_ic = nullptr, *arc = nullptr;
  unsigned *arc32 = nullptr;
  unsigned long long *gate_lut = nullptr;
  unsigned *lut_words = nullptr;
  int *order_ref = nullptr;          // the arena order (levelized order as given)
  std::vector<int> order_host;

  DesignDev dev() const {
    DesignDev D;
    D.P = P;
    D.G = G;
    D.N = N;
    D.order = order;
    D.gate_k = gate_k;
    D.gate_pin = gate_pin;
    D.gate_lut = gate_lut;
    D.lut_words = lut_words;
    D.pin_net = pin_net;
    D.pin_ic = pin_ic;
    D.pin_arc = pin_arc;
    D.arc = arc;
    D.arc32 = arc32;
    return D;
  }
  void release() {
    dfree(order); dfree(gate_k); dfree(gate_pin); dfree(pin_net); dfree(pin_arc);
    dfree(pin_ic); dfree(arc); dfree(arc32); dfree(gate_lut); dfree(lut_words);
    dfree(order_ref);
  }
};

static int design_build(const gs_design_desc *d, int device, gs_design *D) {
  if (!d) return fail(GS_ERR_ARG, "null design descriptor");
  const int64_t P = d->num_pis, G = d->num_gates, L = d->num_levels;
  if (P < 0 || G < 0 || L < 0 || P + G > INT32_MAX)
    return fail(GS_ERR_ARG, "design size out of range");
  if (G > 0 && (!d->order || !d->level_starts || !d->pin_off || !d->lut_off || !d->lut_bits))
    return fail(GS_ERR_ARG, "missing design arrays");
  D->device = device;
  D->P = (int)P;
  D->G = (int)G;
  D->N = (int)(P + G);
  D->L = (int)L;
  const int64_t N = P + G;
  // ---- validation (a bad index must never reach the device)
  std::vector<int> level_of(G, -1);
  D->level_starts.assign(d->level_starts, d->level_starts + (L + 1));
  if (D->level_starts[0] != 0 || D->level_starts[L] != G)
    return fail(GS_ERR_ARG, "level_starts must span [0, G]");
  for (int64_t l = 0; l < L; ++l) {
    if (D->level_starts[l + 1] < D->level_starts[l])
      return fail(GS_ERR_ARG, "level_starts not monotone");
    for (int64_t i = D->level_starts[l]; i < D->level_starts[l + 1]; ++i) {
      const int64_t g = d->order[i];
      if (g < 0 || g >= G || level_of[g] >= 0) return fail(GS_ERR_ARG, "order is not a permutation");
      level_of[g] = (int)l;
    }
  }
  if (G && d->pin_off[0] != 0) return fail(GS_ERR_ARG, "pin_off[0] must be 0");
  D->k_of.resize(G);
  D->fanout.assign(N, 0);
  int64_t n_pins = G ? d->pin_off[G] : 0;
  if (n_pins > INT32_MAX || d->num_arc_rows > INT32_MAX / 2)
    return fail(GS_ERR_ARG, "design too large for 32-bit pin/arc indices");
  for (int64_t g = 0; g < G; ++g) {
    const int64_t k = d->pin_off[g + 1] - d->pin_off[g];
    if (k < 1 || k > kMaxK) return fail(GS_ERR_ARG, "gate fanin count must be in [1, 16]");
    D->k_of[g] = (int)k;
    if (d->lut_off[g] < 0 || d->lut_off[g] + (int64_t(1) << k) > d->num_lut_bits)
      return fail(GS_ERR_ARG, "lut_off out of range");
    for (int64_t p = d->pin_off[g]; p < d->pin_off[g + 1]; ++p) {
      const int64_t n = d->pin_net[p];
      if (n < 0 || n >= N) return fail(GS_ERR_ARG, "pin_net out of range");
      if (n >= P && level_of[n - P] >= level_of[g])
        return fail(GS_ERR_ARG, "fanin is not on an earlier level");
      if (d->pin_ic[p] < 0) return fail(GS_ERR_ARG, "negative interconnect delay");
      D->max_ic = std::max<int64_t>(D->max_ic, d->pin_ic[p]);
      if (d->pin_arc[p] < 0 || d->pin_arc[p] + (int64_t(1) << (k - 1)) > d->num_arc_rows)
        return fail(GS_ERR_ARG, "pin_arc out of range");
      D->fanout[n] += 1;
    }
  }
  for (int64_t r = 0; r < 2 * d->num_arc_rows; ++r) {
    if (d->arc_rows[r] < 0) return fail(GS_ERR_ARG, "negative arc delay");
    D->max_arc = std::max<int64_t>(D->max_arc, d->arc_rows[r]);
  }
  D->sum_k = n_pins;

  // ---- device order: per level, gates grouped k = 1, 2, 3, 4, then k > 4
  // (one kernel instance per group keeps each hot loop small)
  std::vector<int> order(G);
  D->grp.assign((size_t)L * 6, 0);
  for (int64_t l = 0; l < L; ++l) {
    int64_t o = D->level_starts[l];
    for (int gi = 0; gi < 5; ++gi) {
      D->grp[l * 6 + gi] = o;
      for (int64_t i = D->level_starts[l]; i < D->level_starts[l + 1]; ++i) {
        const int64_t g = d->order[i];
        const int kg = std::min(D->k_of[g], 5) - 1;
        if (kg == gi) order[o++] = (int)g;
      }
    }
    D->grp[l * 6 + 5] = o;
  }
  std::vector<int> gate_pin(G);
  std::vector<unsigned long long> gate_lut(G);
  std::vector<unsigned> words;
  for (int64_t g = 0; g < G; ++g) {
    const int k = D->k_of[g];
    gate_pin[g] = (int)d->pin_off[g];
    const uint8_t *t = d->lut_bits + d->lut_off[g];
    if (k <= 6) {
      unsigned long long m = 0;
      for (int i = 0; i < (1 << k); ++i) m |= (unsigned long long)(t[i] & 1u) << i;
      gate_lut[g] = m;
    } else {
      gate_lut[g] = words.size();
      const int nw = (1 << k) / 32;
      for (int w = 0; w < nw; ++w) {
        unsigned m = 0;
        for (int b = 0; b < 32; ++b) m |= (unsigned)(t[w * 32 + b] & 1u) << b;
        words.push_back(m);
      }
    }
  }
  std::vector<int> pin_net(n_pins), pin_arc(n_pins);
  for (int64_t p = 0; p < n_pins; ++p) {
    pin_net[p] = (int)d->pin_net[p];
    pin_arc[p] = (int)d->pin_arc[p];
  }
  TRY(use_device(device));
  TRY(upload(&D->order, order.data(), G));
  D->order_host.assign(d->order, d->order + G);
  TRY(upload(&D->order_ref, D->order_host.data(), G));
  TRY(upload(&D->gate_k, D->k_of.data(), G));
  TRY(upload(&D->gate_pin, gate_pin.data(), G));
  TRY(upload(&D->gate_lut, gate_lut.data(), G));
  TRY(upload(&D->lut_words, words.data(), words.size()));
  TRY(upload(&D->pin_net, pin_net.data(), n_pins));
  TRY(upload(&D->pin_arc, pin_arc.data(), n_pins));
  TRY(upload(&D->pin_ic, (const long long *)d->pin_ic, n_pins));
  TRY(upload(&D->arc, (const long long *)d->arc_rows, 2 * d->num_arc_rows));
  if (D->max_arc < (int64_t(1) << 31) && D->max_ic < (int64_t(1) << 31)) {
    std::vector<unsigned> a32(2 * d->num_arc_rows);
    for (int64_t r = 0; r < 2 * d->num_arc_rows; ++r) a32[r] = (unsigned)d->arc_rows[r];
    TRY(upload(&D->arc32, a32.data(), a32.size()));
  }
  return GS_OK;
}

// =========================================================================
// stimulus

struct gs_stim {
  gs_design *d = nullptr;
  int P = 0;
  int64_t W = 0;
  bool csr = true, wide = false;
  int64_t max_wlen = 0;
  std::vector<int64_t> bnd_host;
  int64_t n_toggles = 0;
  long long *bnd = nullptr, *pi_off = nullptr, *pi_times = nullptr, *buf = nullptr,
            *offsets = nullptr, *counts = nullptr;
  unsigned char *pi_init = nullptr, *initials = nullptr;

  StimDev dev() const {
    StimDev S;
    S.P = P;
    S.W = W;
    S.pi_off = pi_off;
    S.pi_times = pi_times;
    S.pi_init = pi_init;
    S.buf = buf;
    S.offsets = offsets;
    S.counts = counts;
    S.nbuf = n_toggles;
    S.initials = initials;
    return S;
  }
  cudaStream_t us = nullptr;  // upload stream of the device
  void release() {
    // engine runs are synchronous: no engine work reads the stimulus once a
    // run call has returned, so the buffers go back to the pool in order
    // behind the upload stream's own work
    dfree_pooled(bnd, us); dfree_pooled(pi_off, us); dfree_pooled(pi_times, us);
    dfree_pooled(buf, us); dfree_pooled(offsets, us); dfree_pooled(counts, us);
    dfree_pooled(pi_init, us); dfree_pooled(initials, us);
  }
};

static int stim_build(gs_design *D, const gs_stim_desc *s, gs_stim *S) {
  if (!s || !s->boundaries) return fail(GS_ERR_ARG, "null stimulus descriptor");
  if (s->num_pis != D->P) return fail(GS_ERR_ARG, "stimulus input count != design inputs");
  if (s->num_windows < 1) return fail(GS_ERR_ARG, "need at least one window");
  S->d = D;
  S->P = (int)s->num_pis;
  S->W = s->num_windows;
  S->bnd_host.assign(s->boundaries, s->boundaries + s->num_windows + 1);
  int64_t maxlen = 0;
  for (int64_t w = 0; w < S->W; ++w) {
    const int64_t len = S->bnd_host[w + 1] - S->bnd_host[w];
    if (len <= 0) return fail(GS_ERR_ARG, "window boundaries must be strictly ascending");
    maxlen = std::max(maxlen, len);
  }
  S->wide = maxlen > (int64_t)0xFFFFFFFFll;
  S->max_wlen = maxlen;
  S->csr = s->pi_off != nullptr;
  TRY(use_device(D->device));
  TRY(pool_ready(D->device));
  TRY(upload_stream(D->device, &S->us));
  cudaStream_t us = S->us;
  TRY(upload_pooled(&S->bnd, (const long long *)s->boundaries, S->W + 1, us));
  const int64_t P = S->P, W = S->W;
  if (S->csr) {
    if (!s->pi_times || !s->pi_init) return fail(GS_ERR_ARG, "incomplete CSR stimulus");
    if (s->pi_off[0] != 0) return fail(GS_ERR_ARG, "pi_off[0] must be 0");
    for (int64_t p = 0; p < P; ++p)
      if (s->pi_off[p + 1] < s->pi_off[p]) return fail(GS_ERR_ARG, "pi_off not monotone");
    S->n_toggles = s->pi_off[P];
    TRY(upload_pooled(&S->pi_off, (const long long *)s->pi_off, P + 1, us));
    TRY(upload_pooled(&S->pi_times, (const long long *)s->pi_times, S->n_toggles, us));
    TRY(upload_pooled(&S->pi_init, s->pi_init, P, us));
    int bad = 0;
    TRY(device_check(&bad, us, [&](int *flag) {
      stim_check_csr<<<std::max<int64_t>(1, std::min<int64_t>((P + 7) / 8, 4096)), 256, 0, us>>>(
          S->pi_off, S->pi_times, (int)P, flag);
    }));
    if (bad) return fail(GS_ERR_ARG, "input toggle times must be strictly increasing");
  } else {
    if (!s->buf && s->n_buf) return fail(GS_ERR_ARG, "missing stimulus buffer");
    if (!s->offsets || !s->counts || !s->initials) return fail(GS_ERR_ARG, "incomplete windowed stimulus");
    S->n_toggles = s->n_buf;
    TRY(upload_pooled(&S->buf, (const long long *)s->buf, s->n_buf, us));
    TRY(upload_pooled(&S->offsets, (const long long *)s->offsets, P * W, us));
    TRY(upload_pooled(&S->counts, (const long long *)s->counts, P * W, us));
    TRY(upload_pooled(&S->initials, s->initials, P * W, us));
    int bad = 0;
    TRY(device_check(&bad, us, [&](int *flag) {
      stim_check_win<<<(int)std::max<int64_t>(1, std::min<int64_t>((P * W + 255) / 256, 4096)),
                       256, 0, us>>>(S->buf, s->n_buf, S->offsets, S->counts, S->bnd, W, P * W,
                                     flag);
    }));
    if (bad & BAD_REGION) return fail(GS_ERR_ARG, "stimulus window region out of range");
    if (bad) return fail(GS_ERR_ARG, "stimulus toggle outside its window or not increasing");
  }
  return GS_OK;
}

// =========================================================================
// engine

struct gs_engine {
  gs_design *d = nullptr;
  cudaStream_t st = nullptr;
  bool own_stream = false;
  int sms = 0;
  int64_t budget = 0;
  // chunk workspace
  int64_t meta_windows = 0;          // capacity (windows, multiple of 32)
  unsigned *cnt = nullptr;
  unsigned long long *tbase = nullptr;
  unsigned *init = nullptr;
  unsigned *wlen32 = nullptr;
  void *data = nullptr;
  int64_t data_bytes = 0;
  int64_t pool_bytes = 0;            // requested gate-pool bytes
  int ncta_cap = 0;
  unsigned long long *bump = nullptr;
  unsigned *work = nullptr;
  int work_cap = 0;
  long long *acc = nullptr, *acc_run = nullptr;
  int *err = nullptr, *err_host = nullptr;
  unsigned long long *bump_host = nullptr;
  // arena workspace
  int64_t arena_windows = 0;
  long long *a_cnt = nullptr, *a_peak = nullptr, *a_filt = nullptr, *a_icf = nullptr,
            *a_disc = nullptr, *a_off = nullptr, *a_buf = nullptr, *a_capd = nullptr;
  unsigned char *a_init = nullptr;
  unsigned long long *a_pos = nullptr;
  int64_t a_buf_cap = 0;
  // K5: the last count pass's packed arena pieces, one per window chunk
  struct ArenaPiece {
    int64_t w0, wc;
    std::vector<int64_t> rs;      // [G] entries per gate in the chunk
    std::vector<int64_t> piece;   // gate-major (arena order), absolute times
  };
  std::vector<ArenaPiece> kept;
  // one CUDA graph per distinct chunk launch sequence (K1 + every level's K4
  // launches + the chunk's resets and events), keyed by the exact launch
  // parameters; a replay skips the per-launch host cost and the gaps
  struct ChunkGraph {
    cudaGraphExec_t exec = nullptr;
    int k1 = 0, nl = 0;
  };
  std::map<std::string, ChunkGraph> graphs;
  int64_t graph_hits = 0, graph_builds = 0;
  void drop_graphs() {
    for (auto &kv : graphs)
      if (kv.second.exec) cudaGraphExecDestroy(kv.second.exec);
    graphs.clear();
  }
  const gs_stim *kept_stim = nullptr;
  int64_t kept_lo = 0, kept_hi = 0;
  int kept_pct = -1;
  long long *k5_rs = nullptr, *k5_base = nullptr, *k5_part = nullptr, *k5_out = nullptr;
  int64_t k5_out_cap = 0;
  cudaEvent_t ev[4] = {nullptr, nullptr, nullptr, nullptr};
  int64_t chunk_hint[2] = {0, 0};   // per mode family: stats, arena
  // work-item sizing (gs_engine_set_items): workers assumed (0 = the grid),
  // tail re-cut divisor (1 = none), tail share limit
  int64_t item_workers = 0;
  int tail_div = 2, tail_frac = 2;
  gs_timing last{};

  void release_meta() { dfree(cnt); dfree(tbase); dfree(init); dfree(wlen32); meta_windows = 0; }
  void release_arena() {
    dfree(a_cnt); dfree(a_peak); dfree(a_filt); dfree(a_icf); dfree(a_disc); dfree(a_off);
    dfree(a_capd);
    dfree(a_init); dfree(a_pos); arena_windows = 0;
  }
  void release() {
    release_meta();
    release_arena();
    dfree(a_buf);
    dfree(k5_rs); dfree(k5_base); dfree(k5_part); dfree(k5_out);
    dfree(data);
    dfree(bump);
    dfree(work);
    dfree(acc);
    dfree(acc_run);
    dfree(err);
    if (err_host) cudaFreeHost(err_host);
    if (bump_host) cudaFreeHost(bump_host);
    err_host = nullptr;
    bump_host = nullptr;
    for (auto &e : ev)
      if (e) cudaEventDestroy(e), e = nullptr;
    drop_graphs();
    if (own_stream && st) cudaStreamDestroy(st);
    st = nullptr;
  }
};

namespace {

// Per gate_eval instantiation: opt in to its dynamic shared memory (per-warp
// tile state, above the 48 KB static limit) and size its persistent grid from
// its own occupancy.  The opt-in is a per-device function attribute, so it is
// cached per device.  Output regions are indexed by (CTA, warp), so every
// launch of a chunk shares the region array sized by the largest grid.
constexpr int kMaxDevices = 64;

template <typename F>
int kernel_grid(F kernel, size_t smem, int sms, int *cache, int *grid,
                int threads = kEvalThreads) {
  int dev = 0;
  CK(cudaGetDevice(&dev));
  if (dev < 0 || dev >= kMaxDevices) return fail(GS_ERR_ARG, "device index out of range");
  if (!cache[dev]) {
    CK(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    int occ = 0;
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kernel, threads, smem));
    cache[dev] = std::max(1, occ);
  }
  *grid = sms * cache[dev];
  return GS_OK;
}

template <typename TS, typename TT, int MODE, int K, bool P100>
int eval_grid(int sms, int *grid) {
  static int cache[kMaxDevices] = {};
  return kernel_grid(gate_eval<TS, TT, MODE, K, P100>, eval_smem_bytes<TS, TT, K>(), sms, cache,
                     grid);
}

template <int MODE, int K, bool P100>
int lean_grid(int sms, int *grid) {
  static int cache[kMaxDevices] = {};
  return kernel_grid(gate_eval_lean<MODE, K, P100>, lean_smem_bytes<K>(), sms, cache, grid,
                     kLeanThreads);
}

template <typename TS, typename TT, int MODE, int K, bool P100>
int launch_eval(int sms, cudaStream_t st, const DesignDev &Dd, const ChunkDev &C,
                const LevelArgs &A, int max_grid) {
  int grid = 0;
  TRY((eval_grid<TS, TT, MODE, K, P100>(sms, &grid)));
  grid = std::min(grid, max_grid);
  gate_eval<TS, TT, MODE, K, P100><<<grid, kEvalThreads, eval_smem_bytes<TS, TT, K>(), st>>>(Dd, C, A);
  CK(cudaGetLastError());
  return GS_OK;
}

template <int MODE, int K, bool P100>
int launch_lean(int sms, cudaStream_t st, const DesignDev &Dd, const ChunkDev &C,
                const LevelArgs &A, int max_grid) {
  int grid = 0;
  TRY((lean_grid<MODE, K, P100>(sms, &grid)));
  grid = std::min(grid, max_grid);
  gate_eval_lean<MODE, K, P100><<<grid, kLeanThreads, lean_smem_bytes<K>(), st>>>(Dd, C, A);
  CK(cudaGetLastError());
  return GS_OK;
}

#ifndef GS_META_PCT
#define GS_META_PCT 40  // share of the device budget for chunk metadata (dev A/B knob)
#endif

// largest persistent grid any kernel of a run may use (sizes the regions)
template <typename TS, int MODE>
int grid_size(gs_engine *e, bool narrow, bool p100, int *ncta) {
  int g = 0, best = 0;
  if (narrow && p100) {
    TRY((lean_grid<MODE, 1, true>(e->sms, &g))); best = std::max(best, g);
    TRY((lean_grid<MODE, 2, true>(e->sms, &g))); best = std::max(best, g);
    TRY((lean_grid<MODE, 3, true>(e->sms, &g))); best = std::max(best, g);
    TRY((lean_grid<MODE, 4, true>(e->sms, &g))); best = std::max(best, g);
  } else if (narrow) {
    TRY((lean_grid<MODE, 1, false>(e->sms, &g))); best = std::max(best, g);
    TRY((lean_grid<MODE, 2, false>(e->sms, &g))); best = std::max(best, g);
    TRY((lean_grid<MODE, 3, false>(e->sms, &g))); best = std::max(best, g);
    TRY((lean_grid<MODE, 4, false>(e->sms, &g))); best = std::max(best, g);
  }
  TRY((eval_grid<TS, long long, MODE, 0, false>(e->sms, &g))); best = std::max(best, g);
  int o = 0;
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, stim_segment_win<TS>, kEvalThreads, 0));
  best = std::max(best, e->sms * std::max(1, o));
  *ncta = best;
  return GS_OK;
}

// ensure per-chunk metadata arrays hold `wins` windows
int ensure_meta(gs_engine *e, int64_t wins) {
  if (e->meta_windows >= wins) return GS_OK;
  e->release_meta();
  const int64_t N = e->d->N;
  const int64_t Wpad = round_up(wins, kTile);
  TRY(dalloc(&e->cnt, (size_t)(N * Wpad)));
  TRY(dalloc(&e->tbase, (size_t)(N * (Wpad / kTile)) + 2));  // +2: aligned 16-byte prefetch pieces
  TRY(dalloc(&e->init, (size_t)(N * (Wpad / 32))));
  TRY(dalloc(&e->wlen32, (size_t)Wpad));
  e->meta_windows = Wpad;
  return GS_OK;
}

int ensure_arena(gs_engine *e, int64_t wins, bool store) {
  if (e->arena_windows >= wins && (!store || e->a_off)) return GS_OK;
  e->release_arena();
  const size_t n = (size_t)e->d->G * (size_t)round_up(wins, kTile);
  TRY(dalloc(&e->a_cnt, n));
  TRY(dalloc(&e->a_peak, n));
  TRY(dalloc(&e->a_filt, n));
  TRY(dalloc(&e->a_icf, n));
  TRY(dalloc(&e->a_disc, n));
  TRY(dalloc(&e->a_init, n));
  TRY(dalloc(&e->a_off, n));
  TRY(dalloc(&e->a_capd, n));
  TRY(dalloc(&e->a_pos, n));
  e->arena_windows = round_up(wins, kTile);
  return GS_OK;
}

int ensure_data(gs_engine *e, int64_t bytes) {
  if (e->data_bytes >= bytes) return GS_OK;
  dfree(e->data);
  e->data_bytes = 0;
  // 64 bytes of slack: bulk copies of a segment round its end up to 16 bytes
  CK(cudaMalloc(&e->data, (size_t)bytes + 64));
  e->data_bytes = bytes;
  return GS_OK;
}

int64_t meta_bytes_per_window(const gs_design *d, bool arena) {
  // cnt (4 B), tbase (8 B per 128-window tile), init bits (4 B per 32
  // windows) per net-window, plus the window length
  int64_t b = (int64_t)d->N * 4 + ((int64_t)d->N * 8 + kTile - 1) / kTile +
              ((int64_t)d->N * 4 + 31) / 32 + 4;
  if (arena) b += (int64_t)d->G * (6 * 8 + 1);
  return b;
}

// Work-item sizing of a K4 launch over n gates x `units` column units
// (tiles or super-tiles): head items of tpi units -- enough items for dynamic
// balance over `workers` (4 per worker), few enough that per-item setup and
// work-counter atomics stay negligible (at most `cap` units) -- then, where
// the column-aligned tail stays within 1 / tail_frac of the units, about one
// head item per worker re-cut into items of tpi / tail_div units, so the
// workers of a launch finish close together (guided self-scheduling;
// profiles/ab_tail.sh, round 1: C2 -3.0 %, C3 -0.7 %).
constexpr int kItemCap = 12;   // tiles per item (profiles/ab_items_r01.log)
constexpr int kItemDiv = 4;
#ifndef GS_LEAN_ITEM_CAP
#define GS_LEAN_ITEM_CAP 8  // (dev A/B knob)
#endif
constexpr int kLeanItemCap = GS_LEAN_ITEM_CAP;  // super-tiles (of 4 tiles) per item of the lean kernels

struct ItemPlan {
  int tpi, ntg, tpi2, ntg2;
};

ItemPlan plan_items(int64_t n, int units, int64_t workers, int cap, int tail_div, int tail_frac) {
  ItemPlan P;
  workers = std::max<int64_t>(1, workers);
  cap = std::max(1, cap);
  P.tpi = (int)std::max<int64_t>(1, std::min<int64_t>(cap, n * units / (kItemDiv * workers)));
  P.tpi = std::min(P.tpi, std::max(1, units));
  while (n * ((units + P.tpi - 1) / P.tpi) >= (int64_t(1) << 31)) P.tpi *= 2;
  P.ntg = (units + P.tpi - 1) / P.tpi;
  P.tpi2 = std::max(1, P.tpi / std::max(1, tail_div));
  P.ntg2 = 0;
  if (tail_div > 1 && P.tpi > 1 && P.ntg > 1) {
    const int64_t need = std::min<int64_t>((int64_t)(P.ntg - 1) * P.tpi,
                                           (workers * P.tpi + n - 1) / n);
    const int hg = (int)((units - need) / P.tpi);  // head groups (whole)
    if ((int64_t)(units - hg * P.tpi) * std::max(1, tail_frac) <= units) {
      P.ntg2 = (units - hg * P.tpi + P.tpi2 - 1) / P.tpi2;
      P.ntg = hg;
    }
    if (n * (P.ntg + P.ntg2) >= (int64_t(1) << 31)) {
      P.ntg = (units + P.tpi - 1) / P.tpi;
      P.ntg2 = 0;
    }
  }
  return P;
}

struct RunOut {
  long long *acc_dev;       // [3N+3] device accumulators results are added to
  gs_arena_out *arena;      // may be null
  int64_t w_base;           // first window of the arena's column range
  int64_t arena_cols;       // Ws (host row pitch)
  CompareDev *cmp = nullptr;  // device cross-check against a reference arena (K7)
};

// K5: the chunk's gate waveforms (peak entries per window, as the count pass
// left them in the pool) packed gate-major in arena order, absolute int64,
// and kept on the host with the per-gate entry counts for gs_arena_fill.
template <typename TS>
int k5_pack(gs_engine *e, const ChunkDev &C, int64_t w0, int64_t wc) {
  gs_design *D = e->d;
  const int G = D->G;
  gs_engine::ArenaPiece pc;
  pc.w0 = w0;
  pc.wc = wc;
  pc.rs.assign(G, 0);
  if (G > 0) {
    const int nb = (G + kScanBlock - 1) / kScanBlock;
    if (!e->k5_rs) {
      TRY(dalloc(&e->k5_rs, (size_t)G));
      TRY(dalloc(&e->k5_base, (size_t)G));
      TRY(dalloc(&e->k5_part, (size_t)nb + 1));
    }
    const int blocks = (int)std::min<int64_t>((G + 7) / 8, (int64_t)e->sms * 16);
    arena_rowsum<<<blocks, 256, 0, e->st>>>(C.a_peak, G, C.Wc, C.Wpad, e->k5_rs);
    scan_blocks<<<nb, kScanThreads, 0, e->st>>>(e->k5_rs, D->order_ref, G, e->k5_base, e->k5_part);
    scan_parts<<<1, 1024, 0, e->st>>>(e->k5_part, nb);
    scan_add<<<nb, kScanThreads, 0, e->st>>>(e->k5_base, D->order_ref, G, e->k5_part);
    CK(cudaGetLastError());
    long long total = 0;
    CK(cudaMemcpyAsync(&total, e->k5_part + nb, sizeof(long long), cudaMemcpyDeviceToHost, e->st));
    CK(cudaMemcpyAsync(pc.rs.data(), e->k5_rs, sizeof(long long) * G, cudaMemcpyDeviceToHost, e->st));
    CK(cudaStreamSynchronize(e->st));
    if (total > e->k5_out_cap) {
      dfree(e->k5_out);
      e->k5_out_cap = 0;
      TRY(dalloc(&e->k5_out, (size_t)total));
      e->k5_out_cap = total;
    }
    if (total) {
      arena_pack<TS><<<blocks, 256, 0, e->st>>>(C, G, e->k5_base, e->k5_out);
      CK(cudaGetLastError());
      pc.piece.resize((size_t)total);
      CK(cudaMemcpyAsync(pc.piece.data(), e->k5_out, sizeof(long long) * total,
                         cudaMemcpyDeviceToHost, e->st));
      CK(cudaStreamSynchronize(e->st));
    }
  }
  e->kept.push_back(std::move(pc));
  return GS_OK;
}

template <typename TS, int MODE>
int run_chunks(gs_engine *e, gs_stim *s, int64_t w_lo, int64_t w_hi, int pct, RunOut &ro) {
  gs_design *D = e->d;
  const int64_t N = D->N, G = D->G;
  const bool arena = MODE != MODE_STATS;
  const bool store = MODE == MODE_STORE;
  // 32-bit time arithmetic when every sum the event loop forms stays below
  // 2^32-1: relative time < window length, plus interconnect, plus arc delay
  const bool narrow = sizeof(TS) == 4 && D->arc32 != nullptr &&
                      s->max_wlen + D->max_ic + D->max_arc <= (int64_t)0xFFFFFFFEll;
  const bool p100 = pct == 100;
  int ncta = 0;
  TRY((grid_size<TS, MODE>(e, narrow, p100, &ncta)));
  const int nregions = ncta * std::max(kEvalWarps, kLeanWarps);
  if (nregions > e->ncta_cap) {
    dfree(e->bump);
    TRY(dalloc(&e->bump, 2 * (size_t)nregions + 1));  // slot states + block counter
    e->ncta_cap = nregions;
  }
  if (e->work_cap < D->L * 5 + 1) {
    dfree(e->work);
    TRY(dalloc(&e->work, (size_t)D->L * 5 + 1));
    e->work_cap = D->L * 5 + 1;
  }
  const int64_t per_win = meta_bytes_per_window(D, arena);
  const int64_t pi_words = s->csr ? s->n_toggles : 0;
  const int64_t pi_bytes = round_up(pi_words * (int64_t)sizeof(TS), 256);
  const int64_t total = w_hi - w_lo;
  // initial chunk: metadata takes at most GS_META_PCT % of the budget (the
  // hint of the last run of the same mode family may be smaller, never larger)
  const int64_t meta_cap =
      std::max<int64_t>(kTile, (e->budget / 100 * GS_META_PCT) / per_win / kTile * kTile);
  int64_t &hint = e->chunk_hint[arena ? 1 : 0];
  int64_t Wc = hint > 0 ? std::min(hint, meta_cap) : meta_cap;
  Wc = std::min<int64_t>(Wc, round_up(total, kTile));
  Wc = std::max<int64_t>(kTile, Wc / kTile * kTile);
  const double density = (s->P && s->W) ? (double)s->n_toggles / ((double)s->P * s->W) : 0.0;

  if (store) {
    if (ro.arena->n_buf > e->a_buf_cap) {
      dfree(e->a_buf);
      e->a_buf_cap = 0;
      TRY(dalloc(&e->a_buf, (size_t)ro.arena->n_buf));
      e->a_buf_cap = ro.arena->n_buf;
    }
  }

  const DesignDev Dd = D->dev();
  const StimDev Sd = s->dev();
  int64_t w = w_lo;
  float ms_stim = 0.f, ms_eval = 0.f, ms_total = 0.f;
  int64_t launches = 0, eval_launches = 0, chunks = 0, peak_bytes = 0;
  int64_t pool_bytes = e->pool_bytes;
  while (w < w_hi) {
    const int64_t wc = std::min<int64_t>(Wc, w_hi - w);
    const int64_t Wpad = round_up(wc, kTile);
    const int Tc = (int)(Wpad / kTile);
    // room for the gate pool once this chunk's metadata is allocated: halve
    // the chunk (before allocating anything) while it does not fit
    const int64_t meta_now = per_win * Wpad;
    int64_t room = e->budget - meta_now - pi_bytes;
    if (room < (int64_t)nregions * 4096) {
      if (Wc > kTile) { Wc = std::max<int64_t>(kTile, Wc / 2 / kTile * kTile); continue; }
      return fail(GS_ERR_CAPACITY, "device memory budget cannot hold one 128-window chunk");
    }
    TRY(ensure_meta(e, Wpad));
    if (arena) TRY(ensure_arena(e, Wpad, store));
    const double est_words = (double)G * wc * std::max(2.0, 4.0 * density) * 2.0;
    int64_t want = std::max<int64_t>(pool_bytes, std::max<int64_t>(64ll << 20,
                                     (int64_t)(est_words * sizeof(TS))));
    want = std::min(want, room);
    TRY(ensure_data(e, pi_bytes + want));
    const int64_t pool_words = (e->data_bytes - pi_bytes) / (int64_t)sizeof(TS);
    // blocks: small enough that the partially used block of every slot wastes
    // at most ~1/4 of the pool, large enough that block grabs stay rare
    const int64_t block_words =
        std::max<int64_t>(256, std::min<int64_t>(1 << 16, pool_words / (4 * (int64_t)nregions)));

    ChunkDev C;
    memset(&C, 0, sizeof(C));
    C.N = (int)N;
    C.Wc = (int)wc;
    C.Tc = Tc;
    C.Wpad = (int)Wpad;
    C.w0 = w;
    C.bnd = s->bnd;
    C.cnt = e->cnt;
    C.tbase = e->tbase;
    C.init = e->init;
    C.wlen32 = e->wlen32;
    C.data = e->data;
    C.pool_base = (unsigned long long)(pi_bytes / (int64_t)sizeof(TS));
    C.block_words = (unsigned long long)block_words;
    C.pool_blocks = (unsigned long long)(pool_words / block_words);
    C.bump = e->bump;
    C.blk_next = e->bump + 2 * (size_t)nregions;
    C.work = e->work;
    C.acc = e->acc;
    C.err = e->err;
    if (arena) {
      C.a_cnt = e->a_cnt;
      C.a_peak = e->a_peak;
      C.a_filt = e->a_filt;
      C.a_icf = e->a_icf;
      C.a_disc = e->a_disc;
      C.a_init = e->a_init;
      C.a_off = e->a_off;
      C.a_cap = (store && ro.arena->caps) ? e->a_capd : nullptr;
      C.a_buf = e->a_buf;
      C.a_nbuf = store ? ro.arena->n_buf : 0;
      C.a_pos = e->a_pos;
      if (store) {
        CK(cudaMemcpy2DAsync(e->a_off, Wpad * 8, ro.arena->offsets + (w - ro.w_base),
                             ro.arena_cols * 8, wc * 8, G, cudaMemcpyHostToDevice, e->st));
        if (ro.arena->caps)
          CK(cudaMemcpy2DAsync(e->a_capd, Wpad * 8, ro.arena->caps + (w - ro.w_base),
                               ro.arena_cols * 8, wc * 8, G, cudaMemcpyHostToDevice, e->st));
      }
    }
    int k1 = 0, nl = 0;
    auto enqueue = [&]() -> int {
      CK(cudaMemsetAsync(e->acc, 0, sizeof(long long) * ACC_ROWS * N, e->st));
      CK(cudaMemsetAsync(e->bump, 0, sizeof(unsigned long long) * (2 * (size_t)nregions + 1), e->st));
      CK(cudaMemsetAsync(e->work, 0, sizeof(unsigned) * (D->L * 5 + 1), e->st));
      CK(cudaMemsetAsync(e->err, 0, sizeof(int) * ERR_NFLAGS, e->st));
      CK(cudaEventRecordWithFlags(e->ev[0], e->st, cudaEventRecordExternal));
      if (narrow) {
        chunk_windows<<<(int)((Wpad + 255) / 256), 256, 0, e->st>>>(C);
        CK(cudaGetLastError());
      }
      // ---- K1
      if (s->P > 0) {
        // tiles per item: the CSR kernel searches once per item and carries
        // the cut from tile to tile
        const int tpi = std::max(1, std::min(Tc, s->csr ? 16 : 4));
        const int ntg = (Tc + tpi - 1) / tpi;
        const int64_t items = (int64_t)s->P * ntg;
        if (s->csr) {
          const int blocks = (int)std::min<int64_t>((items + 7) / 8, (int64_t)e->sms * 16);
          stim_segment_csr<TS><<<blocks, 256, 0, e->st>>>(Sd, C, tpi, ntg);
        } else {
          stim_segment_win<TS><<<ncta, kEvalThreads, 0, e->st>>>(Sd, C, tpi, ntg);
        }
        CK(cudaGetLastError());
        k1 = 1;
      }
      CK(cudaEventRecordWithFlags(e->ev[1], e->st, cudaEventRecordExternal));
      // ---- K4: per level, one launch per fanin-count group (the launch
      // boundary between levels is the level barrier)
      const int STc = (Tc + kSuper - 1) / kSuper;
      for (int l = 0; l < D->L; ++l) {
        for (int gi = 0; gi < 5; ++gi) {
          const int lo = (int)D->grp[l * 6 + gi];
          const int n = (int)(D->grp[l * 6 + gi + 1] - lo);
          if (n <= 0) continue;
          const bool lean = narrow && gi < 4;
          LevelArgs A;
          A.lo = lo;
          A.n = n;
          // work items: (gate, run of tiles) for the generic kernel, (gate, run
          // of 4-tile super-tiles) for the lean kernels, whose CTA is the worker
          const ItemPlan ip = plan_items(n, lean ? STc : Tc,
                                         e->item_workers > 0 ? e->item_workers
                                                             : (lean ? ncta : nregions),
                                         lean ? kLeanItemCap : kItemCap, e->tail_div,
                                         e->tail_frac);
          A.tpi = ip.tpi;
          A.ntg = ip.ntg;
          A.tpi2 = ip.tpi2;
          A.ntg2 = ip.ntg2;
          A.pct = pct;
          A.counter = l * 5 + gi;
          const int sm = e->sms;
          if (narrow && p100 && gi < 4) {
            if (gi == 0) TRY((launch_lean<MODE, 1, true>(sm, e->st, Dd, C, A, ncta)));
            if (gi == 1) TRY((launch_lean<MODE, 2, true>(sm, e->st, Dd, C, A, ncta)));
            if (gi == 2) TRY((launch_lean<MODE, 3, true>(sm, e->st, Dd, C, A, ncta)));
            if (gi == 3) TRY((launch_lean<MODE, 4, true>(sm, e->st, Dd, C, A, ncta)));
          } else if (narrow && gi < 4) {
            if (gi == 0) TRY((launch_lean<MODE, 1, false>(sm, e->st, Dd, C, A, ncta)));
            if (gi == 1) TRY((launch_lean<MODE, 2, false>(sm, e->st, Dd, C, A, ncta)));
            if (gi == 2) TRY((launch_lean<MODE, 3, false>(sm, e->st, Dd, C, A, ncta)));
            if (gi == 3) TRY((launch_lean<MODE, 4, false>(sm, e->st, Dd, C, A, ncta)));
          } else {
            TRY((launch_eval<TS, long long, MODE, 0, false>(sm, e->st, Dd, C, A, ncta)));
          }
          ++nl;
        }
      }
      CK(cudaEventRecordWithFlags(e->ev[2], e->st, cudaEventRecordExternal));
      return GS_OK;
    };
    {
      // the chunk's launch sequence as a CUDA graph, cached by its exact
      // parameters (pointers, sizes, item plans follow from them)
      std::string key((const char *)&C, sizeof(C));
      const int64_t extra[] = {(int64_t)(intptr_t)D, (int64_t)(intptr_t)s->bnd,
                               (int64_t)(intptr_t)s->pi_off, (int64_t)(intptr_t)s->pi_times,
                               (int64_t)(intptr_t)s->buf, (int64_t)(intptr_t)s->offsets,
                               s->P, s->W, s->csr, pct, MODE, (int64_t)sizeof(TS), narrow,
                               ncta, nregions, e->item_workers, e->tail_div, e->tail_frac};
      key.append((const char *)extra, sizeof(extra));
      auto it = e->graphs.find(key);
      if (it == e->graphs.end()) {
        if (e->graphs.size() >= 64) e->drop_graphs();
        cudaGraph_t gr = nullptr;
        CK(cudaStreamBeginCapture(e->st, cudaStreamCaptureModeThreadLocal));
        const int rc = enqueue();
        const cudaError_t ce = cudaStreamEndCapture(e->st, &gr);
        if (rc != GS_OK) {
          if (gr) cudaGraphDestroy(gr);
          return rc;
        }
        CK(ce);
        gs_engine::ChunkGraph cg;
        const cudaError_t ie = cudaGraphInstantiate(&cg.exec, gr, 0);
        cudaGraphDestroy(gr);
        CK(ie);
        cg.k1 = k1;
        cg.nl = nl;
        it = e->graphs.emplace(std::move(key), cg).first;
        ++e->graph_builds;
      } else {
        ++e->graph_hits;
      }
      k1 = it->second.k1;
      nl = it->second.nl;
      CK(cudaGraphLaunch(it->second.exec, e->st));
    }
    CK(cudaMemcpyAsync(e->err_host, e->err, sizeof(int) * ERR_NFLAGS, cudaMemcpyDeviceToHost, e->st));
    unsigned long long blocks_used = 0;
    CK(cudaMemcpyAsync(&blocks_used, e->bump + 2 * (size_t)nregions, sizeof(unsigned long long),
                       cudaMemcpyDeviceToHost, e->st));
    CK(cudaStreamSynchronize(e->st));
    if (e->err_host[ERR_CAP])
      return fail(GS_ERR_CONSISTENCY, "gate output overran its staging bound or arena region "
                                      "(device-side two-pass invariant violated)");
    if (e->err_host[ERR_POOL]) {
      // the chunk did not fit its output regions: grow the pool, else shrink the chunk
      if (e->data_bytes - pi_bytes < room) {
        pool_bytes = std::min<int64_t>(room, (e->data_bytes - pi_bytes) * 4);
      } else if (Wc > kTile) {
        Wc = std::max<int64_t>(kTile, (wc / 2) / kTile * kTile);
      } else {
        return fail(GS_ERR_CAPACITY, "one 128-window chunk's waveforms exceed the device budget");
      }
      continue;
    }
    const int64_t used_words = (int64_t)blocks_used * block_words;
    peak_bytes = std::max<int64_t>(peak_bytes, used_words * (int64_t)sizeof(TS) + pi_bytes);
    float a = 0.f, b = 0.f;
    CK(cudaEventElapsedTime(&a, e->ev[0], e->ev[1]));
    CK(cudaEventElapsedTime(&b, e->ev[1], e->ev[2]));
    ms_stim += a;
    ms_eval += b;
    ms_total += a + b;
    launches += k1 + nl;
    eval_launches += nl;
    ++chunks;
    // ---- results of the chunk (the chunk is complete here: no pool re-run)
    if (ro.cmp && G > 0) {
      CompareDev X = *ro.cmp;
      X.col0 = w - ro.w_base;
      const int64_t items = G * (int64_t)Tc;
      const int blocks = (int)std::max<int64_t>(1, std::min<int64_t>((items + 7) / 8, e->sms * 16));
      compare_arena<TS><<<blocks, 256, 0, e->st>>>(Dd, C, X);
      CK(cudaGetLastError());
    }
    {
      const int threads = 256;
      const int blocks = (int)std::max<int64_t>(1, std::min<int64_t>((N + threads - 1) / threads, 4096));
      acc_commit<<<blocks, threads, 0, e->st>>>(e->acc, ro.acc_dev, (int)N);
      CK(cudaGetLastError());
    }
    if (arena && ro.arena) {
      gs_arena_out *ar = ro.arena;
      const int64_t col = w - ro.w_base;
      const int64_t dp = ro.arena_cols * 8;
      struct { int64_t *h; long long *d; } rows[] = {{ar->counts, e->a_cnt}, {ar->peak, e->a_peak},
          {ar->filtered, e->a_filt}, {ar->ic_filtered, e->a_icf}, {ar->discarded, e->a_disc}};
      for (auto &r : rows)
        if (r.h && G)
          CK(cudaMemcpy2DAsync(r.h + col, dp, r.d, Wpad * 8, wc * 8, G, cudaMemcpyDeviceToHost, e->st));
      if (ar->initials && G)
        CK(cudaMemcpy2DAsync(ar->initials + col, ro.arena_cols, e->a_init, Wpad, wc, G,
                             cudaMemcpyDeviceToHost, e->st));
      CK(cudaStreamSynchronize(e->st));
      if (!store) TRY(k5_pack<TS>(e, C, w, wc));
    }
    // adapt: a pool well under-filled lets the next chunk grow, but never
    // past the metadata share of the budget the first chunk was sized by
    if (used_words > 0) {
      const double fill = (double)used_words / (double)pool_words;
      if (fill < 0.3 && wc == Wc)
        Wc = std::min<int64_t>({round_up(total, kTile), Wc * 2, std::max<int64_t>(Wc, meta_cap)});
    }
    w += wc;
  }
  e->pool_bytes = pool_bytes;
  hint = Wc;
  if (store && ro.arena->n_buf)
    CK(cudaMemcpyAsync(ro.arena->buf, e->a_buf, sizeof(long long) * ro.arena->n_buf,
                       cudaMemcpyDeviceToHost, e->st));
  CK(cudaStreamSynchronize(e->st));
  e->last.ms_total = ms_total;
  e->last.ms_gate_eval = ms_eval;
  e->last.ms_stim = ms_stim;
  e->last.launches = launches;
  e->last.gate_eval_launches = eval_launches;
  e->last.chunks = chunks;
  e->last.data_bytes_peak = peak_bytes;
  e->last.graph_builds = e->graph_builds;
  e->last.graph_replays = e->graph_hits;
  return GS_OK;
}

template <int MODE>
int run_mode(gs_engine *e, gs_stim *s, int64_t w_lo, int64_t w_hi, int pct, RunOut &ro) {
  if (s->wide) return run_chunks<unsigned long long, MODE>(e, s, w_lo, w_hi, pct, ro);
  return run_chunks<unsigned, MODE>(e, s, w_lo, w_hi, pct, ro);
}

int check_run(gs_engine *e, gs_stim *s, int64_t w_lo, int64_t w_hi, int pct) {
  if (!e || !s) return fail(GS_ERR_ARG, "null engine or stimulus");
  if (s->d != e->d) return fail(GS_ERR_ARG, "stimulus belongs to another design");
  if (w_lo < 0 || w_hi > s->W || w_lo > w_hi) return fail(GS_ERR_ARG, "window range out of bounds");
  if (pct < 0 || pct > 100) return fail(GS_ERR_ARG, "pathpulse_pct must be within [0, 100]");
  TRY(use_device(e->d->device));
  return GS_OK;
}

int finish_stats(gs_engine *e, gs_stats_out *out) {
  const int64_t N = e->d->N;
  std::vector<long long> h(3 * N + 3);
  CK(cudaMemcpy(h.data(), e->acc_run, sizeof(long long) * (3 * N + 3), cudaMemcpyDeviceToHost));
  for (int64_t i = 0; i < N; ++i) {
    if (out->t1) out->t1[i] += h[i];
    if (out->tc) out->tc[i] += h[N + i];
    if (out->ig) out->ig[i] += h[2 * N + i];
  }
  for (int j = 0; j < 3; ++j) out->totals[j] += h[3 * N + j];
  // stored toggles and fanin toggles (sum over pins of the driver's count),
  // the two data-dependent terms of the algorithmic byte count
  long long outs = 0, ins = 0;
  for (int64_t n = 0; n < N; ++n) {
    if (n >= e->d->P) outs += h[N + n];
    ins += h[N + n] * e->d->fanout[n];
  }
  e->last.output_toggles = outs;
  e->last.input_toggles = ins;
  return GS_OK;
}

}  // namespace

// =========================================================================
// C ABI

extern "C" {

int gs_version(void) { return 1; }

const char *gs_last_error(void) { return g_err.c_str(); }

int64_t gs_last_error_line(void) { return g_err_line; }

int64_t gs_last_error_col(void) { return g_err_col; }

int gs_device_count(int *count) {
  int n = 0;
  cudaError_t e = cudaGetDeviceCount(&n);
  if (e != cudaSuccess) {
    (void)cudaGetLastError();
    n = 0;
  }
  if (count) *count = n;
  return GS_OK;
}

int gs_design_create(const gs_design_desc *desc, int device, gs_design **out) {
  if (!out) return fail(GS_ERR_ARG, "null output handle");
  *out = nullptr;
  gs_design *D = new gs_design();
  int rc = design_build(desc, device, D);
  if (rc != GS_OK) {
    D->release();
    delete D;
    return rc;
  }
  *out = D;
  return GS_OK;
}

int gs_design_destroy(gs_design *d) {
  if (!d) return GS_OK;
  cudaSetDevice(d->device);
  d->release();
  delete d;
  return GS_OK;
}

int gs_stim_create(gs_design *d, const gs_stim_desc *desc, gs_stim **out) {
  if (!d || !out) return fail(GS_ERR_ARG, "null design or output handle");
  *out = nullptr;
  gs_stim *S = new gs_stim();
  int rc = stim_build(d, desc, S);
  if (rc != GS_OK) {
    S->release();
    delete S;
    return rc;
  }
  *out = S;
  return GS_OK;
}

int gs_stim_destroy(gs_stim *s) {
  if (!s) return GS_OK;
  cudaSetDevice(s->d->device);
  s->release();
  delete s;
  return GS_OK;
}

static SynthArgs synth_args(const gs_synth_desc *sd) {
  SynthArgs A;
  A.P = (int)sd->num_pis;
  A.ppis = (int)sd->num_ppis;
  A.seed = sd->seed;
  A.ppi_thr = sd->ppi_thr;
  A.pi_thr = sd->pi_thr;
  A.period = sd->period;
  A.ppi_lo = sd->ppi_lo;
  A.ppi_span = sd->ppi_span;
  A.pi_lo = sd->pi_lo;
  A.pi_span = sd->pi_span;
  A.w_lo = sd->w_lo;
  A.w_hi = sd->w_hi;
  return A;
}

static int synth_check(const gs_synth_desc *sd) {
  if (sd->num_pis < 0 || sd->num_pis > INT32_MAX) return fail(GS_ERR_ARG, "num_pis out of range");
  if (sd->num_ppis < 0 || sd->num_ppis > sd->num_pis) return fail(GS_ERR_ARG, "num_ppis out of range");
  if (sd->period <= 0) return fail(GS_ERR_ARG, "window period must be positive");
  if (sd->w_lo < 0 || sd->w_hi <= sd->w_lo) return fail(GS_ERR_ARG, "need a non-empty window range");
  if (sd->ppi_lo < 0 || sd->pi_lo < 0 || sd->ppi_span < 0 || sd->pi_span < 0 ||
      sd->ppi_lo + std::max<int64_t>(sd->ppi_span, 1) > sd->period ||
      sd->pi_lo + std::max<int64_t>(sd->pi_span, 1) > sd->period)
    return fail(GS_ERR_ARG, "toggle offsets must lie inside the window");
  if (sd->w_hi > INT64_MAX / sd->period - 1) return fail(GS_ERR_ARG, "window range overflows int64 time");
  return GS_OK;
}

int gs_synth_window_counts(const gs_synth_desc *sd, int device, int64_t *counts) {
  if (!sd || !counts) return fail(GS_ERR_ARG, "null synthetic-stimulus argument");
  TRY(synth_check(sd));
  TRY(use_device(device));
  const int64_t W = sd->w_hi - sd->w_lo;
  long long *c = nullptr;
  TRY(dalloc(&c, (size_t)W));
  const SynthArgs A = synth_args(sd);
  synth_window_counts<<<(int)std::min<int64_t>((W + 255) / 256, 8192), 256>>>(A, c);
  cudaError_t e = cudaGetLastError();
  if (e == cudaSuccess) e = cudaMemcpy(counts, c, sizeof(long long) * W, cudaMemcpyDeviceToHost);
  dfree(c);
  if (e != cudaSuccess) return fail(GS_ERR_CUDA, cudaGetErrorString(e));
  return GS_OK;
}

int gs_stim_synth(gs_design *d, const gs_synth_desc *sd, gs_stim **out) {
  if (!d || !sd || !out) return fail(GS_ERR_ARG, "null synthetic-stimulus argument");
  *out = nullptr;
  if (sd->num_pis != d->P) return fail(GS_ERR_ARG, "stimulus input count != design inputs");
  TRY(synth_check(sd));
  const int64_t P = sd->num_pis, W = sd->w_hi - sd->w_lo;
  gs_stim *S = new gs_stim();
  S->d = d;
  S->P = (int)P;
  S->W = W;
  S->csr = true;
  S->max_wlen = sd->period;
  S->wide = sd->period > (int64_t)0xFFFFFFFFll;
  long long *cnt = nullptr;
  int rc = [&]() -> int {
    TRY(use_device(d->device));
    TRY(pool_ready(d->device));
    TRY(upload_stream(d->device, &S->us));
    cudaStream_t us = S->us;
    const SynthArgs A = synth_args(sd);
    CK(cudaMallocAsync((void **)&S->bnd, sizeof(long long) * (W + 1), us));
    CK(cudaMallocAsync((void **)&S->pi_off, sizeof(long long) * (P + 1), us));
    CK(cudaMallocAsync((void **)&S->pi_init, std::max<int64_t>(P, 1), us));
    CK(cudaMallocAsync((void **)&cnt, sizeof(long long) * std::max<int64_t>(P, 1), us));
    synth_bounds<<<(int)std::min<int64_t>((W + 256) / 256, 4096), 256, 0, us>>>(S->bnd, sd->w_lo, W,
                                                                                  sd->period);
    CK(cudaGetLastError());
    const int blocks = (int)std::max<int64_t>(1, std::min<int64_t>((P + 7) / 8, 16384));
    std::vector<long long> h(P + 1, 0);
    if (P) {
      synth_count<<<blocks, 256, 0, us>>>(A, cnt, S->pi_init);
      CK(cudaGetLastError());
      CK(cudaMemcpyAsync(h.data() + 1, cnt, sizeof(long long) * P, cudaMemcpyDeviceToHost, us));
      CK(cudaStreamSynchronize(us));
    }
    for (int64_t p = 0; p < P; ++p) h[p + 1] += h[p];
    S->n_toggles = h[P];
    CK(cudaMemcpyAsync(S->pi_off, h.data(), sizeof(long long) * (P + 1), cudaMemcpyHostToDevice, us));
    CK(cudaMallocAsync((void **)&S->pi_times, sizeof(long long) * std::max<int64_t>(S->n_toggles, 1), us));
    if (P) {
      synth_fill<<<blocks, 256, 0, us>>>(A, S->pi_off, S->pi_times);
      CK(cudaGetLastError());
    }
    CK(cudaStreamSynchronize(us));
    return GS_OK;
  }();
  if (cnt) cudaFreeAsync(cnt, S->us);
  if (rc != GS_OK) {
    S->release();
    delete S;
    return rc;
  }
  *out = S;
  return GS_OK;
}

int gs_stim_sizes(const gs_stim *s, int64_t *num_windows, int64_t *num_toggles) {
  if (!s) return fail(GS_ERR_ARG, "null stimulus");
  if (num_windows) *num_windows = s->W;
  if (num_toggles) *num_toggles = s->n_toggles;
  return GS_OK;
}

int gs_stim_download(const gs_stim *s, int64_t *boundaries, int64_t *pi_off, int64_t *pi_times,
                     uint8_t *pi_init) {
  if (!s) return fail(GS_ERR_ARG, "null stimulus");
  if (!s->csr) return fail(GS_ERR_ARG, "only CSR stimuli can be downloaded");
  TRY(use_device(s->d->device));
  cudaStream_t us = s->us;
  if (boundaries)
    CK(cudaMemcpyAsync(boundaries, s->bnd, sizeof(long long) * (s->W + 1), cudaMemcpyDeviceToHost, us));
  if (pi_off)
    CK(cudaMemcpyAsync(pi_off, s->pi_off, sizeof(long long) * (s->P + 1), cudaMemcpyDeviceToHost, us));
  if (pi_times && s->n_toggles)
    CK(cudaMemcpyAsync(pi_times, s->pi_times, sizeof(long long) * s->n_toggles,
                       cudaMemcpyDeviceToHost, us));
  if (pi_init && s->P) CK(cudaMemcpyAsync(pi_init, s->pi_init, s->P, cudaMemcpyDeviceToHost, us));
  CK(cudaStreamSynchronize(us));
  return GS_OK;
}

int gs_engine_create(gs_design *d, int64_t mem_budget, void *stream, gs_engine **out) {
  if (!d || !out) return fail(GS_ERR_ARG, "null design or output handle");
  *out = nullptr;
  TRY(use_device(d->device));
  gs_engine *e = new gs_engine();
  e->d = d;
  int rc = [&]() -> int {
    CK(cudaDeviceGetAttribute(&e->sms, cudaDevAttrMultiProcessorCount, d->device));
    size_t fr = 0, tot = 0;
    CK(cudaMemGetInfo(&fr, &tot));
    e->budget = mem_budget > 0 ? mem_budget : (int64_t)(fr * 3 / 4);
    if (stream) {
      e->st = (cudaStream_t)stream;
    } else {
      CK(cudaStreamCreateWithFlags(&e->st, cudaStreamNonBlocking));
      e->own_stream = true;
    }
    for (auto &ev : e->ev) CK(cudaEventCreate(&ev));
    TRY(dalloc(&e->acc, (size_t)ACC_ROWS * d->N));
    TRY(dalloc(&e->acc_run, (size_t)3 * d->N + 3));
    TRY(dalloc(&e->err, ERR_NFLAGS));
    CK(cudaMallocHost((void **)&e->err_host, sizeof(int) * ERR_NFLAGS));
    return GS_OK;
  }();
  if (rc != GS_OK) {
    e->release();
    delete e;
    return rc;
  }
  *out = e;
  return GS_OK;
}

int gs_slab_words(int k, int narrow) {
  // words of a warp's shared-memory slab in the K4 instance that evaluates
  // k-input gates (narrow: 32-bit time); a tile's fanin segments and outputs
  // are staged there when they fit
  if (narrow && k >= 1 && k <= 4)
    return k == 1 ? lean_slab_words<1>() : k == 2 ? lean_slab_words<2>()
         : k == 3 ? lean_slab_words<3>() : lean_slab_words<4>();
  return slab_words<0>();
}

int gs_engine_set_items(gs_engine *e, int64_t workers, int tail_div, int tail_frac) {
  if (!e) return fail(GS_ERR_ARG, "null engine");
  if (workers < 0 || tail_div < 1 || tail_frac < 1)
    return fail(GS_ERR_ARG, "item sizing: workers >= 0, tail_div >= 1, tail_frac >= 1");
  e->item_workers = workers;
  e->tail_div = tail_div;
  e->tail_frac = tail_frac;
  return GS_OK;
}

int gs_engine_destroy(gs_engine *e) {
  if (!e) return GS_OK;
  cudaSetDevice(e->d->device);
  cudaStreamSynchronize(e->st);
  e->release();
  delete e;
  return GS_OK;
}

int gs_run_stats_device(gs_engine *e, gs_stim *s, int64_t w_lo, int64_t w_hi, int pct,
                        int64_t *acc_dev) {
  TRY(check_run(e, s, w_lo, w_hi, pct));
  if (!acc_dev) return fail(GS_ERR_ARG, "null device accumulator");
  RunOut ro{(long long *)acc_dev, nullptr, w_lo, w_hi - w_lo};
  return run_mode<MODE_STATS>(e, s, w_lo, w_hi, pct, ro);
}

int gs_run_stats(gs_engine *e, gs_stim *s, int64_t w_lo, int64_t w_hi, int pct, gs_stats_out *out) {
  TRY(check_run(e, s, w_lo, w_hi, pct));
  if (!out) return fail(GS_ERR_ARG, "null stats output");
  CK(cudaMemsetAsync(e->acc_run, 0, sizeof(long long) * (3 * (size_t)e->d->N + 3), e->st));
  RunOut ro{e->acc_run, nullptr, w_lo, w_hi - w_lo};
  TRY(run_mode<MODE_STATS>(e, s, w_lo, w_hi, pct, ro));
  return finish_stats(e, out);
}

int gs_run_compare(gs_engine *e, gs_stim *s, int64_t w_lo, int64_t w_hi, int pct,
                   const gs_arena_ref *ref, int64_t *mismatches, int64_t *first_gate,
                   int64_t *first_window) {
  TRY(check_run(e, s, w_lo, w_hi, pct));
  if (!ref || !mismatches || !first_gate || !first_window)
    return fail(GS_ERR_ARG, "null compare argument");
  const int64_t G = e->d->G, Ws = w_hi - w_lo;
  if (ref->cols < Ws || (G * Ws > 0 && (!ref->offsets || !ref->counts || !ref->initials)))
    return fail(GS_ERR_ARG, "reference arena does not cover the window range");
  for (int64_t g = 0; g < G; ++g)
    for (int64_t w = 0; w < Ws; ++w) {
      const int64_t o = ref->offsets[g * ref->cols + w], c = ref->counts[g * ref->cols + w];
      if (c < 0 || o < 0 || o + c > ref->n_buf) return fail(GS_ERR_ARG, "reference arena out of range");
    }
  long long *buf = nullptr, *off = nullptr, *cnt = nullptr;
  unsigned char *ini = nullptr;
  unsigned long long *bad = nullptr;
  int rc = [&]() -> int {
    TRY(upload(&buf, (const long long *)ref->buf, (size_t)ref->n_buf));
    TRY(upload(&off, (const long long *)ref->offsets, (size_t)(G * ref->cols)));
    TRY(upload(&cnt, (const long long *)ref->counts, (size_t)(G * ref->cols)));
    TRY(upload(&ini, ref->initials, (size_t)(G * ref->cols)));
    TRY(dalloc(&bad, 2));
    const unsigned long long init[2] = {0ull, ~0ull};
    CK(cudaMemcpy(bad, init, sizeof(init), cudaMemcpyHostToDevice));
    CompareDev X;
    X.buf = buf;
    X.offsets = off;
    X.counts = cnt;
    X.initials = ini;
    X.cols = ref->cols;
    X.col0 = 0;
    X.G = (int)G;
    X.bad = bad;
    CK(cudaMemsetAsync(e->acc_run, 0, sizeof(long long) * (3 * (size_t)e->d->N + 3), e->st));
    RunOut ro{e->acc_run, nullptr, w_lo, Ws, &X};
    TRY(run_mode<MODE_STATS>(e, s, w_lo, w_hi, pct, ro));
    unsigned long long h[2];
    CK(cudaStreamSynchronize(e->st));
    CK(cudaMemcpy(h, bad, sizeof(h), cudaMemcpyDeviceToHost));
    *mismatches = (int64_t)h[0];
    *first_gate = h[0] ? (int64_t)(h[1] >> 32) : -1;
    *first_window = h[0] ? (int64_t)(h[1] & 0xFFFFFFFFull) + w_lo : -1;
    return GS_OK;
  }();
  dfree(buf);
  dfree(off);
  dfree(cnt);
  dfree(ini);
  dfree(bad);
  return rc;
}

int gs_run_arena(gs_engine *e, gs_stim *s, int64_t w_lo, int64_t w_hi, int pct,
                 gs_arena_out *arena, gs_stats_out *stats) {
  TRY(check_run(e, s, w_lo, w_hi, pct));
  if (!arena) return fail(GS_ERR_ARG, "null arena output");
  const bool store = arena->buf != nullptr;
  if (store) {
    if (!arena->offsets) return fail(GS_ERR_ARG, "store pass needs region offsets");
    const int64_t G = e->d->G, Ws = w_hi - w_lo;
    for (int64_t i = 0; i < G * Ws; ++i)
      if (arena->offsets[i] < 0 || arena->offsets[i] > arena->n_buf)
        return fail(GS_ERR_ARG, "arena offsets out of range");
  }
  CK(cudaMemsetAsync(e->acc_run, 0, sizeof(long long) * (3 * (size_t)e->d->N + 3), e->st));
  RunOut ro{e->acc_run, arena, w_lo, w_hi - w_lo};
  e->kept.clear();
  e->kept_stim = nullptr;
  if (store) {
    TRY(run_mode<MODE_STORE>(e, s, w_lo, w_hi, pct, ro));
  } else {
    TRY(run_mode<MODE_COUNTERS>(e, s, w_lo, w_hi, pct, ro));
    e->kept_stim = s;
    e->kept_lo = w_lo;
    e->kept_hi = w_hi;
    e->kept_pct = pct;
  }
  if (stats) return finish_stats(e, stats);
  return GS_OK;
}

int gs_arena_fill(gs_engine *e, const gs_stim *s, int64_t w_lo, int64_t w_hi, int pct,
                  int64_t *buf, int64_t n_buf, const int64_t *offsets, int64_t cols,
                  int *filled) {
  if (!e || !filled || (!buf && n_buf) || cols < w_hi - w_lo || n_buf < 0)
    return fail(GS_ERR_ARG, "bad arena fill arguments");
  *filled = 0;
  if (!e->kept_stim || e->kept_stim != s || e->kept_lo != w_lo || e->kept_hi != w_hi ||
      e->kept_pct != pct)
    return GS_OK;  // no count pass of this run to fill from
  const gs_design *D = e->d;
  const int64_t G = D->G;
  if (G && !offsets) return fail(GS_ERR_ARG, "arena fill needs region offsets");
  for (const auto &pc : e->kept) {
    int64_t base = 0;
    for (int64_t i = 0; i < G; ++i) {
      const int g = D->order_host[i];
      const int64_t len = pc.rs[g];
      if (len) {
        const int64_t dst = offsets[(int64_t)g * cols + (pc.w0 - w_lo)];
        if (dst < 0 || dst + len > n_buf || base + len > (int64_t)pc.piece.size())
          return fail(GS_ERR_ARG, "arena regions do not match the count pass");
        memcpy(buf + dst, pc.piece.data() + base, sizeof(int64_t) * len);
      }
      base += len;
    }
  }
  *filled = 1;
  return GS_OK;
}

#ifdef GS_PROF
// debug builds only (not part of the ABI header): read and clear the counters
int gs_prof_read(unsigned long long *out16) {
  CK(cudaMemcpyFromSymbol(out16, gs_prof_counters, sizeof(unsigned long long) * 16));
  unsigned long long z[16] = {0};
  CK(cudaMemcpyToSymbol(gs_prof_counters, z, sizeof(z)));
  return GS_OK;
}
#endif

int gs_last_timing(gs_engine *e, gs_timing *t) {
  if (!e || !t) return fail(GS_ERR_ARG, "null argument");
  *t = e->last;
  return GS_OK;
}

int gs_dwell_sweep(int64_t num_nets, const uint8_t *net_kind, const int64_t *net_slot,
                   const int64_t *stim_buf, int64_t n_stim_buf, const int64_t *stim_off,
                   const int64_t *stim_cnt, const uint8_t *stim_init, int64_t num_pis,
                   int64_t num_windows, const int64_t *gbuf, int64_t n_gbuf, const int64_t *g_off,
                   const int64_t *g_cnt, const uint8_t *g_init, int64_t num_gates, int64_t g_cols,
                   const int64_t *boundaries, int64_t w_lo, int64_t w_hi, int64_t w_off,
                   int64_t *t0_out, int64_t *t1_out, int64_t *tc_out) {
  if (num_nets < 0 || w_lo < 0 || w_hi > num_windows || w_lo > w_hi || w_lo < w_off ||
      w_hi - w_off > g_cols)
    return fail(GS_ERR_ARG, "dwell_sweep: bad sizes or window range");
  // bounds of every region the kernel will read
  for (int64_t n = 0; n < num_nets; ++n) {
    const int64_t s = net_slot[n];
    const bool pi = net_kind[n] == 0;
    if (s < 0 || s >= (pi ? num_pis : num_gates)) return fail(GS_ERR_ARG, "dwell_sweep: bad net slot");
    for (int64_t w = w_lo; w < w_hi; ++w) {
      const int64_t o = pi ? stim_off[s * num_windows + w] : g_off[s * g_cols + (w - w_off)];
      const int64_t c = pi ? stim_cnt[s * num_windows + w] : g_cnt[s * g_cols + (w - w_off)];
      if (o < 0 || c < 0 || o + c > (pi ? n_stim_buf : n_gbuf))
        return fail(GS_ERR_ARG, "dwell_sweep: waveform region out of range");
    }
  }
  int dev = 0;
  CK(cudaGetDevice(&dev));
  TRY(use_device(dev));
  DwellArgs A;
  memset(&A, 0, sizeof(A));
  unsigned char *nk = nullptr, *si = nullptr, *gi = nullptr;
  long long *ns = nullptr, *sb = nullptr, *so = nullptr, *sc = nullptr, *gb = nullptr,
            *go = nullptr, *gc = nullptr, *bd = nullptr, *out = nullptr;
  int rc = [&]() -> int {
    TRY(upload(&nk, net_kind, num_nets));
    TRY(upload(&ns, (const long long *)net_slot, num_nets));
    TRY(upload(&sb, (const long long *)stim_buf, n_stim_buf));
    TRY(upload(&so, (const long long *)stim_off, num_pis * num_windows));
    TRY(upload(&sc, (const long long *)stim_cnt, num_pis * num_windows));
    TRY(upload(&si, stim_init, num_pis * num_windows));
    TRY(upload(&gb, (const long long *)gbuf, n_gbuf));
    TRY(upload(&go, (const long long *)g_off, num_gates * g_cols));
    TRY(upload(&gc, (const long long *)g_cnt, num_gates * g_cols));
    TRY(upload(&gi, g_init, num_gates * g_cols));
    TRY(upload(&bd, (const long long *)boundaries, num_windows + 1));
    TRY(dalloc(&out, (size_t)3 * num_nets));
    CK(cudaMemset(out, 0, sizeof(long long) * 3 * (num_nets ? num_nets : 1)));
    A.N = (int)num_nets;
    A.net_kind = nk;
    A.net_slot = ns;
    A.sbuf = sb;
    A.soff = so;
    A.scnt = sc;
    A.sinit = si;
    A.sW = num_windows;
    A.gbuf = gb;
    A.goff = go;
    A.gcnt = gc;
    A.ginit = gi;
    A.gW = g_cols;
    A.bnd = bd;
    A.w_lo = w_lo;
    A.w_hi = w_hi;
    A.w_off = w_off;
    A.t0 = out;
    A.t1 = out + num_nets;
    A.tc = out + 2 * num_nets;
    if (num_nets && w_hi > w_lo) {
      const int64_t warps = num_nets * ((w_hi - w_lo + 31) / 32);
      const int blocks = (int)std::min<int64_t>((warps + 7) / 8, 148 * 32);
      dwell_arena<<<blocks, 256>>>(A);
      CK(cudaGetLastError());
    }
    std::vector<long long> h(3 * num_nets);
    if (num_nets) CK(cudaMemcpy(h.data(), out, sizeof(long long) * 3 * num_nets, cudaMemcpyDeviceToHost));
    for (int64_t n = 0; n < num_nets; ++n) {
      t0_out[n] += h[n];
      t1_out[n] += h[num_nets + n];
      tc_out[n] += h[2 * num_nets + n];
    }
    return GS_OK;
  }();
  dfree(nk); dfree(ns); dfree(sb); dfree(so); dfree(sc); dfree(si); dfree(gb); dfree(go);
  dfree(gc); dfree(gi); dfree(bd); dfree(out);
  return rc;
}

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
                int64_t *out_disc, int64_t *out_err, int64_t *out_peak, int64_t pct) {
  (void)out_net;  // gate g drives net out_net[g]; sim_span itself never reads it
  const int64_t G = num_gates, N = num_nets;
  if (oi_lo < 0 || oi_hi > G || oi_lo > oi_hi || w_lo < 0 || w_hi < w_lo ||
      w_hi > stim_cols || w_hi > init_cols || w_off > w_lo || w_hi - w_off > g_cols ||
      pct < 0 || pct > 100 || G < 0 || N < G || n_gbuf < 0 || n_stim_buf < 0)
    return fail(GS_ERR_ARG, "sim_span range or size out of bounds");
  // every index the span will follow, checked before anything reaches the GPU
  const int64_t n_pins = G ? pin_off[G] : 0;
  for (int64_t oi = oi_lo; oi < oi_hi; ++oi) {
    const int64_t g = order[oi];
    if (g < 0 || g >= G) return fail(GS_ERR_ARG, "order entry out of range");
    const int64_t p0 = pin_off[g], k = pin_off[g + 1] - p0;
    if (k < 1 || k > kMaxK || p0 < 0 || p0 + k > n_pins)
      return fail(GS_ERR_ARG, "gate fanin count out of range");
    if (lut_off[g] < 0 || lut_off[g] + (int64_t(1) << k) > num_lut_bits)
      return fail(GS_ERR_ARG, "lut_off out of range");
    for (int64_t p = p0; p < p0 + k; ++p) {
      const int64_t n = pin_net[p];
      if (n < 0 || n >= N || pin_arc[p] < 0 ||
          pin_arc[p] + (int64_t(1) << (k - 1)) > num_arc_rows)
        return fail(GS_ERR_ARG, "pin entry out of range");
      const int64_t sl = net_slot[n];
      for (int64_t w = w_lo; w < w_hi; ++w) {
        int64_t o, c, lim;
        if (net_kind[n] == 0) {
          if (sl < 0 || sl >= stim_rows) return fail(GS_ERR_ARG, "input slot out of range");
          o = stim_off[sl * stim_cols + w], c = stim_cnt[sl * stim_cols + w], lim = n_stim_buf;
        } else {
          if (sl < 0 || sl >= G) return fail(GS_ERR_ARG, "gate slot out of range");
          o = g_off[sl * g_cols + (w - w_off)], c = g_cnt[sl * g_cols + (w - w_off)];
          lim = n_gbuf;
        }
        if (o < 0 || c < 0 || o + c > lim) return fail(GS_ERR_ARG, "fanin region out of range");
      }
    }
    for (int64_t w = w_lo; w < w_hi; ++w) {
      const int64_t o = g_off[g * g_cols + (w - w_off)], c = g_cap[g * g_cols + (w - w_off)];
      if (o < 0 || c < 0 || o + c > n_gbuf) return fail(GS_ERR_ARG, "output region out of range");
    }
  }
  TRY(use_device(0));
  std::vector<void *> bufs;
  auto up = [&](const void *src, size_t bytes, void **dst) -> int {
    *dst = nullptr;
    CK(cudaMalloc(dst, bytes ? bytes : 8));
    bufs.push_back(*dst);
    if (bytes && src) CK(cudaMemcpy(*dst, src, bytes, cudaMemcpyHostToDevice));
    return GS_OK;
  };
  const size_t gw = (size_t)(G * g_cols) * 8, nw = (size_t)N;
  int rc = [&]() -> int {
    SpanArgs A;
    void *p;
    A.oi_lo = oi_lo; A.oi_hi = oi_hi; A.w_lo = w_lo; A.w_hi = w_hi; A.w_off = w_off;
    A.stim_cols = stim_cols; A.init_cols = init_cols; A.g_cols = g_cols; A.pct = pct;
    TRY(up(order, (size_t)G * 8, &p)); A.order = (const long long *)p;
    TRY(up(pin_off, (size_t)(G + 1) * 8, &p)); A.pin_off = (const long long *)p;
    TRY(up(pin_net, (size_t)n_pins * 8, &p)); A.pin_net = (const long long *)p;
    TRY(up(pin_ic, (size_t)n_pins * 8, &p)); A.pin_ic = (const long long *)p;
    TRY(up(pin_arc, (size_t)n_pins * 8, &p)); A.pin_arc = (const long long *)p;
    TRY(up(arc_rows, (size_t)num_arc_rows * 16, &p)); A.arc_rows = (const long long *)p;
    TRY(up(lut_off, (size_t)G * 8, &p)); A.lut_off = (const long long *)p;
    TRY(up(lut_bits, (size_t)num_lut_bits, &p)); A.lut_bits = (const unsigned char *)p;
    TRY(up(net_kind, nw, &p)); A.net_kind = (const unsigned char *)p;
    TRY(up(net_slot, nw * 8, &p)); A.net_slot = (const long long *)p;
    TRY(up(stim_buf, (size_t)n_stim_buf * 8, &p)); A.stim_buf = (const long long *)p;
    TRY(up(stim_off, (size_t)(stim_rows * stim_cols) * 8, &p)); A.stim_off = (const long long *)p;
    TRY(up(stim_cnt, (size_t)(stim_rows * stim_cols) * 8, &p)); A.stim_cnt = (const long long *)p;
    TRY(up(init_vals, nw * (size_t)init_cols, &p)); A.init_vals = (const unsigned char *)p;
    TRY(up(boundaries, (size_t)(stim_cols + 1) * 8, &p)); A.bnd = (const long long *)p;
    TRY(up(gbuf, (size_t)n_gbuf * 8, &p)); A.gbuf = (long long *)p;
    TRY(up(g_off, gw, &p)); A.g_off = (const long long *)p;
    TRY(up(g_cap, gw, &p)); A.g_cap = (const long long *)p;
    TRY(up(g_cnt, gw, &p)); A.g_cnt = (long long *)p;
    TRY(up(out_filt, gw, &p)); A.out_filt = (long long *)p;
    TRY(up(out_icf, gw, &p)); A.out_icf = (long long *)p;
    TRY(up(out_disc, gw, &p)); A.out_disc = (long long *)p;
    TRY(up(out_err, gw, &p)); A.out_err = (long long *)p;
    TRY(up(out_peak, gw, &p)); A.out_peak = (long long *)p;
    const int64_t total = (oi_hi - oi_lo) * (w_hi - w_lo);
    if (total) {
      sim_span_seam<<<(int)std::min<int64_t>((total + 127) / 128, 148 * 32), 128>>>(A);
      CK(cudaGetLastError());
    }
    struct { int64_t *h; void *d; size_t n; } back[] = {
        {gbuf, A.gbuf, (size_t)n_gbuf * 8}, {g_cnt, A.g_cnt, gw}, {out_filt, A.out_filt, gw},
        {out_icf, A.out_icf, gw}, {out_disc, A.out_disc, gw}, {out_err, A.out_err, gw},
        {out_peak, A.out_peak, gw}};
    for (auto &b : back)
      if (b.n) CK(cudaMemcpy(b.h, b.d, b.n, cudaMemcpyDeviceToHost));
    return GS_OK;
  }();
  for (void *b : bufs) cudaFree(b);
  return rc;
}

int gs_init_values(const gs_design_desc *desc, const uint8_t *stim_init, int64_t num_windows,
                   uint8_t *vals_out) {
  int dev = 0;
  CK(cudaGetDevice(&dev));
  gs_design D;
  int rc = design_build(desc, dev, &D);
  if (rc != GS_OK) {
    D.release();
    return rc;
  }
  const int64_t N = D.N, W = num_windows;
  unsigned char *vals = nullptr;
  rc = [&]() -> int {
    TRY(dalloc(&vals, (size_t)(N * W)));
    if (D.P && W) CK(cudaMemcpy(vals, stim_init, (size_t)D.P * W, cudaMemcpyHostToDevice));
    const DesignDev Dd = D.dev();
    for (int l = 0; l < D.L; ++l) {
      const int lo = (int)D.level_starts[l], n = (int)(D.level_starts[l + 1] - lo);
      const int64_t tot = (int64_t)n * W;
      if (!tot) continue;
      const int blocks = (int)std::min<int64_t>((tot + 255) / 256, 148 * 16);
      zero_delay_level<<<blocks, 256>>>(Dd, vals, W, lo, n);
      CK(cudaGetLastError());
    }
    if (N * W) CK(cudaMemcpy(vals_out, vals, (size_t)(N * W), cudaMemcpyDeviceToHost));
    return GS_OK;
  }();
  dfree(vals);
  D.release();
  return rc;
}

// ---- VCD reader

}  // extern "C"

struct gs_vcd {
  gsvcd::Result r;
};

extern "C" {

int gs_vcd_parse(const char *text, int64_t len, const char *const *pi_names, int64_t num_pis,
                 gs_vcd **out) {
  if (!out || (len > 0 && !text) || num_pis < 0 || (num_pis > 0 && !pi_names))
    return fail(GS_ERR_ARG, "null VCD text, input names or output handle");
  if (num_pis > INT32_MAX) return fail(GS_ERR_ARG, "too many inputs");
  *out = nullptr;
  std::vector<std::string> names;
  names.reserve((size_t)num_pis);
  for (int64_t i = 0; i < num_pis; ++i) {
    if (!pi_names[i]) return fail(GS_ERR_ARG, "null input name");
    names.emplace_back(pi_names[i]);
  }
  gs_vcd *v = new gs_vcd();
  const gsvcd::Status st = gsvcd::parse(text, len, names, v->r);
  if (st != gsvcd::VCD_OK) {
    const std::string msg = v->r.msg;
    const int64_t line = v->r.line;
    delete v;
    if (st == gsvcd::VCD_FALLBACK)
      return fail(GS_ERR_UNSUPPORTED, "VCD text outside the native reader's subset");
    const int rc = fail(st == gsvcd::VCD_PARSE ? GS_ERR_PARSE : GS_ERR_SEMANTIC, msg);
    g_err_line = st == gsvcd::VCD_PARSE ? line : 0;
    return rc;
  }
  *out = v;
  return GS_OK;
}

int gs_vcd_sizes(const gs_vcd *v, int64_t *num_toggles, int64_t *duration) {
  if (!v || !num_toggles || !duration) return fail(GS_ERR_ARG, "null argument");
  *num_toggles = (int64_t)v->r.pi_times.size();
  *duration = v->r.duration;
  return GS_OK;
}

int gs_vcd_copy(const gs_vcd *v, int64_t *pi_off, int64_t *pi_times, uint8_t *pi_init) {
  if (!v || !pi_off || (!pi_times && !v->r.pi_times.empty()) || (!pi_init && !v->r.pi_init.empty()))
    return fail(GS_ERR_ARG, "null argument");
  std::copy(v->r.pi_off.begin(), v->r.pi_off.end(), pi_off);
  std::copy(v->r.pi_times.begin(), v->r.pi_times.end(), pi_times);
  std::copy(v->r.pi_init.begin(), v->r.pi_init.end(), pi_init);
  return GS_OK;
}

int gs_vcd_destroy(gs_vcd *v) {
  delete v;
  return GS_OK;
}

// ---- SDF reader

}  // extern "C"

struct gs_sdf {
  gssdf::Result r;
};

extern "C" {

int gs_sdf_parse(const char *text, int64_t len, const gs_sdf_design *dd, int corner,
                 const char *path, gs_sdf **out) {
  if (!out || !dd || (len > 0 && !text) || corner < 0 || corner > 2)
    return fail(GS_ERR_ARG, "bad SDF reader argument");
  *out = nullptr;
  const int64_t G = dd->num_gates, Nn = dd->num_nets, Cn = dd->num_cells;
  if (G < 0 || Nn < 0 || Cn < 0 || G > INT32_MAX || Nn > INT32_MAX)
    return fail(GS_ERR_ARG, "design size out of range");
  gssdf::Design d;
  auto names = [](const char *blob, const int64_t *off, int64_t n, std::vector<std::string> &o) {
    o.resize((size_t)n);
    for (int64_t i = 0; i < n; ++i) o[i].assign(blob + off[i], (size_t)(off[i + 1] - off[i]));
  };
  names(dd->gate_names, dd->gate_name_off, G, d.gate_names);
  names(dd->net_names, dd->net_name_off, Nn, d.net_names);
  std::vector<std::string> pins;
  const int64_t npins = Cn ? dd->cell_pin_first[Cn] : 0;
  names(dd->pin_names, dd->pin_name_off, npins, pins);
  names(dd->cell_outputs, dd->cell_output_off, Cn, d.cell_output);
  d.cell_inputs.resize((size_t)Cn);
  for (int64_t c = 0; c < Cn; ++c)
    d.cell_inputs[c].assign(pins.begin() + dd->cell_pin_first[c],
                            pins.begin() + dd->cell_pin_first[c + 1]);
  d.gate_cell.resize((size_t)G);
  d.pin_off.assign(dd->pin_off, dd->pin_off + G + 1);
  d.out_net.assign(dd->out_net, dd->out_net + G);
  for (int64_t g = 0; g < G; ++g) {
    const int64_t c = dd->gate_cell[g];
    if (c < 0 || c >= Cn) return fail(GS_ERR_ARG, "gate cell index out of range");
    d.gate_cell[g] = (int)c;
    const int64_t k = d.pin_off[g + 1] - d.pin_off[g];
    if (k < 1 || k > 30 || k != (int64_t)d.cell_inputs[c].size())
      return fail(GS_ERR_ARG, "gate fanin does not match its cell");
    if (d.out_net[g] < 0 || d.out_net[g] >= Nn) return fail(GS_ERR_ARG, "out_net out of range");
  }
  const int64_t P = G ? d.pin_off[G] : 0;
  d.pin_net.assign(dd->pin_net, dd->pin_net + P);
  gs_sdf *h = new gs_sdf();
  const gssdf::Status st = gssdf::parse(text, len, d, corner, path ? path : "<sdf>", h->r);
  if (st != gssdf::SDF_OK) {
    const std::string msg = h->r.msg;
    const int64_t line = h->r.line, col = h->r.col;
    delete h;
    if (st == gssdf::SDF_FALLBACK)
      return fail(GS_ERR_UNSUPPORTED, "SDF text outside the native reader's subset");
    const int rc = fail(st == gssdf::SDF_PARSE ? GS_ERR_PARSE : GS_ERR_SEMANTIC, msg);
    if (st == gssdf::SDF_PARSE) {
      g_err_line = line;
      g_err_col = col;
    }
    return rc;
  }
  *out = h;
  return GS_OK;
}

int gs_sdf_sizes(const gs_sdf *h, int64_t *num_rows, int64_t *num_pins, int64_t *timescale_fs,
                 int64_t *num_warnings) {
  if (!h || !num_rows || !num_pins || !timescale_fs || !num_warnings)
    return fail(GS_ERR_ARG, "null argument");
  *num_rows = (int64_t)h->r.arc_rows.size() / 2;
  *num_pins = (int64_t)h->r.pin_ic.size();
  *timescale_fs = h->r.timescale_fs;
  *num_warnings = (int64_t)h->r.warnings.size();
  return GS_OK;
}

int gs_sdf_copy(const gs_sdf *h, int64_t *arc_rows, int64_t *pin_ic) {
  if (!h || (!arc_rows && !h->r.arc_rows.empty()) || (!pin_ic && !h->r.pin_ic.empty()))
    return fail(GS_ERR_ARG, "null argument");
  std::copy(h->r.arc_rows.begin(), h->r.arc_rows.end(), arc_rows);
  std::copy(h->r.pin_ic.begin(), h->r.pin_ic.end(), pin_ic);
  return GS_OK;
}

const char *gs_sdf_warning(const gs_sdf *h, int64_t i) {
  if (!h || i < 0 || i >= (int64_t)h->r.warnings.size()) return nullptr;
  return h->r.warnings[(size_t)i].c_str();
}

int gs_sdf_destroy(gs_sdf *h) {
  delete h;
  return GS_OK;
}

// ---- SAIF writer

int gs_saif_format(const char *names, const int64_t *name_off, int64_t num_nets,
                   const int64_t *t0, const int64_t *t1, const int64_t *tc, const int64_t *ig,
                   int64_t duration, const char *design_name, const char *saif_version,
                   int include_ig, char *out, int64_t out_cap, int64_t *out_len) {
  if (!out_len || !design_name || !saif_version || num_nets < 0 ||
      (num_nets > 0 && (!names || !name_off || !t0 || !t1 || !tc || (include_ig && !ig))))
    return fail(GS_ERR_ARG, "null SAIF writer argument");
  std::string head;
  head += "(SAIFILE\n  (SAIFVERSION \"";
  head += saif_version;
  head += "\")\n  (DIRECTION \"backward\")\n  (DESIGN \"";
  head += design_name;
  head += "\")\n  (TIMESCALE 1 fs)\n  (DURATION ";
  head += std::to_string(duration);
  head += ")\n  (INSTANCE ";
  head += design_name;
  head += "\n    (NET\n";
  static const char tail[] = "    )\n  )\n)\n";
  // size: every byte of a name may double; 20 digits + sign per number
  int64_t need = (int64_t)head.size() + (int64_t)sizeof(tail) - 1;
  for (int64_t i = 0; i < num_nets; ++i)
    need += 2 * (name_off[i + 1] - name_off[i]) + 128 + 4 * 21;
  if (!out || out_cap < need) {
    *out_len = need;
    return fail(GS_ERR_ARG, "SAIF output buffer too small");
  }
  char *p = out;
  auto put = [&](const char *s, size_t n) { memcpy(p, s, n); p += n; };
  auto lit = [&](const char *s) { put(s, strlen(s)); };
  auto num = [&](int64_t v) { p = std::to_chars(p, p + 21, (long long)v).ptr; };
  put(head.data(), head.size());
  for (int64_t i = 0; i < num_nets; ++i) {
    lit("      (");
    for (int64_t j = name_off[i]; j < name_off[i + 1]; ++j) {
      const char c = names[j];
      if (c == '[' || c == ']' || c == '/' || c == '\\') *p++ = '\\';
      *p++ = c;
    }
    lit("\n        (T0 ");
    num(t0[i]);
    lit(") (T1 ");
    num(t1[i]);
    lit(") (TX 0)\n        (TC ");
    num(tc[i]);
    if (include_ig) {
      lit(") (IG ");
      num(ig[i]);
    }
    lit(")\n      )\n");
  }
  put(tail, sizeof(tail) - 1);
  *out_len = p - out;
  return GS_OK;
}

}  // extern "C"

// =========================================================================
// VCD writer (report.py:144-214)

struct gs_vcdw {
  gsvcd::NameTable names;
  std::vector<int8_t> last;
  std::string text;
  int64_t num = 0;
};

extern "C" {

int gs_vcdw_create(const char *names, const int64_t *name_off, int64_t num_names,
                   const char *design_name, gs_vcdw **out) {
  if (!out || num_names < 0 || (num_names && (!names || !name_off)) || !design_name)
    return fail(GS_ERR_ARG, "bad VCD writer arguments");
  *out = nullptr;
  for (int64_t i = 0; i < num_names; ++i)
    if (name_off[i + 1] < name_off[i]) return fail(GS_ERR_ARG, "name offsets not monotone");
  gs_vcdw *w = new gs_vcdw();
  w->num = num_names;
  w->names.build(names, name_off, num_names);
  w->last.assign(w->names.id.size(), (int8_t)-1);
  gsvcd::header(w->text, names, name_off, num_names, w->names, design_name);
  *out = w;
  return GS_OK;
}

int gs_vcdw_feed(gs_vcdw *w, const uint8_t *net_src, const int64_t *net_row,
                 const gs_wave_src *src, const int64_t *boundaries, int64_t w_lo, int64_t w_hi) {
  if (!w || !src || !boundaries || w_hi < w_lo || (w->num && (!net_src || !net_row)))
    return fail(GS_ERR_ARG, "bad VCD feed arguments");
  gsvcd::Source S[2];
  for (int k = 0; k < 2; ++k)
    S[k] = {src[k].buf, src[k].offsets, src[k].counts, src[k].initials, src[k].cols,
            src[k].col0, src[k].n_buf};
  for (int64_t i = 0; i < w->num; ++i) {
    const gsvcd::Source &q = S[net_src[i] ? 1 : 0];
    if (!q.offsets || !q.counts || !q.initials || net_row[i] < 0 || q.col0 < 0 ||
        q.col0 + (w_hi - w_lo) > q.cols)
      return fail(GS_ERR_ARG, "VCD feed: waveform source does not cover the net / windows");
  }
  if (!gsvcd::feed(w->text, w->num, net_src, net_row, S, boundaries, w_lo, w_hi, w->names,
                   w->last))
    return fail(GS_ERR_ARG, "VCD feed: waveform region outside its buffer");
  return GS_OK;
}

int gs_vcdw_finish(gs_vcdw *w, int64_t end_time) {
  if (!w) return fail(GS_ERR_ARG, "null VCD writer");
  w->text.push_back('#');
  gsvcd::put_int(w->text, end_time);
  w->text.push_back('\n');
  return GS_OK;
}

int gs_vcdw_take(gs_vcdw *w, char *buf, int64_t cap, int64_t *len) {
  if (!w || !len) return fail(GS_ERR_ARG, "bad VCD take arguments");
  *len = (int64_t)w->text.size();
  if (!buf) return GS_OK;
  if (cap < *len) return fail(GS_ERR_ARG, "VCD text buffer too small");
  memcpy(buf, w->text.data(), w->text.size());
  w->text.clear();
  return GS_OK;
}

int gs_vcdw_destroy(gs_vcdw *w) {
  delete w;
  return GS_OK;
}

}  // extern "C"

// =========================================================================
// netlist JSON reader (netlist.py:190-275)

struct gs_netlist {
  gsnl::Result r;
};


extern "C" {

int gs_netlist_parse(const char *text, int64_t len, const char *cell_names,
                     const int64_t *cell_name_off, int64_t num_cells, const char *pin_names,
                     const int64_t *pin_name_off, const int64_t *cell_pin_first,
                     const char *cell_outputs, const int64_t *cell_output_off, gs_netlist **out) {
  if (!out || (len && !text) || num_cells < 0 ||
      (num_cells && (!cell_names || !cell_name_off || !cell_pin_first || !cell_outputs ||
                     !cell_output_off)))
    return fail(GS_ERR_ARG, "bad netlist reader arguments");
  *out = nullptr;
  std::vector<gsnl::Cell> cells((size_t)num_cells);
  for (int64_t c = 0; c < num_cells; ++c) {
    cells[c].name.assign(cell_names + cell_name_off[c], cell_name_off[c + 1] - cell_name_off[c]);
    cells[c].out.assign(cell_outputs + cell_output_off[c],
                        cell_output_off[c + 1] - cell_output_off[c]);
    for (int64_t q = cell_pin_first[c]; q < cell_pin_first[c + 1]; ++q)
      cells[c].pins.emplace_back(pin_names + pin_name_off[q], pin_name_off[q + 1] - pin_name_off[q]);
  }
  gs_netlist *h = new gs_netlist();
  if (!gsnl::read(text, (size_t)len, cells, h->r)) {
    delete h;
    return fail(GS_ERR_UNSUPPORTED, "netlist document outside the native reader's scope");
  }
  *out = h;
  return GS_OK;
}

int gs_netlist_sizes(const gs_netlist *h, int64_t *counts, int64_t *bytes) {
  if (!h || !counts || !bytes) return fail(GS_ERR_ARG, "bad netlist size arguments");
  const gsnl::Result &r = h->r;
  counts[0] = (int64_t)r.pis.size();
  counts[1] = (int64_t)r.pos.size();
  counts[2] = (int64_t)r.gates.size();
  counts[3] = (int64_t)r.pin_net.size();
  bytes[0] = (int64_t)r.name.size();
  bytes[1] = (int64_t)r.pis.blob.size();
  bytes[2] = (int64_t)r.pos.blob.size();
  bytes[3] = (int64_t)r.gates.blob.size();
  bytes[4] = (int64_t)r.outs.blob.size();
  return GS_OK;
}

int gs_netlist_copy(const gs_netlist *h, char *name, char *pis, int64_t *pis_off, char *pos,
                    int64_t *pos_off, char *gates, int64_t *gates_off, char *outs,
                    int64_t *outs_off, int64_t *gate_cell, int64_t *pin_off, int64_t *pin_net) {
  if (!h) return fail(GS_ERR_ARG, "null netlist");
  const gsnl::Result &r = h->r;
  struct { const gsnl::Names *v; char *b; int64_t *o; } lists[] = {
      {&r.pis, pis, pis_off}, {&r.pos, pos, pos_off}, {&r.gates, gates, gates_off},
      {&r.outs, outs, outs_off}};
  for (auto &L : lists) {
    if (L.b && !L.v->blob.empty()) memcpy(L.b, L.v->blob.data(), L.v->blob.size());
    if (L.o) memcpy(L.o, L.v->off.data(), sizeof(int64_t) * L.v->off.size());
  }
  if (name && !r.name.empty()) memcpy(name, r.name.data(), r.name.size());
  if (gate_cell && !r.gate_cell.empty())
    memcpy(gate_cell, r.gate_cell.data(), sizeof(int64_t) * r.gate_cell.size());
  if (pin_off) memcpy(pin_off, r.pin_off.data(), sizeof(int64_t) * r.pin_off.size());
  if (pin_net && !r.pin_net.empty())
    memcpy(pin_net, r.pin_net.data(), sizeof(int64_t) * r.pin_net.size());
  return GS_OK;
}

int gs_netlist_destroy(gs_netlist *h) {
  delete h;
  return GS_OK;
}

}  // extern "C"

// =========================================================================
// NCCL: the cross-GPU merge of the per-net sums (
// ActivityStats.merge, report.py:46-54).  libnccl.so.2 is bound at run time
// (dlopen), so the process's NCCL -- the one torch.distributed loaded, when
// it did -- is the one used, and the library has no link-time NCCL dependency.

namespace {
struct NcclApi {
  ncclResult_t (*getUniqueId)(ncclUniqueId *);
  ncclResult_t (*commInitRank)(ncclComm_t *, int, ncclUniqueId, int);
  ncclResult_t (*commDestroy)(ncclComm_t);
  ncclResult_t (*allReduce)(const void *, void *, size_t, ncclDataType_t, ncclRedOp_t,
                            ncclComm_t, cudaStream_t);
  const char *(*getErrorString)(ncclResult_t);
};

int nccl_api(NcclApi **out) {
  static NcclApi api;
  static int state = 0;  // 0 unloaded, 1 ok, -1 unavailable
  if (state == 0) {
    void *h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    state = -1;
    if (h) {
      api.getUniqueId = (decltype(api.getUniqueId))dlsym(h, "ncclGetUniqueId");
      api.commInitRank = (decltype(api.commInitRank))dlsym(h, "ncclCommInitRank");
      api.commDestroy = (decltype(api.commDestroy))dlsym(h, "ncclCommDestroy");
      api.allReduce = (decltype(api.allReduce))dlsym(h, "ncclAllReduce");
      api.getErrorString = (decltype(api.getErrorString))dlsym(h, "ncclGetErrorString");
      if (api.getUniqueId && api.commInitRank && api.commDestroy && api.allReduce &&
          api.getErrorString)
        state = 1;
    }
  }
  if (state != 1) return fail(GS_ERR_CUDA, "libnccl.so.2 is not available");
  *out = &api;
  return GS_OK;
}

int nccl_fail(NcclApi *api, ncclResult_t r, const char *what) {
  return fail(GS_ERR_CUDA, std::string(what) + ": " + api->getErrorString(r));
}
}  // namespace

extern "C" {

int gs_nccl_unique_id(uint8_t *id) {
  if (!id) return fail(GS_ERR_ARG, "null id buffer");
  NcclApi *api;
  TRY(nccl_api(&api));
  ncclUniqueId u;
  ncclResult_t r = api->getUniqueId(&u);
  if (r != ncclSuccess) return nccl_fail(api, r, "ncclGetUniqueId");
  static_assert(sizeof(u.internal) == GS_NCCL_ID_BYTES, "NCCL unique id size");
  memcpy(id, u.internal, GS_NCCL_ID_BYTES);
  return GS_OK;
}

int gs_nccl_comm_create(const uint8_t *id, int nranks, int rank, int device, void **comm) {
  if (!id || !comm || nranks < 1 || rank < 0 || rank >= nranks)
    return fail(GS_ERR_ARG, "bad NCCL communicator arguments");
  *comm = nullptr;
  NcclApi *api;
  TRY(nccl_api(&api));
  TRY(use_device(device));
  ncclUniqueId u;
  memcpy(u.internal, id, GS_NCCL_ID_BYTES);
  ncclComm_t c = nullptr;
  ncclResult_t r = api->commInitRank(&c, nranks, u, rank);
  if (r != ncclSuccess) return nccl_fail(api, r, "ncclCommInitRank");
  *comm = (void *)c;
  return GS_OK;
}

int gs_nccl_comm_destroy(void *comm) {
  if (!comm) return GS_OK;
  NcclApi *api;
  TRY(nccl_api(&api));
  api->commDestroy((ncclComm_t)comm);
  return GS_OK;
}

int gs_allreduce_stats(int64_t *acc_dev, int64_t n, void *comm, void *stream) {
  if (!acc_dev || n < 0 || !comm) return fail(GS_ERR_ARG, "bad all-reduce arguments");
  NcclApi *api;
  TRY(nccl_api(&api));
  ncclResult_t r = api->allReduce(acc_dev, acc_dev, (size_t)n, ncclInt64, ncclSum,
                                  (ncclComm_t)comm, (cudaStream_t)stream);
  if (r != ncclSuccess) return nccl_fail(api, r, "ncclAllReduce");
  return GS_OK;
}

}  // extern "C"
