// synth.cuh -- the benchmark configs' synthetic stimulus, generated on the
// device (counter-based RNG, so any window range of a config is
// reproducible independently -- a window shard, or the CPU baseline's sample).
// Bit-identical to paper_2203_06117_b200/synth.py stimulus_arrays():
//   key = seed << 56 ^ input << 32 ^ window,  h1 = splitmix64(key),
//   h2 = splitmix64(h1 ^ 0xD1B54A32D192ED03)
//   input p toggles in window w  iff  (h1 >> 11) < thr_p  (= u < alpha with
//   u = (h1 >> 11) * 2^-53, thr = ceil(alpha * 2^53)), at
//   w * period + lo_p + h2 % span_p;
//   initial value = splitmix64(seed * 1000003 + p) & 1, xor the parity of
//   the input's toggles in windows [0, w_lo).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace gs {

struct SynthArgs {
  int P, ppis;
  unsigned long long seed, ppi_thr, pi_thr;
  long long period, ppi_lo, ppi_span, pi_lo, pi_span;
  long long w_lo, w_hi;
};

__device__ __forceinline__ unsigned long long splitmix64(unsigned long long x) {
  x += 0x9E3779B97F4A7C15ull;
  unsigned long long z = x;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

// warp per input: toggles in [w_lo, w_hi) and the initial value at w_lo
__global__ void synth_count(SynthArgs A, long long *__restrict__ cnt,
                            unsigned char *__restrict__ init) {
  const unsigned lane = threadIdx.x & 31u;
  const int warps = gridDim.x * (blockDim.x / 32);
  for (int p = blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32; p < A.P; p += warps) {
    const unsigned long long base = (A.seed << 56) ^ ((unsigned long long)p << 32);
    const unsigned long long thr = p < A.ppis ? A.ppi_thr : A.pi_thr;
    long long c = 0;
    unsigned par = 0;
    for (long long w = lane; w < A.w_lo; w += 32)
      par ^= (splitmix64(base ^ (unsigned long long)w) >> 11) < thr ? 1u : 0u;
    for (long long w = A.w_lo + lane; w < A.w_hi; w += 32)
      c += (splitmix64(base ^ (unsigned long long)w) >> 11) < thr ? 1 : 0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      c += __shfl_xor_sync(0xffffffffu, c, o);
      par ^= __shfl_xor_sync(0xffffffffu, par, o);
    }
    if (lane == 0) {
      cnt[p] = c;
      init[p] = (unsigned char)((splitmix64(A.seed * 1000003ull + (unsigned long long)p) & 1ull) ^
                                (par & 1u));
    }
  }
}

// warp per input: the toggle times, in window order, at pi_off[p]
__global__ void synth_fill(SynthArgs A, const long long *__restrict__ pi_off,
                           long long *__restrict__ times) {
  const unsigned lane = threadIdx.x & 31u;
  const int warps = gridDim.x * (blockDim.x / 32);
  for (int p = blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32; p < A.P; p += warps) {
    const unsigned long long base = (A.seed << 56) ^ ((unsigned long long)p << 32);
    const bool ppi = p < A.ppis;
    const unsigned long long thr = ppi ? A.ppi_thr : A.pi_thr;
    const unsigned long long lo = (unsigned long long)(ppi ? A.ppi_lo : A.pi_lo);
    long long sp = ppi ? A.ppi_span : A.pi_span;
    const unsigned long long span = (unsigned long long)(sp < 1 ? 1 : sp);
    long long pos = pi_off[p];
    for (long long w0 = A.w_lo; w0 < A.w_hi; w0 += 32) {
      const long long w = w0 + lane;
      unsigned long long h1 = 0;
      bool hit = false;
      if (w < A.w_hi) {
        h1 = splitmix64(base ^ (unsigned long long)w);
        hit = (h1 >> 11) < thr;
      }
      const unsigned b = __ballot_sync(0xffffffffu, hit);
      if (hit) {
        const unsigned long long h2 = splitmix64(h1 ^ 0xD1B54A32D192ED03ull);
        times[pos + __popc(b & ((1u << lane) - 1u))] =
            w * A.period + (long long)(lo + h2 % span);
      }
      pos += __popc(b);
    }
  }
}

// thread per window: input toggles of window w (the activity weight that
// window shards are balanced by)
__global__ void synth_window_counts(SynthArgs A, long long *__restrict__ out) {
  for (long long w = A.w_lo + (long long)blockIdx.x * blockDim.x + threadIdx.x; w < A.w_hi;
       w += (long long)gridDim.x * blockDim.x) {
    long long c = 0;
    for (int p = 0; p < A.P; ++p) {
      const unsigned long long base = (A.seed << 56) ^ ((unsigned long long)p << 32);
      const unsigned long long thr = p < A.ppis ? A.ppi_thr : A.pi_thr;
      c += (splitmix64(base ^ (unsigned long long)w) >> 11) < thr ? 1 : 0;
    }
    out[w - A.w_lo] = c;
  }
}

__global__ void synth_bounds(long long *__restrict__ bnd, long long w_lo, long long W,
                             long long period) {
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i <= W;
       i += (long long)gridDim.x * blockDim.x)
    bnd[i] = (w_lo + i) * period;
}

}  // namespace gs
