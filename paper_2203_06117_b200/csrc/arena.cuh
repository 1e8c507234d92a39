// arena.cuh -- K5: pack one window chunk's gate waveforms into the
// reference arena layout (allocate_arena + store_pass, waveform.py:321-346,
// simcore.py:382-410) from the single simulation pass.
//
// During an arena run every gate-window's outputs stay in the chunk's pool
// (K4 records where: a_pos), including entries stored and later popped below
// 100 % pathpulse, so `peak` entries per window are kept exactly as the
// reference's store pass leaves them in the region [offset, offset + peak).
// K5 then lays the chunk out gate-major in level order (the arena order),
// absolute int64 times:
//   rowsum   rs[g]   = sum over the chunk's windows of peak[g][w]
//   scan     base[g] = exclusive prefix of rs over the level order
//   pack     region (g, w) at base[g] + prefix over w of peak[g][w]
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "kernels.cuh"

namespace gs {

constexpr int kScanThreads = 256;
constexpr int kScanItems = 4;                          // per thread
constexpr int kScanBlock = kScanThreads * kScanItems;  // items per block

// warp per gate: rs[g] = sum of peak[g][0 .. Wc)
__global__ void arena_rowsum(const long long *__restrict__ peak, int G, int Wc, int Wpad,
                             long long *__restrict__ rs) {
  const unsigned lane = lane_id();
  const int warps = gridDim.x * (blockDim.x / kWarp);
  for (int g = blockIdx.x * (blockDim.x / kWarp) + threadIdx.x / kWarp; g < G; g += warps) {
    long long s = 0;
    for (int w = lane; w < Wc; w += kWarp) s += peak[(size_t)g * Wpad + w];
    s = warp_sum(s);
    if (lane == 0) rs[g] = s;
  }
}

// exclusive scan of rs[order[i]] over i, written back by gate: base[order[i]];
// per block of kScanBlock items, block totals into part[]
__global__ void __launch_bounds__(kScanThreads) scan_blocks(const long long *__restrict__ rs,
                                                            const int *__restrict__ order, int G,
                                                            long long *__restrict__ base,
                                                            long long *__restrict__ part) {
  __shared__ long long wsum[kScanThreads / kWarp];
  const int i0 = blockIdx.x * kScanBlock + threadIdx.x * kScanItems;
  long long v[kScanItems], s = 0;
#pragma unroll
  for (int q = 0; q < kScanItems; ++q) {
    v[q] = i0 + q < G ? rs[order[i0 + q]] : 0;
    s += v[q];
  }
  long long tot;
  long long ex = warp_excl_scan(s, &tot);
  const int warp = threadIdx.x / kWarp;
  if (lane_id() == 0) wsum[warp] = tot;
  __syncthreads();
  long long wb = 0, bt = 0;
  for (int k = 0; k < kScanThreads / kWarp; ++k) {
    wb += k < warp ? wsum[k] : 0;
    bt += wsum[k];
  }
  ex += wb;
#pragma unroll
  for (int q = 0; q < kScanItems; ++q) {
    if (i0 + q < G) base[order[i0 + q]] = ex;
    ex += v[q];
  }
  if (threadIdx.x == 0) part[blockIdx.x] = bt;
}

// one block: exclusive scan of the block totals in place; total in part[n]
__global__ void scan_parts(long long *part, int n) {
  __shared__ long long carry;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  for (int b = 0; b < n; b += blockDim.x) {
    const int i = b + threadIdx.x;
    const long long v = i < n ? part[i] : 0;
    // block-wide scan by warps (blockDim.x = 1024 at most)
    __shared__ long long ws[32];
    long long tot;
    long long ex = warp_excl_scan(v, &tot);
    if (lane_id() == 0) ws[threadIdx.x / kWarp] = tot;
    __syncthreads();
    long long wb = 0, bt = 0;
    for (int k = 0; k < (int)(blockDim.x / kWarp); ++k) {
      wb += k < (int)(threadIdx.x / kWarp) ? ws[k] : 0;
      bt += ws[k];
    }
    if (i < n) part[i] = carry + wb + ex;
    __syncthreads();
    if (threadIdx.x == 0) carry += bt;
    __syncthreads();
  }
  if (threadIdx.x == 0) part[n] = carry;
}

__global__ void __launch_bounds__(kScanThreads) scan_add(long long *__restrict__ base,
                                                         const int *__restrict__ order, int G,
                                                         const long long *__restrict__ part) {
  const int i0 = blockIdx.x * kScanBlock + threadIdx.x * kScanItems;
  const long long add = part[blockIdx.x];
#pragma unroll
  for (int q = 0; q < kScanItems; ++q)
    if (i0 + q < G) base[order[i0 + q]] += add;
}

// warp per gate: copy each window's peak entries (window-relative TS in the
// pool at a_pos) to out[base[g] + prefix] as absolute int64 times
template <typename TS>
__global__ void arena_pack(ChunkDev C, int G, const long long *__restrict__ base,
                           long long *__restrict__ out) {
  const unsigned lane = lane_id();
  const TS *data = reinterpret_cast<const TS *>(C.data);
  const int warps = gridDim.x * (blockDim.x / kWarp);
  for (int g = blockIdx.x * (blockDim.x / kWarp) + threadIdx.x / kWarp; g < G; g += warps) {
    long long off = base[g];
    for (int w0 = 0; w0 < C.Wc; w0 += kWarp) {
      const int w = w0 + (int)lane;
      const size_t gw = (size_t)g * C.Wpad + w;
      const long long pk = w < C.Wc ? C.a_peak[gw] : 0;
      long long tot;
      const long long ex = warp_excl_scan(pk, &tot);
      if (pk > 0) {
        const TS *src = data + C.a_pos[gw];
        const long long b_lo = C.bnd[C.w0 + w];
        for (long long j = 0; j < pk; ++j) out[off + ex + j] = (long long)src[j] + b_lo;
      }
      off += tot;
    }
  }
}

}  // namespace gs
