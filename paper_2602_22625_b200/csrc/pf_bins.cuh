// Binning scratch layout and block-wide scan helpers shared by the kernels.
#pragma once

#include "pf_common.cuh"

namespace pf {

struct BinScratch {
  int4* rect;        // [n] band-clipped tile rect per z position (tx0, ty0, tx1, ty1)
  int32_t* zprim;    // [n] primitive index per z position (static, set by pf_scratch_init)
  int2* rowlist;     // [capacity] per-row z-ordered lists: (z position, tx0 | tx1 << 16)
  uint32_t* done;    // [4] last-block ticket
  double* fold;      // [prim blocks][3] per-block loss-partial folds (pf_adam_preprocess)
  size_t total;
};

static inline size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

static inline BinScratch carve(void* base, int n, int cap) {
  BinScratch s;
  char* p = (char*)base;
  size_t off = 0;
  auto take = [&](size_t bytes) {
    char* q = p ? p + off : nullptr;
    off = align_up(off + (bytes > 0 ? bytes : 1), 256);
    return (void*)q;
  };
  s.rect = (int4*)take(sizeof(int4) * (size_t)n);
  s.zprim = (int32_t*)take(sizeof(int32_t) * (size_t)n);
  s.rowlist = (int2*)take(sizeof(int2) * (size_t)cap);
  s.done = (uint32_t*)take(sizeof(uint32_t) * 4);
  s.fold = (double*)take(sizeof(double) * 3 * (size_t)((8 * (size_t)n + 255) / 256 + 1));
  s.total = off;
  return s;
}

// Block-wide exclusive scan of one int per thread (<= 1024 threads).
// Returns the exclusive prefix; *total receives the block sum.
__device__ __forceinline__ int block_excl_scan(int v, int* warp_sums, int* total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nw = (blockDim.x + 31) >> 5;
  int x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(kFull, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) warp_sums[warp] = x;
  __syncthreads();
  if (warp == 0) {
    int w = lane < nw ? warp_sums[lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(kFull, w, o);
      if (lane >= o) w += y;
    }
    if (lane < nw) warp_sums[lane] = w;  // inclusive warp prefix
  }
  __syncthreads();
  const int excl_warp = warp > 0 ? warp_sums[warp - 1] : 0;
  *total = warp_sums[nw - 1];
  const int r = excl_warp + x - v;
  __syncthreads();  // warp_sums reusable by the caller afterwards
  return r;
}

}  // namespace pf
