// Binning scratch layout and block-wide scan helpers shared by the kernels.
#pragma once

#include "pf_common.cuh"

namespace pf {

// Static per-primitive structure (template geometry, z rank), built once by
// pf_scratch_init so that K1 has no dependent loads before its math.
struct __align__(16) PrimInfo {
  int32_t wt, ht, base, pbase;  // template size, atlas base, padded-atlas base
  double q, hyp;                // v-axis aspect, bbox factor hypot(1, max(1, q))
  int32_t zrank, tid, pad0, pad1;
};
static_assert(sizeof(PrimInfo) == 48, "PrimInfo must be 48 bytes");

struct BinScratch {
  int4* rect;        // [n] per z rank: (tx0 | tx1 << 16, ty0, primitive, ty1); empty: ty0 > ty1
  int32_t* zprim;    // [n] primitive index per z position (static, set by pf_scratch_init)
  PrimInfo* pinfo;   // [n] static per-primitive structure (pf_scratch_init)
  int2* rowlist;     // [capacity] per-row z-ordered lists: (z position, tx0 | tx1 << 16)
  uint32_t* done;    // [4] last-block ticket
  double* fold;      // [prim blocks][3] per-block loss-partial folds (pf_adam_preprocess)
  // two-level binning (large n x rows; sized from n_tiles >= rows, 0 = absent)
  int2* rowcnt;      // [row chunks][n_rows] per chunk of kRowChunk z positions: (pairs, entries)
  int4* rowinfo;     // [n_rows] per row (row-list pairs, tile entries, 0, 0)
  size_t total;
};

constexpr int kRowChunk = 128;  // z positions per block of the two-level row pass
constexpr int kMaxRows2 = 1024;  // band rows the two-level path handles

static inline size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

static inline BinScratch carve(void* base, int n, int cap, int n_tiles = 0) {
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
  s.pinfo = (PrimInfo*)take(sizeof(PrimInfo) * (size_t)n);
  s.rowlist = (int2*)take(sizeof(int2) * (size_t)cap);
  s.done = (uint32_t*)take(sizeof(uint32_t) * 4);
  s.fold = (double*)take(sizeof(double) * 3 * (size_t)((8 * (size_t)n + 255) / 256 + 1));
  // (appended: the offsets above do not depend on n_tiles)
  // (rows <= n_tiles, and the two-level path runs only for <= kMaxRows2 rows)
  const size_t chunks = ((size_t)n + kRowChunk - 1) / kRowChunk;
  const size_t rows = n_tiles < kMaxRows2 ? (size_t)n_tiles : (size_t)kMaxRows2;
  s.rowcnt = (int2*)take(sizeof(int2) * chunks * rows);
  s.rowinfo = (int4*)take(sizeof(int4) * (rows + 1));
  s.total = off;
  return s;
}

// Slot binning (the fit step's tile lists without a binning kernel).  K1 puts
// every (tile, primitive) pair of a primitive's band-clipped rect straight into
// the tile's slot array -- slot = atomicAdd(cnt[tile], 1), value = the
// primitive's z rank -- so the lists come out in arrival order; pf_fit_step's
// producer warp sorts each tile's list by z rank before staging it, which gives
// exactly the reference's z-ascending list (z ranks are a permutation).
// Entries past a tile's m slots go to an overflow list of (tile, z rank); the
// producer's general path gathers them.  Sized from the exact capacity bound,
// so nothing is ever dropped (a second scatter of host-edited primitives in
// one step is covered by the factor 2; the error word catches anything else).
enum SlotCtl : int {
  kSlotOvf = 0,     // overflow entries used
  kSlotPool = 1,    // general-path list pool bump (entries), reset per fit step
  kSlotDirty = 2,   // pf_preprocess_sync re-scattered edited primitives this step
  kSlotK = 3,       // total list entries of the fit step being run (published to status[0])
  kSlotGather = 4,  // gather-scratch bump of the producer's general path
  kSlotErr = 5,     // overflow list exhausted (never with the capacity bound)
  kSlotCtlWords = 64
};
struct SlotBins {
  uint32_t* ctl;   // [kSlotCtlWords]
  int32_t* cnt;    // [n_tiles] arrivals (K1 atomics; the producer re-zeroes its tile)
  uint32_t* slot;  // [n_tiles][m] z ranks, arrival order (z-sorted by pf_fit_step's prologue)
  int2* ovf;       // [ovf_cap] (tile, z rank) past a tile's m slots
  uint32_t* pool;  // [pool_cap] (= slot + n_tiles * m) z-sorted general-path lists
  uint32_t* gat;   // [gat_cap] the general path's gather scratch
  int m, n_tiles, ovf_cap, pool_cap, gat_cap;
  size_t total;
};

static inline SlotBins slot_carve(void* base, int n_tiles, int m, int cap) {
  SlotBins s;
  char* p = (char*)base;
  size_t off = 0;
  auto take = [&](size_t bytes) {
    char* q = p ? p + off : nullptr;
    off = align_up(off + (bytes > 0 ? bytes : 1), 256);
    return (void*)q;
  };
  s.m = m;
  s.n_tiles = n_tiles;
  s.ovf_cap = 2 * cap + 64;
  s.pool_cap = cap + 64;
  s.gat_cap = 4 * cap + 256;
  s.ctl = (uint32_t*)take(sizeof(uint32_t) * kSlotCtlWords);
  s.cnt = (int32_t*)take(sizeof(int32_t) * (size_t)n_tiles);
  // (the pool follows the slots: one list array, base tile * m or n_tiles * m + offset)
  s.slot = (uint32_t*)take(sizeof(uint32_t) * ((size_t)n_tiles * (size_t)m + (size_t)s.pool_cap));
  s.pool = s.slot ? s.slot + (size_t)n_tiles * (size_t)m : nullptr;
  s.ovf = (int2*)take(sizeof(int2) * (size_t)s.ovf_cap);
  s.gat = (uint32_t*)take(sizeof(uint32_t) * (size_t)s.gat_cap);
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

// Block-wide exclusive scan of four ints per thread at once (one barrier pass).
__device__ __forceinline__ int4 block_excl_scan4(int4 v, int4* warp_sums, int4* total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nw = (blockDim.x + 31) >> 5;
  int4 x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y0 = __shfl_up_sync(kFull, x.x, o), y1 = __shfl_up_sync(kFull, x.y, o);
    const int y2 = __shfl_up_sync(kFull, x.z, o), y3 = __shfl_up_sync(kFull, x.w, o);
    if (lane >= o) {
      x.x += y0;
      x.y += y1;
      x.z += y2;
      x.w += y3;
    }
  }
  if (lane == 31) warp_sums[warp] = x;
  __syncthreads();
  if (warp == 0) {
    int4 w = lane < nw ? warp_sums[lane] : make_int4(0, 0, 0, 0);
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y0 = __shfl_up_sync(kFull, w.x, o), y1 = __shfl_up_sync(kFull, w.y, o);
      const int y2 = __shfl_up_sync(kFull, w.z, o), y3 = __shfl_up_sync(kFull, w.w, o);
      if (lane >= o) {
        w.x += y0;
        w.y += y1;
        w.z += y2;
        w.w += y3;
      }
    }
    if (lane < nw) warp_sums[lane] = w;  // inclusive warp prefix
  }
  __syncthreads();
  const int4 ew = warp > 0 ? warp_sums[warp - 1] : make_int4(0, 0, 0, 0);
  *total = warp_sums[nw - 1];
  const int4 r = make_int4(ew.x + x.x - v.x, ew.y + x.y - v.y, ew.z + x.z - v.z, ew.w + x.w - v.w);
  __syncthreads();
  return r;
}

}  // namespace pf
