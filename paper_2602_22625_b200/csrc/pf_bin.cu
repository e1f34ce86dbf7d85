// K1 preprocess + K2 tile binning.
//
// Reference: bin_tiles (pkg/src/primfit/raster.py:227-265) walks primitives in
// ascending z, computes a conservative square bbox of half side
// r = scale*hypot(1, max(1, q)) + padding (bbox_half_side, raster.py:222-224),
// clips it to the canvas in float64 (ceil/floor, raster.py:248-253) and appends
// the primitive index to every tile the clipped pixel range touches.
//
// B200 restatement: one thread per z position computes the bbox (float64,
// no FMA, same rounding as Python) and the per-primitive tile count; an
// exclusive scan in z order gives each primitive a contiguous slot range; the
// fill kernel writes (tile) keys + (primitive) values in z order; a STABLE
// LSD radix sort on the tile key (CUB onesweep, only ceil(log2(tiles+1)) bits)
// groups entries per tile while keeping z order inside each tile.  Per-tile
// counts (histogram via atomics in K1) are scanned into the CSR offsets.
// The result is bit-identical to the reference's offsets/indices.
#include <cub/cub.cuh>

#include "../../include/primfit_b200.h"
#include "pf_common.cuh"

namespace pf {

struct BinScratch {
  int32_t* pcount;   // [n+1] per-z-position tile count (last = 0)
  int32_t* poff;     // [n+1] exclusive scan
  int4* rect;        // [n] band-clipped tile rect (tx0, ty0, tx1, ty1), empty: tx0 > tx1
  int32_t* zprim;    // [n] primitive index per z position (copy of zorder)
  int32_t* tcount;   // [n_tiles+1] per-tile counts (last = 0)
  uint32_t* keys_in;   // [cap]
  uint32_t* keys_out;  // [cap]
  int32_t* vals_in;    // [cap]
  void* cub_tmp;
  size_t cub_bytes;
  size_t total;
};

static size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

static int end_bit_for(int n_tiles) {
  int b = 1;
  while ((1u << b) <= (unsigned)n_tiles) ++b;  // sentinel key == n_tiles must fit
  return b;
}

static size_t cub_temp_bytes(int n, int n_tiles, int cap) {
  size_t a = 0, b = 0, c = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, a, (int32_t*)nullptr, (int32_t*)nullptr, n + 1);
  cub::DeviceScan::ExclusiveSum(nullptr, b, (int32_t*)nullptr, (int32_t*)nullptr, n_tiles + 1);
  if (cap > 0)
    cub::DeviceRadixSort::SortPairs(nullptr, c, (uint32_t*)nullptr, (uint32_t*)nullptr,
                                    (int32_t*)nullptr, (int32_t*)nullptr, cap, 0,
                                    end_bit_for(n_tiles));
  size_t m = a > b ? a : b;
  return m > c ? m : c;
}

static BinScratch carve(void* base, int n, int n_tiles, int cap) {
  BinScratch s;
  char* p = (char*)base;
  size_t off = 0;
  auto take = [&](size_t bytes) {
    char* q = p ? p + off : nullptr;
    off = align_up(off + bytes, 256);
    return (void*)q;
  };
  s.pcount = (int32_t*)take(sizeof(int32_t) * (n + 1));
  s.poff = (int32_t*)take(sizeof(int32_t) * (n + 1));
  s.rect = (int4*)take(sizeof(int4) * (n > 0 ? n : 1));
  s.zprim = (int32_t*)take(sizeof(int32_t) * (n > 0 ? n : 1));
  s.tcount = (int32_t*)take(sizeof(int32_t) * (n_tiles + 1));
  s.keys_in = (uint32_t*)take(sizeof(uint32_t) * (cap > 0 ? cap : 1));
  s.keys_out = (uint32_t*)take(sizeof(uint32_t) * (cap > 0 ? cap : 1));
  s.vals_in = (int32_t*)take(sizeof(int32_t) * (cap > 0 ? cap : 1));
  s.cub_bytes = cub_temp_bytes(n, n_tiles, cap);
  s.cub_tmp = take(s.cub_bytes);
  s.total = off;
  return s;
}

struct PreArgs {
  const double* params;
  const int32_t* tid;
  const int32_t* zorder;
  int n;
  const int32_t* tpl_base;
  const int32_t* tpl_w;
  const int32_t* tpl_h;
  const double* tpl_q;
  const double* tpl_hyp;
  double alpha_max, mu_blend, padding;
  int W, H, tile, ntx, ty_begin, ty_end;
  RecF* recf;
  RecB* recb;
  BinScratch s;
};

// K1: one thread per z position j (primitive zorder[j]).
__global__ void __launch_bounds__(256) k_preprocess(PreArgs a) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j == 0) a.s.pcount[a.n] = 0;
  if (j >= a.n) return;
  const int i = __ldg(a.zorder + j);
  a.s.zprim[j] = i;
  const double* p = a.params + (size_t)i * 8;
  const double x = p[0], y = p[1], s = p[2], rot = p[3], nu = p[4];
  const double cl0 = p[5], cl1 = p[6], cl2 = p[7];
  const int t = __ldg(a.tid + i);
  const int wt = __ldg(a.tpl_w + t), ht = __ldg(a.tpl_h + t);
  const double q = __ldg(a.tpl_q + t);
  const double hyp = __ldg(a.tpl_hyp + t);

  double st, ct;
  sincos(rot, &st, &ct);
  const double sig = sigmoid(nu);
  const double sc0 = sigmoid(cl0), sc1 = sigmoid(cl1), sc2 = sigmoid(cl2);
  const double omm = __dsub_rn(1.0, a.mu_blend);

  RecF rf;
  rf.px = x;
  rf.py = y;
  rf.ct = ct;
  rf.st = st;
  rf.s = s;
  rf.sq = __dmul_rn(s, q);
  rf.sa = __dmul_rn(a.alpha_max, sig);
  rf.c0 = __dmul_rn(omm, sc0);
  rf.c1 = __dmul_rn(omm, sc1);
  rf.c2 = __dmul_rn(omm, sc2);
  rf.base = __ldg(a.tpl_base + t);
  rf.wt = wt;
  rf.ht = ht;
  rf.tid = t;
  a.recf[i] = rf;

  RecB rb;
  rb.sd = a.alpha_max * sig * (1.0 - sig);
  rb.cd0 = sc0 * (1.0 - sc0);
  rb.cd1 = sc1 * (1.0 - sc1);
  rb.cd2 = sc2 * (1.0 - sc2);
  const double sqv = rf.sq;
  rb.gxu = -ct / s;
  rb.gxv = st / sqv;
  rb.gyu = -st / s;
  rb.gyv = -ct / sqv;
  rb.inv_s = 1.0 / s;
  rb.q = q;
  rb.inv_q = 1.0 / q;
  rb.one_minus_mu = omm;
  a.recb[i] = rb;

  // bbox, float64 with Python's rounding: r = s*hyp + pad, ceil(x-r), floor(x+r)
  const double r = __dadd_rn(__dmul_rn(s, hyp), a.padding);
  double lo_x = ceil(__dsub_rn(x, r)), hi_x = floor(__dadd_rn(x, r));
  double lo_y = ceil(__dsub_rn(y, r)), hi_y = floor(__dadd_rn(y, r));
  lo_x = fmax(lo_x, 0.0);
  lo_y = fmax(lo_y, 0.0);
  hi_x = fmin(hi_x, (double)(a.W - 1));
  hi_y = fmin(hi_y, (double)(a.H - 1));
  int4 rc = make_int4(1, 1, 0, 0);  // empty
  int cnt = 0;
  // NaN-safe: every comparison with NaN is false -> treated as empty
  if (lo_x <= hi_x && lo_y <= hi_y) {
    const int tx0 = (int)lo_x / a.tile, tx1 = (int)hi_x / a.tile;
    int ty0 = (int)lo_y / a.tile, ty1 = (int)hi_y / a.tile;
    ty0 = max(ty0, a.ty_begin);
    ty1 = min(ty1, a.ty_end - 1);
    if (ty0 <= ty1) {
      rc = make_int4(tx0, ty0, tx1, ty1);
      cnt = (tx1 - tx0 + 1) * (ty1 - ty0 + 1);
      for (int ty = ty0; ty <= ty1; ++ty) {
        const int row = (ty - a.ty_begin) * a.ntx;
        for (int tx = tx0; tx <= tx1; ++tx) atomicAdd(a.s.tcount + row + tx, 1);
      }
    }
  }
  a.s.rect[j] = rc;
  a.s.pcount[j] = cnt;
}

struct FillArgs {
  int n, cap, ntx, ty_begin, n_tiles;
  BinScratch s;
  int32_t* status;
};

// Fill (tile key, primitive value) pairs in z order; pad [K, cap) with the
// sentinel key n_tiles so a fixed-size sort keeps graph capture possible.
__global__ void __launch_bounds__(256) k_fill(FillArgs a) {
  const int g = blockIdx.x * blockDim.x + threadIdx.x;
  const int K = a.s.poff[a.n];
  if (g == 0) {
    a.status[0] = K;
    a.status[1] = K > a.cap ? 1 : 0;
  }
  if (g < a.n) {
    const int4 rc = a.s.rect[g];
    const int i = a.s.zprim[g];
    int off = a.s.poff[g];
    for (int ty = rc.y; ty <= rc.w; ++ty) {
      const int row = (ty - a.ty_begin) * a.ntx;
      for (int tx = rc.x; tx <= rc.z; ++tx) {
        if (off < a.cap) {
          a.s.keys_in[off] = (uint32_t)(row + tx);
          a.s.vals_in[off] = i;
        }
        ++off;
      }
    }
  }
  for (int k = K + g; k < a.cap; k += gridDim.x * blockDim.x) {
    a.s.keys_in[k] = (uint32_t)a.n_tiles;
    a.s.vals_in[k] = 0;
  }
}

}  // namespace pf

using namespace pf;

extern "C" size_t pf_bin_scratch_bytes(int n, int n_tiles, int capacity) {
  if (n < 0 || n_tiles < 0 || capacity < 0) return 0;
  return carve(nullptr, n, n_tiles, capacity).total;
}

extern "C" int pf_preprocess(const double* params, const int32_t* template_id,
                             const int32_t* zorder, int n, const int32_t* tpl_base,
                             const int32_t* tpl_w, const int32_t* tpl_h, const double* tpl_q,
                             const double* tpl_hyp, int n_tpl, double alpha_max, double mu_blend,
                             double padding, int W, int H, int tile, int ty_begin, int ty_end,
                             int capacity, void* rec, void* scratch, size_t scratch_bytes,
                             void* stream) {
  if (n < 0 || W < 1 || H < 1 || tile < 1 || n_tpl < 0 || capacity < 0) return PF_ERR_ARG;
  const int ntx = div_up(W, tile), nty = div_up(H, tile);
  if (ty_begin < 0 || ty_end > nty || ty_begin > ty_end) return PF_ERR_ARG;
  const int n_tiles = (ty_end - ty_begin) * ntx;
  if (!scratch || scratch_bytes < pf_bin_scratch_bytes(n, n_tiles, capacity)) return PF_ERR_SCRATCH;
  if (n > 0 && (!params || !template_id || !zorder || !rec || !tpl_base || !tpl_w || !tpl_h ||
                !tpl_q || !tpl_hyp))
    return PF_ERR_ARG;
  cudaStream_t st = (cudaStream_t)stream;
  PreArgs a;
  a.params = params;
  a.tid = template_id;
  a.zorder = zorder;
  a.n = n;
  a.tpl_base = tpl_base;
  a.tpl_w = tpl_w;
  a.tpl_h = tpl_h;
  a.tpl_q = tpl_q;
  a.tpl_hyp = tpl_hyp;
  a.alpha_max = alpha_max;
  a.mu_blend = mu_blend;
  a.padding = padding;
  a.W = W;
  a.H = H;
  a.tile = tile;
  a.ntx = ntx;
  a.ty_begin = ty_begin;
  a.ty_end = ty_end;
  a.recf = (RecF*)rec;
  a.recb = (RecB*)((char*)rec + sizeof(RecF) * (size_t)n);
  a.s = carve(scratch, n, n_tiles, capacity);
  cudaError_t e = cudaMemsetAsync(a.s.tcount, 0, sizeof(int32_t) * (n_tiles + 1), st);
  if (e != cudaSuccess) return (int)e;
  const int blocks = div_up(n > 0 ? n : 1, 256);
  k_preprocess<<<blocks, 256, 0, st>>>(a);
  return (int)cudaGetLastError();
}

extern "C" int pf_bin(int n, int W, int H, int tile, int ty_begin, int ty_end, int capacity,
                      void* scratch, size_t scratch_bytes, int32_t* bin_off, int32_t* bin_idx,
                      int32_t* status, void* stream) {
  if (n < 0 || W < 1 || H < 1 || tile < 1 || capacity < 0) return PF_ERR_ARG;
  const int ntx = div_up(W, tile), nty = div_up(H, tile);
  if (ty_begin < 0 || ty_end > nty || ty_begin > ty_end) return PF_ERR_ARG;
  if (!bin_off || !status || (capacity > 0 && !bin_idx)) return PF_ERR_ARG;
  const int n_tiles = (ty_end - ty_begin) * ntx;
  if (!scratch || scratch_bytes < pf_bin_scratch_bytes(n, n_tiles, capacity)) return PF_ERR_SCRATCH;
  cudaStream_t st = (cudaStream_t)stream;
  BinScratch s = carve(scratch, n, n_tiles, capacity);
  size_t tb = s.cub_bytes;
  cudaError_t e =
      cub::DeviceScan::ExclusiveSum(s.cub_tmp, tb, s.pcount, s.poff, n + 1, st);
  if (e != cudaSuccess) return (int)e;
  FillArgs f;
  f.n = n;
  f.cap = capacity;
  f.ntx = ntx;
  f.ty_begin = ty_begin;
  f.n_tiles = n_tiles;
  f.s = s;
  f.status = status;
  int work = n > capacity ? n : capacity;
  int blocks = div_up(work > 0 ? work : 1, 256);
  if (blocks > 148 * 16) blocks = 148 * 16;
  if (blocks < div_up(n > 0 ? n : 1, 256)) blocks = div_up(n, 256);
  k_fill<<<blocks, 256, 0, st>>>(f);
  e = cudaGetLastError();
  if (e != cudaSuccess) return (int)e;
  if (capacity > 0) {
    tb = s.cub_bytes;
    e = cub::DeviceRadixSort::SortPairs(s.cub_tmp, tb, s.keys_in, s.keys_out, s.vals_in, bin_idx,
                                        capacity, 0, end_bit_for(n_tiles), st);
    if (e != cudaSuccess) return (int)e;
  }
  tb = s.cub_bytes;
  e = cub::DeviceScan::ExclusiveSum(s.cub_tmp, tb, s.tcount, bin_off, n_tiles + 1, st);
  return (int)e;
}
