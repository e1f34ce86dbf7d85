// K1 preprocess + K2 tile binning.
//
// Reference: bin_tiles (pkg/src/primfit/raster.py:227-265) walks primitives in
// ascending z, computes a conservative square bbox of half side
// r = scale*hypot(1, max(1, q)) + padding (bbox_half_side, raster.py:222-224),
// clips it to the canvas in float64 (ceil/floor, raster.py:248-253) and appends
// the primitive index to every tile the clipped pixel range touches.
//
// B200 restatement (three launches, no host sync, no sort scratch):
//   K1  k_preprocess   one thread per z position: primitive records, float64
//                      bbox with Python's rounding, per-tile and per-tile-row
//                      counts (atomics; final values are order independent).
//   K2a k_bin_scan     block 0: exclusive scan of the per-tile counts -> CSR
//                      offsets (TileBins.offsets) + K + overflow flag;
//                      blocks 1..rows: for each tile row, a STABLE block-wide
//                      compaction of the z-ordered primitive stream (contiguous
//                      per-thread chunks + one block scan) -> row lists in z order.
//   K2b k_bin_fill     one block per tile: stable compaction of its row list by
//                      column range -> the tile's z-ascending primitive list.
// Together K2a/K2b are a two-digit (tile row, tile column) stable MSD radix
// bucketing of the z-sorted stream: the output equals a stable radix sort of
// (tile, z) keys and is bit-identical to the reference's offsets/indices.
#include "../../include/primfit_b200.h"
#include "pf_common.cuh"

namespace pf {

struct BinScratch {
  int4* rect;        // [n] band-clipped tile rect per z position (tx0, ty0, tx1, ty1)
  int32_t* zprim;    // [n] primitive index per z position
  int32_t* tcount;   // [n_tiles] per-tile counts
  int32_t* rcount;   // [n_rows] per-row counts
  int32_t* rowlist;  // [capacity] z positions, grouped by row
  int32_t* rowoff;   // [n_rows + 1]
  size_t total;
};

static size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

static BinScratch carve(void* base, int n, int n_tiles, int n_rows, int cap) {
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
  s.tcount = (int32_t*)take(sizeof(int32_t) * (size_t)n_tiles);
  s.rcount = (int32_t*)take(sizeof(int32_t) * (size_t)n_rows);
  s.rowlist = (int32_t*)take(sizeof(int32_t) * (size_t)cap);
  s.rowoff = (int32_t*)take(sizeof(int32_t) * (size_t)(n_rows + 1));
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
  RecC* recc;
  BinScratch s;
};

// K1: one thread per z position j (primitive zorder[j]).
__global__ void __launch_bounds__(32) k_preprocess(PreArgs a) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
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
  rf.inv_s = __ddiv_rn(1.0, s);
  rf.inv_sq = __ddiv_rn(1.0, rf.sq);
  rf.wm1 = (double)(wt - 1);
  rf.hm1 = (double)(ht - 1);
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

  // cull record (see RecC): fp32 centre and axes, conservative slack
  {
    RecC rc;
    const double is = rf.inv_s, isq = rf.inv_sq;
    rc.px = (float)x;
    rc.py = (float)y;
    rc.au = (float)(ct * is);
    rc.bu = (float)(st * is);
    rc.av = (float)(ct * isq);
    rc.bv = (float)(st * isq);
    const double hx = 0.5 * (kWarpW - 1), hy = 0.5 * (kWarpH - 1);
    const double e_px = fabs(x - (double)rc.px) + fabs(y - (double)rc.py);
    const double span = e_px + 1e-6 * (fabs(r) + 2.0 * kTile);
    const double su = (fabs(ct) + fabs(st)) * is, sv = (fabs(ct) + fabs(st)) * isq;
    rc.eu = (float)((fabs(ct) * hx + fabs(st) * hy) * is + su * span + 1e-5);
    rc.ev = (float)((fabs(st) * hx + fabs(ct) * hy) * isq + sv * span + 1e-5);
    a.recc[i] = rc;
  }
  double lo_x = ceil(__dsub_rn(x, r)), hi_x = floor(__dadd_rn(x, r));
  double lo_y = ceil(__dsub_rn(y, r)), hi_y = floor(__dadd_rn(y, r));
  lo_x = fmax(lo_x, 0.0);
  lo_y = fmax(lo_y, 0.0);
  hi_x = fmin(hi_x, (double)(a.W - 1));
  hi_y = fmin(hi_y, (double)(a.H - 1));
  int4 rc = make_int4(1, 1, 0, 0);  // empty
  // NaN-safe: every comparison with NaN is false -> treated as empty
  if (lo_x <= hi_x && lo_y <= hi_y) {
    const int tx0 = (int)lo_x / a.tile, tx1 = (int)hi_x / a.tile;
    int ty0 = (int)lo_y / a.tile, ty1 = (int)hi_y / a.tile;
    ty0 = max(ty0, a.ty_begin);
    ty1 = min(ty1, a.ty_end - 1);
    if (ty0 <= ty1) {
      rc = make_int4(tx0, ty0, tx1, ty1);
      for (int ty = ty0; ty <= ty1; ++ty) {
        const int row = ty - a.ty_begin;
        atomicAdd(a.s.rcount + row, 1);
        for (int tx = tx0; tx <= tx1; ++tx) atomicAdd(a.s.tcount + row * a.ntx + tx, 1);
      }
    }
  }
  a.s.rect[j] = rc;
}

__device__ __forceinline__ int div_up_d(int a, int b) { return (a + b - 1) / b; }

// Block-wide exclusive scan of one int per thread (1024 threads max).
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

struct ScanArgs {
  int n, n_tiles, n_rows, ntx, ty_begin, cap;
  BinScratch s;
  int32_t* bin_off;
  int32_t* status;
};

constexpr int kScanThreads = 1024;

// K2a: block 0 scans the tile counts; block 1 + r builds row r's list.  Each
// thread owns a contiguous chunk, so one block scan per block keeps z order.
__global__ void __launch_bounds__(kScanThreads) k_bin_scan(ScanArgs a) {
  __shared__ int warp_sums[32];
  if (blockIdx.x == 0) {
    const int chunk = div_up_d(a.n_tiles, kScanThreads);
    const int t0 = min(a.n_tiles, threadIdx.x * chunk), t1 = min(a.n_tiles, t0 + chunk);
    int local = 0;
    for (int t = t0; t < t1; ++t) local += a.s.tcount[t];
    int tot;
    int run = block_excl_scan(local, warp_sums, &tot);
    for (int t = t0; t < t1; ++t) {
      a.bin_off[t] = run;
      run += a.s.tcount[t];
    }
    if (threadIdx.x == 0) {
      a.bin_off[a.n_tiles] = tot;
      a.status[0] = tot;
      a.status[1] = tot > a.cap ? 1 : 0;
    }
    return;
  }
  const int r = blockIdx.x - 1;
  const int ty = a.ty_begin + r;
  // row offset = sum of the counts of the rows before r (rows are few)
  int part = 0;
  for (int q = threadIdx.x; q < r; q += kScanThreads) part += a.s.rcount[q];
  int row_base;
  (void)block_excl_scan(part, warp_sums, &row_base);
  const int chunk = div_up_d(a.n, kScanThreads);
  const int j0 = min(a.n, threadIdx.x * chunk), j1 = min(a.n, j0 + chunk);
  int local = 0;
  for (int j = j0; j < j1; ++j) {
    const int4 rc = a.s.rect[j];
    local += (rc.y <= ty && ty <= rc.w) ? 1 : 0;
  }
  int tot;
  int pos = row_base + block_excl_scan(local, warp_sums, &tot);
  for (int j = j0; j < j1; ++j) {
    const int4 rc = a.s.rect[j];
    if (rc.y <= ty && ty <= rc.w) {
      if (pos < a.cap) a.s.rowlist[pos] = j;
      ++pos;
    }
  }
  if (threadIdx.x == 0) {
    a.s.rowoff[r] = row_base;
    if (r == a.n_rows - 1) a.s.rowoff[a.n_rows] = row_base + tot;
  }
}

struct FillArgs {
  int n_tiles, ntx, cap;
  BinScratch s;
  const int32_t* bin_off;
  int32_t* bin_idx;
  const int32_t* status;
};

constexpr int kFillThreads = 128;

// K2b: one block per tile, stable compaction of its row list by column range.
__global__ void __launch_bounds__(kFillThreads) k_bin_fill(FillArgs a) {
  __shared__ int warp_sums[32];
  if (a.status[1]) return;  // overflow: lists would not fit
  const int t = blockIdx.x;
  const int r = t / a.ntx, tx = t - r * a.ntx;
  const int r0 = a.s.rowoff[r], n = a.s.rowoff[r + 1] - r0;
  const int chunk = div_up_d(n, kFillThreads);
  const int k0 = min(n, (int)threadIdx.x * chunk), k1 = min(n, k0 + chunk);
  int local = 0;
  for (int k = k0; k < k1; ++k) {
    const int4 rc = a.s.rect[a.s.rowlist[r0 + k]];
    local += (rc.x <= tx && tx <= rc.z) ? 1 : 0;
  }
  int tot;
  int out = a.bin_off[t] + block_excl_scan(local, warp_sums, &tot);
  for (int k = k0; k < k1; ++k) {
    const int j = a.s.rowlist[r0 + k];
    const int4 rc = a.s.rect[j];
    if (rc.x <= tx && tx <= rc.z) a.bin_idx[out++] = a.s.zprim[j];
  }
}

// Alpha quad atlas (see Quad in pf_common.cuh): one thread per texel.
struct QuadArgs {
  const double* tex;  // planar [4][texels]
  int texels, n_tpl;
  const int32_t* base;
  const int32_t* w;
  const int32_t* h;
  float* quad;
};

__global__ void k_atlas_quad(QuadArgs a) {
  const int g = blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= a.texels) return;
  int t = 0;
  while (t + 1 < a.n_tpl && a.base[t + 1] <= g) ++t;
  const int wt = a.w[t], ht = a.h[t], local = g - a.base[t];
  const int v = local / wt, u = local - v * wt;
  const double* al = a.tex + 3 * (size_t)a.texels + a.base[t];
  auto at = [&](int uu, int vv) { return (uu < wt && vv < ht) ? al[vv * wt + uu] : 0.0; };
  reinterpret_cast<float4*>(a.quad)[g] =
      make_float4((float)at(u, v), (float)at(u + 1, v), (float)at(u, v + 1), (float)at(u + 1, v + 1));
}

}  // namespace pf

using namespace pf;

extern "C" size_t pf_bin_scratch_bytes(int n, int n_tiles, int capacity) {
  if (n < 0 || n_tiles < 0 || capacity < 0) return 0;
  // rows <= tiles; size for the worst case (one tile per row)
  return carve(nullptr, n, n_tiles, n_tiles, capacity).total;
}

static bool band_ok(int W, int H, int tile, int ty_begin, int ty_end, int* ntx, int* n_rows) {
  if (W < 1 || H < 1 || tile < 1) return false;
  *ntx = div_up(W, tile);
  const int nty = div_up(H, tile);
  if (ty_begin < 0 || ty_end > nty || ty_begin > ty_end) return false;
  *n_rows = ty_end - ty_begin;
  return true;
}

extern "C" int pf_preprocess(const double* params, const int32_t* template_id,
                             const int32_t* zorder, int n, const int32_t* tpl_base,
                             const int32_t* tpl_w, const int32_t* tpl_h, const double* tpl_q,
                             const double* tpl_hyp, int n_tpl, double alpha_max, double mu_blend,
                             double padding, int W, int H, int tile, int ty_begin, int ty_end,
                             int capacity, void* rec, void* scratch, size_t scratch_bytes,
                             void* stream) {
  int ntx, n_rows;
  if (n < 0 || n_tpl < 0 || capacity < 0 || !band_ok(W, H, tile, ty_begin, ty_end, &ntx, &n_rows))
    return PF_ERR_ARG;
  const int n_tiles = n_rows * ntx;
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
  a.recc = (RecC*)((char*)rec + (sizeof(RecF) + sizeof(RecB)) * (size_t)n);
  a.s = carve(scratch, n, n_tiles, n_tiles, capacity);
  cudaError_t e = cudaMemsetAsync(a.s.tcount, 0, sizeof(int32_t) * (size_t)n_tiles, st);
  if (e == cudaSuccess) e = cudaMemsetAsync(a.s.rcount, 0, sizeof(int32_t) * (size_t)n_rows, st);
  if (e != cudaSuccess) return (int)e;
  // small blocks spread the (latency-bound, sincos/exp heavy) threads over many SMs
  if (n > 0) k_preprocess<<<div_up(n, 32), 32, 0, st>>>(a);
  return (int)cudaGetLastError();
}

extern "C" int pf_bin(int n, int W, int H, int tile, int ty_begin, int ty_end, int capacity,
                      void* scratch, size_t scratch_bytes, int32_t* bin_off, int32_t* bin_idx,
                      int32_t* status, void* stream) {
  int ntx, n_rows;
  if (n < 0 || capacity < 0 || !band_ok(W, H, tile, ty_begin, ty_end, &ntx, &n_rows))
    return PF_ERR_ARG;
  if (!bin_off || !status || (capacity > 0 && !bin_idx)) return PF_ERR_ARG;
  const int n_tiles = n_rows * ntx;
  if (!scratch || scratch_bytes < pf_bin_scratch_bytes(n, n_tiles, capacity)) return PF_ERR_SCRATCH;
  cudaStream_t st = (cudaStream_t)stream;
  BinScratch s = carve(scratch, n, n_tiles, n_tiles, capacity);
  ScanArgs sa;
  sa.n = n;
  sa.n_tiles = n_tiles;
  sa.n_rows = n_rows;
  sa.ntx = ntx;
  sa.ty_begin = ty_begin;
  sa.cap = capacity;
  sa.s = s;
  sa.bin_off = bin_off;
  sa.status = status;
  k_bin_scan<<<1 + n_rows, kScanThreads, 0, st>>>(sa);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return (int)e;
  if (n_tiles == 0) return PF_OK;
  FillArgs f;
  f.n_tiles = n_tiles;
  f.ntx = ntx;
  f.cap = capacity;
  f.s = s;
  f.bin_off = bin_off;
  f.bin_idx = bin_idx;
  f.status = status;
  k_bin_fill<<<n_tiles, kFillThreads, 0, st>>>(f);
  return (int)cudaGetLastError();
}

extern "C" int pf_atlas_quad(const double* tex, int texels, const int32_t* tpl_base,
                             const int32_t* tpl_w, const int32_t* tpl_h, int n_tpl, float* quad,
                             void* stream) {
  if (texels < 0 || n_tpl < 0 || (texels > 0 && (!tex || !tpl_base || !tpl_w || !tpl_h || !quad)))
    return PF_ERR_ARG;
  if (texels == 0) return PF_OK;
  QuadArgs a{tex, texels, n_tpl, tpl_base, tpl_w, tpl_h, quad};
  k_atlas_quad<<<div_up(texels, 256), 256, 0, (cudaStream_t)stream>>>(a);
  return (int)cudaGetLastError();
}
