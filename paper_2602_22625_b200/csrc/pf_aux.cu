// the video-fit heuristics and the layered export,
// restated as sm_100a kernels behind the same C ABI.
//
// f4 layered export (reference exportio.py:272-346, "3D-grid
// export kernel"): every primitive rendered ALONE over its own conservative
// pixel box of the rho-times denser canvas, premultiplied RGBA -- primitive
// parallel, no compositing, no atomics.
//   k_layer_bbox     one thread per primitive: scale_scene (x' = rho x + (rho-1)/2,
//                    s' = rho s) + layer_bbox (floor / ceil outward, pad 1 px)
//   k_layer_offsets  one block: exclusive scan of the box areas (int64)
//   k_render_layers  one block per primitive, threads over its box: the
//                    reference's canvas_to_prim / prim_to_texel / _bilinear_plane
//                    chain in float64 without contraction (raster.py:159-200),
//                    a = alpha_max * expit(nu) * m, colour blend (raster.py:214-219)
// f3 video heuristics (reference dyn.py:86-177):
//   k_diff_mask      one thread per pixel: max_c |prev - cur| > tau
//   k_freeze         one warp per primitive: any changed pixel inside the
//                    binning box (ballot early exit)
//   k_remove_stuck   one block per grid region: stable compaction of the
//                    region's members (index order), depth rank by counting,
//                    eligibility, top-k by (scale * alpha desc, index asc),
//                    opacity logit *= eta.
#include "../../include/primfit_b200.h"
#include "pf_bins.cuh"
#include "pf_common.cuh"

namespace pf {

namespace {

constexpr double kLayerPad = 1.0;  // exportio.py:78 LAYER_BBOX_PAD

__device__ __forceinline__ double expit(double x) { return sigmoid(x); }

// scale_scene (exportio.py:272-288), Python's operation order
__device__ __forceinline__ void scaled_prim(const double* p, int rho, double& x, double& y,
                                            double& s) {
  const double shift = (double)(rho - 1) / 2.0;
  x = __dadd_rn(__dmul_rn((double)rho, p[0]), shift);
  y = __dadd_rn(__dmul_rn((double)rho, p[1]), shift);
  s = __dmul_rn((double)rho, p[2]);
}

__global__ void k_layer_bbox(const double* __restrict__ params, const int32_t* __restrict__ tid,
                             const double* __restrict__ tpl_hyp, int n, int W, int H, int rho,
                             int4* __restrict__ bbox, long long* __restrict__ area) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double x, y, s;
  scaled_prim(params + (size_t)i * 8, rho, x, y, s);
  const double r = __dadd_rn(__dmul_rn(s, tpl_hyp[tid[i]]), kLayerPad);
  const double x0 = fmax(floor(__dsub_rn(x, r)), 0.0);
  const double x1 = fmin(ceil(__dadd_rn(x, r)), (double)(rho * W - 1));
  const double y0 = fmax(floor(__dsub_rn(y, r)), 0.0);
  const double y1 = fmin(ceil(__dadd_rn(y, r)), (double)(rho * H - 1));
  if (x0 <= x1 && y0 <= y1) {
    bbox[i] = make_int4((int)x0, (int)y0, (int)x1, (int)y1);
    area[i] = (long long)(x1 - x0 + 1.0) * (long long)(y1 - y0 + 1.0);
  } else {  // DegenerateBBox: fully off-canvas
    bbox[i] = make_int4(-1, -1, -1, -1);
    area[i] = 0;
  }
}

// offsets[i] = sum of area[0..i) (offsets[n] = total); one block
__global__ void __launch_bounds__(1024) k_layer_offsets(const long long* __restrict__ area, int n,
                                                        long long* __restrict__ offsets) {
  __shared__ long long warp_sums[32];
  __shared__ long long carry;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int base = 0; base < n; base += 1024) {
    const int i = base + threadIdx.x;
    const long long v = i < n ? area[i] : 0;
    long long x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const long long y = __shfl_up_sync(kFull, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) warp_sums[warp] = x;
    __syncthreads();
    if (warp == 0) {
      long long w = warp_sums[lane];
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const long long y = __shfl_up_sync(kFull, w, o);
        if (lane >= o) w += y;
      }
      warp_sums[lane] = w;
    }
    __syncthreads();
    const long long ex = carry + (warp > 0 ? warp_sums[warp - 1] : 0) + x - v;
    if (i < n) offsets[i] = ex;
    __syncthreads();
    if (threadIdx.x == 0) carry += warp_sums[31];
    __syncthreads();
  }
  if (threadIdx.x == 0) offsets[n] = carry;
}

struct LayerArgs {
  const double* params;
  const int32_t* tid;
  const double* tex;  // planar [4][texels]
  int texels;
  const int32_t* tpl_base;
  const int32_t* tpl_w;
  const int32_t* tpl_h;
  const double* tpl_q;
  double alpha_max, mu_blend;
  int rho;
  const int4* bbox;
  const long long* offsets;
  float4* rgba;
};

// _bilinear_plane (raster.py:182-200): zero outside the box, edge-clamped taps
__device__ __forceinline__ double plane_sample(const double* __restrict__ pl, int wt, int ht,
                                               double U, double V) {
  if (!(U >= 0.0 && U <= wt - 1.0 && V >= 0.0 && V <= ht - 1.0)) return 0.0;
  const int u0 = min(max((int)floor(U), 0), wt - 1), v0 = min(max((int)floor(V), 0), ht - 1);
  const int u1 = min(u0 + 1, wt - 1), v1 = min(v0 + 1, ht - 1);
  const double wu = fmin(fmax(__dsub_rn(U, (double)u0), 0.0), 1.0);
  const double wv = fmin(fmax(__dsub_rn(V, (double)v0), 0.0), 1.0);
  const double iu = __dsub_rn(1.0, wu), iv = __dsub_rn(1.0, wv);
  double acc = __dmul_rn(__dmul_rn(iu, iv), __ldg(pl + v0 * wt + u0));
  acc = __dadd_rn(acc, __dmul_rn(__dmul_rn(wu, iv), __ldg(pl + v0 * wt + u1)));
  acc = __dadd_rn(acc, __dmul_rn(__dmul_rn(iu, wv), __ldg(pl + v1 * wt + u0)));
  acc = __dadd_rn(acc, __dmul_rn(__dmul_rn(wu, wv), __ldg(pl + v1 * wt + u1)));
  return acc;
}

__global__ void __launch_bounds__(256) k_render_layers(LayerArgs a) {
  const int i = blockIdx.x;
  const int4 b = a.bbox[i];
  if (b.x < 0) return;
  const double* p = a.params + (size_t)i * 8;
  double x, y, s;
  scaled_prim(p, a.rho, x, y, s);
  const int t = a.tid[i];
  const int wt = a.tpl_w[t], ht = a.tpl_h[t];
  const double q = a.tpl_q[t];
  double st, ct;
  sincos(p[3], &st, &ct);
  const double sq = __dmul_rn(s, q);
  const double sa = __dmul_rn(a.alpha_max, expit(p[4]));
  const double cv0 = expit(p[5]), cv1 = expit(p[6]), cv2 = expit(p[7]);
  const double* pa = a.tex + 3 * (size_t)a.texels + a.tpl_base[t];
  const int bw = b.z - b.x + 1, bh = b.w - b.y + 1;
  float4* out = a.rgba + a.offsets[i];
  for (int k = threadIdx.x; k < bw * bh; k += blockDim.x) {
    const int ly = k / bw, lx = k - ly * bw;
    const double dx = __dsub_rn((double)(b.x + lx), x), dy = __dsub_rn((double)(b.y + ly), y);
    // canvas_to_prim / prim_to_texel (raster.py:159-179)
    const double u = __ddiv_rn(__dadd_rn(__dmul_rn(ct, dx), __dmul_rn(st, dy)), s);
    const double v = __ddiv_rn(__dadd_rn(__dmul_rn(-st, dx), __dmul_rn(ct, dy)), sq);
    const double U = __dmul_rn(__dmul_rn(__dadd_rn(u, 1.0), 0.5), (double)(wt - 1));
    const double V = __dmul_rn(__dmul_rn(__dadd_rn(v, 1.0), 0.5), (double)(ht - 1));
    const double m = plane_sample(pa, wt, ht, U, V);
    const double al = __dmul_rn(sa, m);
    double c0 = cv0, c1 = cv1, c2 = cv2;
    if (a.mu_blend > 0.0) {  // blend_color: mu * c_org + (1 - mu) * c_var
      const double om = __dsub_rn(1.0, a.mu_blend);
      const double* pr = a.tex + a.tpl_base[t];
      c0 = __dadd_rn(__dmul_rn(a.mu_blend, plane_sample(pr, wt, ht, U, V)), __dmul_rn(om, cv0));
      c1 = __dadd_rn(__dmul_rn(a.mu_blend, plane_sample(pr + a.texels, wt, ht, U, V)),
                     __dmul_rn(om, cv1));
      c2 = __dadd_rn(__dmul_rn(a.mu_blend, plane_sample(pr + 2 * (size_t)a.texels, wt, ht, U, V)),
                     __dmul_rn(om, cv2));
    }
    out[k] = make_float4((float)(al * c0), (float)(al * c1), (float)(al * c2), (float)al);
  }
}

__global__ void k_diff_mask(const double* __restrict__ prev, const double* __restrict__ cur, int P,
                            double tau, uint8_t* __restrict__ mask) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= P) return;
  double d = 0.0;
#pragma unroll
  for (int c = 0; c < 3; ++c) d = fmax(d, fabs(prev[3 * (size_t)k + c] - cur[3 * (size_t)k + c]));
  mask[k] = d > tau ? 1 : 0;
}

// freeze_flags (dyn.py:100-130): one warp per primitive
__global__ void k_freeze(const double* __restrict__ params, const int32_t* __restrict__ tid,
                         const double* __restrict__ tpl_hyp, int n, int W, int H, double padding,
                         const uint8_t* __restrict__ mask, uint8_t* __restrict__ frozen) {
  const int i = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (i >= n) return;
  const double* p = params + (size_t)i * 8;
  const double r = __dadd_rn(__dmul_rn(p[2], tpl_hyp[tid[i]]), padding);
  const double x0 = fmax(ceil(__dsub_rn(p[0], r)), 0.0);
  const double x1 = fmin(floor(__dadd_rn(p[0], r)), (double)(W - 1));
  const double y0 = fmax(ceil(__dsub_rn(p[1], r)), 0.0);
  const double y1 = fmin(floor(__dadd_rn(p[1], r)), (double)(H - 1));
  bool hit = false;
  if (x0 <= x1 && y0 <= y1) {
    const int bx = (int)x0, by = (int)y0, bw = (int)x1 - bx + 1, bh = (int)y1 - by + 1;
    for (int k0 = 0; k0 < bw * bh && !hit; k0 += 32) {
      const int k = k0 + lane;
      bool h = false;
      if (k < bw * bh) {
        const int ly = k / bw;
        h = mask[(size_t)(by + ly) * W + bx + (k - ly * bw)] != 0;
      }
      hit = __any_sync(kFull, h);
    }
  }
  if (lane == 0) frozen[i] = hit ? 0 : 1;
}

struct StuckArgs {
  double* params;
  const int32_t* z;
  const uint8_t* frozen;
  int n, W, H, rows, cols, k;
  double tau_scale, tau_alpha, zeta, eta, alpha_max;
  uint8_t* decayed;
  int32_t* members;  // [2][regions][n] scratch: member lists, eligibility flags
};

constexpr int kStuckThreads = 1024;

// remove_stuck (dyn.py:133-177): one block per region
__global__ void __launch_bounds__(kStuckThreads) k_remove_stuck(StuckArgs a) {
  __shared__ int ws[32];
  __shared__ int s_best_i;
  const int reg = blockIdx.x;
  const int tid = threadIdx.x;
  int32_t* mem = a.members + (size_t)reg * a.n;
  int32_t* flag = a.members + (size_t)(gridDim.x + reg) * a.n;
  auto region_of = [&](int i) {
    const double* p = a.params + (size_t)i * 8;
    const int ry = min(max((int)(p[1] * a.rows / a.H), 0), a.rows - 1);
    const int rx = min(max((int)(p[0] * a.cols / a.W), 0), a.cols - 1);
    return ry * a.cols + rx;
  };
  // (1) members in index order: contiguous chunks + block scan
  const int chunk = (a.n + kStuckThreads - 1) / kStuckThreads;
  const int j0 = min(a.n, tid * chunk), j1 = min(a.n, j0 + chunk);
  int cnt = 0;
  for (int j = j0; j < j1; ++j) cnt += region_of(j) == reg;
  int m;
  int pos = block_excl_scan(cnt, ws, &m);
  for (int j = j0; j < j1; ++j)
    if (region_of(j) == reg) mem[pos++] = j;
  __syncthreads();
  // (2) eligibility and score per member; rank = members strictly behind (larger z)
  for (int e = tid; e < m; e += kStuckThreads) {
    const int i = mem[e];
    const double* p = a.params + (size_t)i * 8;
    int rank = 0;
    const int zi = a.z[i];
    for (int f = 0; f < m; ++f) rank += a.z[mem[f]] > zi;
    const double alpha = a.alpha_max * sigmoid(p[4]);
    const bool ok = !(a.frozen && a.frozen[i]) && p[2] >= a.tau_scale * a.W &&
                    alpha >= a.tau_alpha && (double)rank >= a.zeta * m;
    flag[e] = ok ? 1 : 0;
  }
  __syncthreads();
  // negative member slot = not eligible (or, below, already picked)
  for (int e = tid; e < m; e += kStuckThreads)
    if (!flag[e]) mem[e] = -1 - mem[e];
  __syncthreads();
  // (3) top-k by (scale * alpha desc, index asc), one block argmax per pick
  for (int pick = 0; pick < a.k; ++pick) {
    double best = -1.0;
    int best_i = 0x7fffffff, best_e = -1;
    for (int e = tid; e < m; e += kStuckThreads) {
      const int i = mem[e];
      if (i < 0) continue;
      const double* p = a.params + (size_t)i * 8;
      const double sc = p[2] * (a.alpha_max * sigmoid(p[4]));
      if (sc > best || (sc == best && i < best_i)) {
        best = sc;
        best_i = i;
        best_e = e;
      }
    }
    // block reduction: warp argmax, then warp 0 over the warps
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double ob = __shfl_xor_sync(kFull, best, o);
      const int oi = __shfl_xor_sync(kFull, best_i, o);
      const int oe = __shfl_xor_sync(kFull, best_e, o);
      if (ob > best || (ob == best && oi < best_i)) {
        best = ob;
        best_i = oi;
        best_e = oe;
      }
    }
    __shared__ double wb[32];
    __shared__ int wi[32], we[32];
    if ((tid & 31) == 0) {
      wb[tid >> 5] = best;
      wi[tid >> 5] = best_i;
      we[tid >> 5] = best_e;
    }
    __syncthreads();
    if (tid == 0) {
      double b = -1.0;
      int bi = 0x7fffffff, be = -1;
      for (int w = 0; w < kStuckThreads / 32; ++w)
        if (wb[w] > b || (wb[w] == b && wi[w] < bi)) {
          b = wb[w];
          bi = wi[w];
          be = we[w];
        }
      s_best_i = be;
      if (be >= 0) {
        const int i = mem[be];
        a.decayed[i] = 1;
        a.params[(size_t)i * 8 + 4] = a.eta * a.params[(size_t)i * 8 + 4];
        mem[be] = -1 - i;  // taken
      }
    }
    __syncthreads();
    if (s_best_i < 0) break;
  }
}

}  // namespace

}  // namespace pf

using namespace pf;

// Upstream image gradients of the autograd backward into the fit step's
// per-pixel float4 rows: (dL/dI r, g, b, dL/dA), dL/dA = 0 when `alpha` is NULL.
__global__ void k_pack4(const float* __restrict__ rgb, const float* __restrict__ alpha, int P,
                        float4* __restrict__ out) {
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= P) return;
  out[p] = make_float4(rgb[3 * (size_t)p], rgb[3 * (size_t)p + 1], rgb[3 * (size_t)p + 2],
                       alpha ? alpha[p] : 0.0f);
}

extern "C" int pf_pack_grad4(const float* rgb, const float* alpha, int P, float* out4,
                             void* stream) {
  if (P < 0 || (P > 0 && (!rgb || !out4))) return PF_ERR_ARG;
  if (P == 0) return PF_OK;
  k_pack4<<<(P + 255) / 256, 256, 0, (cudaStream_t)stream>>>(rgb, alpha, P,
                                                              reinterpret_cast<float4*>(out4));
  return (int)cudaGetLastError();
}

// loss_mse (fit.py:110-115) on the autograd path: the image is the renderer's
// (r, g, b, alpha) rows, the target (P, 3).  Per-pixel squared error in fp32 (as
// the fit step's MSE), float64 per-block partials, folded in block order by the
// last block to finish (deterministic for a given grid); the counter self-resets.
constexpr int kMseThreads = 256;
constexpr int kMseBlocks = 148 * 8;  // <= PF_MSE4_SCRATCH - 1 partials

__global__ void __launch_bounds__(kMseThreads)
    k_mse4(const float4* __restrict__ img4, const float* __restrict__ tgt, int P,
           double* __restrict__ part, unsigned* __restrict__ ctr, double inv_n,
           float* __restrict__ loss) {
  double s = 0.0;
  for (int p = blockIdx.x * kMseThreads + threadIdx.x; p < P; p += gridDim.x * kMseThreads) {
    const float4 I = img4[p];
    const float r0 = I.x - tgt[3 * (size_t)p], r1 = I.y - tgt[3 * (size_t)p + 1],
                r2 = I.z - tgt[3 * (size_t)p + 2];
    s += (double)fmaf(r0, r0, fmaf(r1, r1, r2 * r2));
  }
  __shared__ double ws[kMseThreads / 32];
  __shared__ bool last;
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if ((threadIdx.x & 31) == 0) ws[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double b = 0.0;
    for (int w = 0; w < kMseThreads / 32; ++w) b += ws[w];
    part[blockIdx.x] = b;
    __threadfence();
    last = atomicAdd(ctr, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (!last || threadIdx.x >= 32) return;
  __threadfence();
  double t = 0.0;
  for (int b = threadIdx.x; b < (int)gridDim.x; b += 32) t += __ldcg(part + b);
  for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
  if (threadIdx.x == 0) {
    loss[0] = (float)(t * inv_n);
    *ctr = 0u;
  }
}

// dL/dI = grad_out * 2 (I - t) / (3 P) into the fit step's (r, g, b, 0) rows
__global__ void k_mse4_grad(const float4* __restrict__ img4, const float* __restrict__ tgt, int P,
                            const float* __restrict__ grad_out, float k,
                            float4* __restrict__ out) {
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= P) return;
  const float g = k * grad_out[0];
  const float4 I = img4[p];
  out[p] = make_float4(g * (I.x - tgt[3 * (size_t)p]), g * (I.y - tgt[3 * (size_t)p + 1]),
                       g * (I.z - tgt[3 * (size_t)p + 2]), 0.0f);
}

extern "C" int pf_mse4(const float* img4, const float* target, int P, double* scratch,
                       float* loss, void* stream) {
  if (P < 1 || !img4 || !target || !scratch || !loss) return PF_ERR_ARG;
  const int blocks = min(div_up(P, kMseThreads), kMseBlocks);
  k_mse4<<<blocks, kMseThreads, 0, (cudaStream_t)stream>>>(
      reinterpret_cast<const float4*>(img4), target, P, scratch + 1,
      reinterpret_cast<unsigned*>(scratch), 1.0 / (3.0 * (double)P), loss);
  return (int)cudaGetLastError();
}

extern "C" int pf_mse4_grad(const float* img4, const float* target, int P, const float* grad_out,
                            float* out4, void* stream) {
  if (P < 1 || !img4 || !target || !grad_out || !out4) return PF_ERR_ARG;
  k_mse4_grad<<<div_up(P, 256), 256, 0, (cudaStream_t)stream>>>(
      reinterpret_cast<const float4*>(img4), target, P, grad_out, (float)(2.0 / (3.0 * (double)P)),
      reinterpret_cast<float4*>(out4));
  return (int)cudaGetLastError();
}

extern "C" int pf_layer_bboxes(const double* params, const int32_t* template_id,
                               const double* tpl_hyp, int n, int W, int H, int rho, int32_t* bbox,
                               long long* area, long long* offsets, void* stream) {
  if (n < 0 || W < 1 || H < 1 || rho < 1 || (n > 0 && (!params || !template_id || !tpl_hyp ||
                                                        !bbox || !area || !offsets)))
    return PF_ERR_ARG;
  cudaStream_t st = (cudaStream_t)stream;
  if (n > 0)
    k_layer_bbox<<<div_up(n, 256), 256, 0, st>>>(params, template_id, tpl_hyp, n, W, H, rho,
                                                 reinterpret_cast<int4*>(bbox), area);
  k_layer_offsets<<<1, 1024, 0, st>>>(area, n, offsets);
  return (int)cudaGetLastError();
}

extern "C" int pf_render_layers(const double* params, const int32_t* template_id,
                                const double* tex, int texels, const int32_t* tpl_base,
                                const int32_t* tpl_w, const int32_t* tpl_h, const double* tpl_q,
                                int n, double alpha_max, double mu_blend, int rho,
                                const int32_t* bbox, const long long* offsets, float* rgba,
                                void* stream) {
  if (n < 0 || rho < 1 || (n > 0 && (!params || !template_id || !tex || !tpl_base || !tpl_w ||
                                      !tpl_h || !tpl_q || !bbox || !offsets || !rgba)))
    return PF_ERR_ARG;
  if (n == 0) return PF_OK;
  LayerArgs a{params, template_id, tex, texels, tpl_base, tpl_w, tpl_h, tpl_q, alpha_max,
              mu_blend, rho, reinterpret_cast<const int4*>(bbox), offsets,
              reinterpret_cast<float4*>(rgba)};
  k_render_layers<<<n, 256, 0, (cudaStream_t)stream>>>(a);
  return (int)cudaGetLastError();
}

extern "C" int pf_diff_mask(const double* prev, const double* cur, int W, int H, double tau,
                            uint8_t* mask, void* stream) {
  if (W < 1 || H < 1 || !prev || !cur || !mask) return PF_ERR_ARG;
  const int P = W * H;
  k_diff_mask<<<div_up(P, 256), 256, 0, (cudaStream_t)stream>>>(prev, cur, P, tau, mask);
  return (int)cudaGetLastError();
}

extern "C" int pf_freeze_flags(const double* params, const int32_t* template_id,
                               const double* tpl_hyp, int n, int W, int H, double padding,
                               const uint8_t* mask, uint8_t* frozen, void* stream) {
  if (n < 0 || W < 1 || H < 1 || (n > 0 && (!params || !template_id || !tpl_hyp || !mask ||
                                            !frozen)))
    return PF_ERR_ARG;
  if (n == 0) return PF_OK;
  k_freeze<<<div_up(n * 32, 256), 256, 0, (cudaStream_t)stream>>>(
      params, template_id, tpl_hyp, n, W, H, padding, mask, frozen);
  return (int)cudaGetLastError();
}

extern "C" size_t pf_stuck_scratch_bytes(int n, int regions) {
  return 2 * sizeof(int32_t) * (size_t)(n > 0 ? n : 1) * (size_t)(regions > 0 ? regions : 1);
}

extern "C" int pf_remove_stuck(double* params, const int32_t* z, const uint8_t* frozen, int n,
                               int W, int H, int grid_rows, int grid_cols, int k, double tau_scale,
                               double tau_alpha, double zeta, double eta, double alpha_max,
                               uint8_t* decayed, void* scratch, size_t scratch_bytes,
                               void* stream) {
  if (n < 0 || W < 1 || H < 1 || grid_rows < 1 || grid_cols < 1 || k < 0 ||
      (n > 0 && (!params || !z || !decayed)))
    return PF_ERR_ARG;
  if (!scratch || scratch_bytes < pf_stuck_scratch_bytes(n, grid_rows * grid_cols))
    return PF_ERR_SCRATCH;
  if (n == 0) return PF_OK;
  cudaStream_t st = (cudaStream_t)stream;
  cudaError_t e = cudaMemsetAsync(decayed, 0, (size_t)n, st);
  if (e != cudaSuccess) return (int)e;
  StuckArgs a{params, z, frozen, n, W, H, grid_rows, grid_cols, k, tau_scale, tau_alpha, zeta,
              eta, alpha_max, decayed, reinterpret_cast<int32_t*>(scratch)};
  k_remove_stuck<<<grid_rows * grid_cols, kStuckThreads, 0, st>>>(a);
  return (int)cudaGetLastError();
}
