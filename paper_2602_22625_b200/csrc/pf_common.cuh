// Shared device-side definitions for the primfit B200 kernels.
//
// Precision policy:
//   * the coordinate chain dx,dy -> u,v -> U,V, the inside-box test, the
//     bilinear mask sample and the eps_skip test are float64 with the
//     reference's exact operation order and no FMA contraction
//     (__dmul_rn/__dadd_rn/__ddiv_rn), so every branch decision matches the
//     reference's float64 numba code (_kernels.py:106-119);
//   * compositing state (T, C) and the per-pixel gradient math are float64;
//   * pixel-sized buffers (image, alpha, target, dL/dI) are float32.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace pf {

constexpr int kTile = 16;                 // render tile edge (16x16 pixels / block)
constexpr int kTilePix = kTile * kTile;   // 256 threads per render block
constexpr unsigned kFull = 0xffffffffu;

// Forward record: everything the per-pair forward math reads.  96 bytes,
// staged into shared memory with cp.async (6 x 16 B per record).
struct __align__(16) RecF {
  double px, py;   // centre (canvas px; pixel centres at integer coords)
  double ct, st;   // cos / sin of rotation
  double s, sq;    // scale, scale * aspect   (v divisor, _kernels.py:112)
  double sa;       // alpha_max * sigmoid(opacity_logit)
  double c0, c1, c2;  // (1 - mu_blend) * sigmoid(color_logit)
  int32_t base, wt, ht, tid;  // template atlas slot
};
static_assert(sizeof(RecF) == 96, "RecF must be 96 bytes");

// Backward-only record extras (precomputed per primitive, 96 bytes).
struct __align__(16) RecB {
  double sd;              // alpha_max * sig * (1 - sig)
  double cd0, cd1, cd2;   // sigmoid'(color logit) = sc * (1 - sc)
  double gxu, gxv;        // -ct/s, st/(s q)
  double gyu, gyv;        // -st/s, -ct/(s q)
  double inv_s, q, inv_q, one_minus_mu;
};
static_assert(sizeof(RecB) == 96, "RecB must be 96 bytes");

// Stable two-branch logistic, _kernels.py:27-32.
__device__ __forceinline__ double sigmoid(double x) {
  if (x >= 0.0) return 1.0 / (1.0 + exp(-x));
  double e = exp(x);
  return e / (1.0 + e);
}

// Canvas pixel -> texel coordinates, reference op order (_kernels.py:109-115),
// no contraction.  Returns the inside-box predicate (inclusive at W-1).
__device__ __forceinline__ bool texel_coords(const RecF& r, double xx, double yy,
                                             double& U, double& V) {
  const double dx = __dsub_rn(xx, r.px);
  const double dy = __dsub_rn(yy, r.py);
  const double u = __ddiv_rn(__dadd_rn(__dmul_rn(r.ct, dx), __dmul_rn(r.st, dy)), r.s);
  const double v = __ddiv_rn(__dadd_rn(__dmul_rn(-r.st, dx), __dmul_rn(r.ct, dy)), r.sq);
  const double wm1 = (double)(r.wt - 1);
  const double hm1 = (double)(r.ht - 1);
  U = __dmul_rn(__dmul_rn(__dadd_rn(u, 1.0), 0.5), wm1);
  V = __dmul_rn(__dmul_rn(__dadd_rn(v, 1.0), 0.5), hm1);
  return !(U < 0.0 || U > wm1 || V < 0.0 || V > hm1);
}

// Zero-padded texel fetch (_kernels.py:35-40).
__device__ __forceinline__ double texel(const double* __restrict__ plane, int base, int wt,
                                        int ht, int u, int v) {
  if (u < 0 || u > wt - 1 || v < 0 || v > ht - 1) return 0.0;
  return __ldg(plane + base + v * wt + u);
}

struct Cell {
  int u0, v0;
  double wu, wv;
};

__device__ __forceinline__ Cell make_cell(double U, double V) {
  Cell c;
  const double fu = floor(U), fv = floor(V);
  c.u0 = (int)fu;
  c.v0 = (int)fv;
  c.wu = __dsub_rn(U, fu);
  c.wv = __dsub_rn(V, fv);
  return c;
}

// Bilinear sample, _kernels.py:43-58, same association, no contraction.
__device__ __forceinline__ double bilinear(const double* __restrict__ plane, int base, int wt,
                                           int ht, const Cell& c) {
  const double p00 = texel(plane, base, wt, ht, c.u0, c.v0);
  const double p01 = texel(plane, base, wt, ht, c.u0 + 1, c.v0);
  const double p10 = texel(plane, base, wt, ht, c.u0, c.v0 + 1);
  const double p11 = texel(plane, base, wt, ht, c.u0 + 1, c.v0 + 1);
  const double iu = __dsub_rn(1.0, c.wu), iv = __dsub_rn(1.0, c.wv);
  double acc = __dmul_rn(__dmul_rn(iu, iv), p00);
  acc = __dadd_rn(acc, __dmul_rn(__dmul_rn(c.wu, iv), p01));
  acc = __dadd_rn(acc, __dmul_rn(__dmul_rn(iu, c.wv), p10));
  acc = __dadd_rn(acc, __dmul_rn(__dmul_rn(c.wu, c.wv), p11));
  return acc;
}

// Bilinear value and (U, V) derivative in one fetch (_kernels.py:61-73).
__device__ __forceinline__ double bilinear_grad(const double* __restrict__ plane, int base, int wt,
                                                int ht, const Cell& c, double& gu, double& gv) {
  const double p00 = texel(plane, base, wt, ht, c.u0, c.v0);
  const double p01 = texel(plane, base, wt, ht, c.u0 + 1, c.v0);
  const double p10 = texel(plane, base, wt, ht, c.u0, c.v0 + 1);
  const double p11 = texel(plane, base, wt, ht, c.u0 + 1, c.v0 + 1);
  const double iu = __dsub_rn(1.0, c.wu), iv = __dsub_rn(1.0, c.wv);
  gu = iv * (p01 - p00) + c.wv * (p11 - p10);
  gv = iu * (p10 - p00) + c.wu * (p11 - p01);
  double acc = __dmul_rn(__dmul_rn(iu, iv), p00);
  acc = __dadd_rn(acc, __dmul_rn(__dmul_rn(c.wu, iv), p01));
  acc = __dadd_rn(acc, __dmul_rn(__dmul_rn(iu, c.wv), p10));
  acc = __dadd_rn(acc, __dmul_rn(__dmul_rn(c.wu, c.wv), p11));
  return acc;
}

__device__ __forceinline__ void cp_async16(void* smem_dst, const void* gmem_src) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem_dst);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem_src));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

inline int div_up(int a, int b) { return (a + b - 1) / b; }

}  // namespace pf
