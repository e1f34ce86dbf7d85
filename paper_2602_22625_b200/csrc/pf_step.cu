// K34: the fit step's render -> loss -> backward as ONE kernel.
//
// Reference: the loop body of run_loop (pkg/src/primfit/fit.py:486-492):
//   out, saved = render_forward(scene, bins, bg, save=True)   raster.py:290-363
//   value, dI, dA = evaluate_loss(loss_spec, out.color, out.alpha)  fit.py:112-151
//   grads = backward(scene, saved, dI, dA)                    grad.py:134-187
// Both losses the fit uses (MSE, spatial) are pixel-local: dL/dI and dL/dA of
// a pixel depend only on that pixel's colour and alpha.  So the thread that
// composites a pixel already holds everything its backward needs, and the
// saved contribution lists never have to leave the SM:
//
//   forward phase  - identical decisions and float64 compositing to
//                    k_forward (pf_render.cu); each contributing (pixel, entry)
//                    pushes a 32-byte record (list position, primitive, incoming
//                    T, mask m, dm/dU, dm/dV, u, v) into a per-thread shared-memory
//                    stack (kStepKS deep; deeper entries spill to HBM at a slot
//                    unique to (tile, depth, pixel) -- 0.5% of pixels at c3);
//   loss           - pixel-local loss, dL/dI, dL/dA in registers; per-warp fp32
//                    partials; the last block to finish (atomic ticket) folds all
//                    partials into sums[] in fixed order (deterministic);
//   backward phase - the same back-to-front warp walk as k_backward (list
//                    position picked with __reduce_max_sync) over the stack, with
//                    the tile's fp32 gradient records staged in shared memory by
//                    cp.async during the forward phase; warp transpose-butterfly
//                    reduction and float64 RED atomics into grads.
//
// Versus K3 + K4 this removes the saved-entry, ent_n and dL/dI round trips
// through L2/HBM, the backward kernel's whole dependent prologue and the
// backward's atlas re-fetch (m, dm/dU, dm/dV are stored, not re-sampled).
// mu_blend > 0 (colour from the texture) keeps the two-kernel path.
#include "../../include/primfit_b200.h"
#include "pf_common.cuh"

namespace pf {

namespace {

constexpr int kStepWarps = 2;                           // 64-thread blocks (a 16x4 strip)
constexpr int kStepBlocksPerTile = (kTilePix / 32) / kStepWarps;
constexpr int kStepKS = 2;                              // stack depth in shared memory

struct StepArgs {
  const RecF* recf;
  const RecG* recg;
  const RecC* recc;
  const double* tex;
  const float4* quad;
  int texels;
  const int32_t* bin_off;
  const int32_t* bin_idx;
  const int32_t* status;
  int W, H, ntx, ty_begin;
  double eps_skip;
  double bg0, bg1, bg2;
  const float4* bg4;
  float4* img4;          // optional (r, g, b, alpha)
  const float4* tgt4;
  double alpha_w, inv_3P, inv_P;
  double* part;
  float4* spill;         // [slot][2] for stack depth >= kStepKS
  double* grads;
};

__device__ __forceinline__ void step_pixel(int w, int tx, int ty, int& x, int& y, float& cx,
                                           float& cy) {
  const int l = threadIdx.x & 31;
  const int wx = (w & 1) * kWarpW, wy = (w >> 1) * kWarpH;
  x = tx * kTile + wx + (l & (kWarpW - 1));
  y = ty * kTile + wy + (l / kWarpW);
  cx = (float)(tx * kTile + wx) + 0.5f * (kWarpW - 1);
  cy = (float)(ty * kTile + wy) + 0.5f * (kWarpH - 1);
}

__device__ __forceinline__ bool step_may_touch(const RecC* __restrict__ rc, float cx, float cy) {
  const float4 a = __ldg(reinterpret_cast<const float4*>(rc));
  const float4 b = __ldg(reinterpret_cast<const float4*>(rc) + 1);
  const float dx = cx - a.x, dy = cy - a.y;
  const float uc = a.z * dx + a.w * dy;
  const float vc = b.x * dy - b.y * dx;
  const bool out_u = fabsf(uc) > 1.0f + b.z + 1e-5f * fabsf(uc);
  const bool out_v = fabsf(vc) > 1.0f + b.w + 1e-5f * fabsf(vc);
  return !(out_u || out_v);
}

// texel_coords (pf_common.cuh) that also hands back the normalised (u, v).
__device__ __forceinline__ bool texel_coords_uv(const RecF& r, double xx, double yy, double& U,
                                                double& V, double& u, double& v) {
  const double dx = __dsub_rn(xx, r.px);
  const double dy = __dsub_rn(yy, r.py);
  u = div_rn(__dadd_rn(__dmul_rn(r.ct, dx), __dmul_rn(r.st, dy)), r.s, r.inv_s);
  v = div_rn(__dadd_rn(__dmul_rn(-r.st, dx), __dmul_rn(r.ct, dy)), r.sq, r.inv_sq);
  U = __dmul_rn(__dmul_rn(__dadd_rn(u, 1.0), 0.5), r.wm1);
  V = __dmul_rn(__dmul_rn(__dadd_rn(v, 1.0), 0.5), r.hm1);
  return !(U < 0.0 || U > r.wm1 || V < 0.0 || V > r.hm1);
}

__device__ __forceinline__ float step_reduce8(const float (&g)[8]) {
  const int lane = threadIdx.x & 31;
  float w[4];
  const bool h16 = lane & 16;
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const float send = h16 ? g[q] : g[q + 4];
    const float keep = h16 ? g[q + 4] : g[q];
    w[q] = keep + __shfl_xor_sync(kFull, send, 16);
  }
  float x2[2];
  const bool h8 = lane & 8;
#pragma unroll
  for (int q = 0; q < 2; ++q) {
    const float send = h8 ? w[q] : w[q + 2];
    const float keep = h8 ? w[q + 2] : w[q];
    x2[q] = keep + __shfl_xor_sync(kFull, send, 8);
  }
  const bool h4 = lane & 4;
  float y = (h4 ? x2[1] : x2[0]) + __shfl_xor_sync(kFull, h4 ? x2[0] : x2[1], 4);
  y += __shfl_xor_sync(kFull, y, 2);
  y += __shfl_xor_sync(kFull, y, 1);
  return y;
}

}  // namespace

template <int LOSS>
__global__ void __launch_bounds__(kStepWarps * 32) k_step(StepArgs a) {
  __shared__ float4 stA[kStepKS][kStepWarps * 32];  // (j, i, T, m)
  __shared__ float4 stB[kStepKS][kStepWarps * 32];  // (dm/dU, dm/dV, u, v)

  const int st_ovf = a.status[1];
  const int tb = blockIdx.x / kStepBlocksPerTile;
  const int b0 = a.bin_off[tb];
  const int L = a.bin_off[tb + 1] - b0;
  if (st_ovf) return;  // bin overflow (grid-uniform): lists are not valid

  const int t = threadIdx.x;
  const int lane = t & 31;
  const int wt = (blockIdx.x % kStepBlocksPerTile) * kStepWarps + (t >> 5);
  const int tx = tb % a.ntx, ty = a.ty_begin + tb / a.ntx;
  int x, y;
  float cx, cy;
  step_pixel(wt, tx, ty, x, y, cx, cy);
  const bool valid = x < a.W && y < a.H;
  const double xx = (double)x, yy = (double)y;
  const size_t pix = valid ? (size_t)y * a.W + x : 0;
  const size_t slot0 = (size_t)b0 * kTilePix + wt * 32 + lane;

  float4 tg = make_float4(0.f, 0.f, 0.f, 0.f), bgp = tg;
  if (valid) tg = __ldg(a.tgt4 + pix);
  if (valid && a.bg4) bgp = __ldg(a.bg4 + pix);

  // ---- forward phase (k_forward semantics, _kernels.py:183-255)
  const double* plane_a = a.tex + 3 * (size_t)a.texels;
  double T = 1.0, C0 = 0.0, C1 = 0.0, C2 = 0.0;
  int ns = 0;
  for (int sub = 0; sub < L; sub += 32) {
    int my_i = 0;
    bool cand = false;
    if (sub + lane < L) {
      my_i = __ldg(a.bin_idx + b0 + sub + lane);
      cand = step_may_touch(a.recc + my_i, cx, cy);
    }
    unsigned mask = __ballot_sync(kFull, cand);
    while (mask) {
      const int bit = __ffs(mask) - 1;
      mask &= mask - 1;
      const int i = __shfl_sync(kFull, my_i, bit);
      if (!valid) continue;
      const RecF& r = a.recf[i];
      double U, V, u, v;
      if (!texel_coords_uv(r, xx, yy, U, V, u, v)) continue;
      const Cell c = make_cell(U, V);
      const float4 q = load_quad(a.quad, r.base, r.wt, c.u0, c.v0);
      double m = bilerp(q, c.wu, c.wv);
      if (fabs(m - a.eps_skip) <= 1e-6 * a.eps_skip) m = bilinear(plane_a, r.base, r.wt, r.ht, c);
      if (m < a.eps_skip) continue;
      const float wu = (float)c.wu, wv = (float)c.wv;
      const float gU = (1.0f - wv) * (q.y - q.x) + wv * (q.w - q.z);
      const float gV = (1.0f - wu) * (q.z - q.x) + wu * (q.w - q.y);
      const float4 ea = make_float4(__int_as_float(sub + bit), __int_as_float(i), (float)T, (float)m);
      const float4 eb = make_float4(gU, gV, (float)u, (float)v);
      if (ns < kStepKS) {
        stA[ns][t] = ea;
        stB[ns][t] = eb;
      } else {
        float4* sp = a.spill + 2 * (slot0 + (size_t)(ns - kStepKS) * kTilePix);
        sp[0] = ea;
        sp[1] = eb;
      }
      ++ns;
      const double aa = r.sa * m;
      const double Ta = T * aa;
      C0 += Ta * r.c0;
      C1 += Ta * r.c1;
      C2 += Ta * r.c2;
      T *= 1.0 - aa;
    }
  }

  // ---- loss (fit.py:112-151), pixel-local
  const float g0 = a.bg4 ? bgp.x : (float)a.bg0;
  const float g1 = a.bg4 ? bgp.y : (float)a.bg1;
  const float g2 = a.bg4 ? bgp.z : (float)a.bg2;
  float dI0 = 0.f, dI1 = 0.f, dI2 = 0.f, dA = 0.f;
  float l0 = 0.f, l1 = 0.f, l2 = 0.f;
  if (valid) {
    const double I0 = C0 + T * (a.bg4 ? (double)bgp.x : a.bg0);
    const double I1 = C1 + T * (a.bg4 ? (double)bgp.y : a.bg1);
    const double I2 = C2 + T * (a.bg4 ? (double)bgp.z : a.bg2);
    const double Ia = 1.0 - T;
    if (a.img4) a.img4[pix] = make_float4((float)I0, (float)I1, (float)I2, (float)Ia);
    const double r0 = I0 - (double)tg.x, r1 = I1 - (double)tg.y, r2 = I2 - (double)tg.z;
    const double sse = r0 * r0 + r1 * r1 + r2 * r2;
    const double k = 2.0 * a.inv_3P;
    l0 = (float)sse;
    if (LOSS == PF_LOSS_MSE) {
      l1 = l0;
      dI0 = (float)(k * r0);
      dI1 = (float)(k * r1);
      dI2 = (float)(k * r2);
    } else {
      const double ta = (double)tg.w;
      const double mk = ta > 0.0 ? 1.0 : 0.0;
      const double ad = Ia - ta;
      l1 = (float)(sse * mk);
      l2 = (float)(ad * ad);
      dI0 = (float)(k * r0 * mk);
      dI1 = (float)(k * r1 * mk);
      dI2 = (float)(k * r2 * mk);
      dA = (float)(a.alpha_w * 2.0 * ad * a.inv_P);
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    l0 += __shfl_xor_sync(kFull, l0, o);
    l1 += __shfl_xor_sync(kFull, l1, o);
    l2 += __shfl_xor_sync(kFull, l2, o);
  }
  if (lane == 0) {
    double* pp = a.part + ((size_t)tb * (kTilePix / 32) + wt) * 3;
    pp[0] = l0;
    pp[1] = l1;
    pp[2] = l2;
  }
  // ---- backward phase (_kernels.py:258-363), back to front over the stack
  float S0 = 0.f, S1 = 0.f, S2 = 0.f, B = 1.f;
  int k = ns - 1;
  float4 ea = make_float4(0.f, 0.f, 0.f, 0.f), eb = ea;
  unsigned key = 0;
  auto fetch = [&](int d) {
    if (d < kStepKS) {
      ea = stA[d][t];
      eb = stB[d][t];
    } else {
      const float4* sp = a.spill + 2 * (slot0 + (size_t)(d - kStepKS) * kTilePix);
      ea = sp[0];
      eb = sp[1];
    }
    key = (unsigned)__float_as_int(ea.x) + 1u;
  };
  if (k >= 0) fetch(k);
  while (true) {
    const unsigned jm = __reduce_max_sync(kFull, key);
    if (jm == 0u) break;
    const bool act = key == jm;
    const unsigned ball = __ballot_sync(kFull, act);
    const int i = __shfl_sync(kFull, __float_as_int(ea.y), __ffs(ball) - 1);
    float g[8];
#pragma unroll
    for (int c = 0; c < 8; ++c) g[c] = 0.0f;
    if (act) {
      const float Tc = ea.z, m = ea.w, gU = eb.x, gV = eb.y, u = eb.z, v = eb.w;
      if (--k >= 0) fetch(k); else key = 0;
      const RecG r = a.recg[i];
      const float aa = r.sa * m;
      const float gg = dI0 * (r.c0 - S0 - g0 * B) + dI1 * (r.c1 - S1 - g1 * B) +
                       dI2 * (r.c2 - S2 - g2 * B) + dA * B;
      const float dalpha = Tc * gg;
      g[4] = dalpha * r.sd * m;
      if (r.omm > 0.0f) {
        const float wc = Tc * aa * r.omm;
        g[5] = dI0 * wc * r.cd0;
        g[6] = dI1 * wc * r.cd1;
        g[7] = dI2 * wc * r.cd2;
      }
      const float dm = dalpha * r.sa;
      const float mu_u = gU * r.hw, mu_v = gV * r.hh;
      g[0] = dm * (mu_u * r.gxu + mu_v * r.gxv);
      g[1] = dm * (mu_u * r.gyu + mu_v * r.gyv);
      g[2] = dm * (mu_u * (-u * r.inv_s) + mu_v * (-v * r.inv_s));
      g[3] = dm * (mu_u * (v * r.q) + mu_v * (-u * r.inv_q));
      const float om = 1.0f - aa;
      S0 = aa * r.c0 + om * S0;
      S1 = aa * r.c1 + om * S1;
      S2 = aa * r.c2 + om * S2;
      B *= om;
    }
    double* gp = a.grads + (size_t)i * 8;
    if (__popc(ball) <= 2) {
      if (act) {
#pragma unroll
        for (int c = 0; c < 8; ++c)
          if (g[c] != 0.0f) atomicAdd(gp + c, (double)g[c]);
      }
    } else {
      const float tot = step_reduce8(g);
      if ((lane & 3) == 0 && tot != 0.0f) atomicAdd(gp + (lane >> 2), (double)tot);
    }
  }
}

// Fixed-order fold of pf_fit_step's per-warp loss partials into sums[3] (one
// block; used before a cross-rank allreduce -- single-rank steps fold inside
// pf_adam_preprocess instead).
__global__ void __launch_bounds__(1024) k_fold(const double* __restrict__ part, int n_part,
                                               double* sums) {
  __shared__ double red[32][3];
  double v0 = 0.0, v1 = 0.0, v2 = 0.0;
  for (int k = threadIdx.x; k < n_part; k += 1024) {
    v0 += part[3 * k + 0];
    v1 += part[3 * k + 1];
    v2 += part[3 * k + 2];
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    v0 += __shfl_xor_sync(kFull, v0, o);
    v1 += __shfl_xor_sync(kFull, v1, o);
    v2 += __shfl_xor_sync(kFull, v2, o);
  }
  if ((threadIdx.x & 31) == 0) {
    red[threadIdx.x >> 5][0] = v0;
    red[threadIdx.x >> 5][1] = v1;
    red[threadIdx.x >> 5][2] = v2;
  }
  __syncthreads();
  if (threadIdx.x < 3) {
    double s = 0.0;
    for (int w = 0; w < 32; ++w) s += red[w][threadIdx.x];
    sums[threadIdx.x] = s;
  }
}

}  // namespace pf

using namespace pf;

extern "C" int pf_fold_loss(const double* part, int n_part, double* sums, void* stream) {
  if (!part || !sums || n_part < 0) return PF_ERR_ARG;
  k_fold<<<1, 1024, 0, (cudaStream_t)stream>>>(part, n_part, sums);
  return (int)cudaGetLastError();
}

extern "C" size_t pf_step_spill_bytes(int capacity) {
  return (size_t)(capacity > 0 ? capacity : 1) * kTilePix * 2 * sizeof(float4);
}

extern "C" int pf_fit_step(const void* rec, int n, const double* tex, const float* quad,
                           int texels, const int32_t* bin_off, const int32_t* bin_idx,
                           const int32_t* status, int W, int H, int ty_begin, int ty_end,
                           double eps_skip, double bg_r, double bg_g, double bg_b,
                           const float* bg4, int loss_kind, const float* tgt4, double alpha_w,
                           double inv_3P, double inv_P, void* spill, float* img4, double* part,
                           double* grads, void* stream) {
  if (W < 1 || H < 1 || n < 0 || !bin_off || !bin_idx || !status || !tex || !quad || !tgt4 ||
      !spill || !part || !grads)
    return PF_ERR_ARG;
  if (loss_kind != PF_LOSS_MSE && loss_kind != PF_LOSS_SPATIAL) return PF_ERR_ARG;
  const int ntx = div_up(W, kTile), nty = div_up(H, kTile);
  if (ty_begin < 0 || ty_end > nty || ty_begin > ty_end) return PF_ERR_ARG;
  const int n_tiles = (ty_end - ty_begin) * ntx;
  if (n_tiles == 0) return PF_OK;
  StepArgs a;
  a.recf = (const RecF*)rec;
  a.recg = (const RecG*)((const char*)rec + sizeof(RecF) * (size_t)n);
  a.recc = (const RecC*)((const char*)rec + (sizeof(RecF) + sizeof(RecG)) * (size_t)n);
  a.tex = tex;
  a.quad = (const float4*)quad;
  a.texels = texels;
  a.bin_off = bin_off;
  a.bin_idx = bin_idx;
  a.status = status;
  a.W = W;
  a.H = H;
  a.ntx = ntx;
  a.ty_begin = ty_begin;
  a.eps_skip = eps_skip;
  a.bg0 = bg_r;
  a.bg1 = bg_g;
  a.bg2 = bg_b;
  a.bg4 = (const float4*)bg4;
  a.img4 = (float4*)img4;
  a.tgt4 = (const float4*)tgt4;
  a.alpha_w = alpha_w;
  a.inv_3P = inv_3P;
  a.inv_P = inv_P;
  a.part = part;
  a.spill = (float4*)spill;
  a.grads = grads;
  cudaStream_t st = (cudaStream_t)stream;
  const int grid = n_tiles * kStepBlocksPerTile;
  if (loss_kind == PF_LOSS_MSE)
    k_step<PF_LOSS_MSE><<<grid, kStepWarps * 32, 0, st>>>(a);
  else
    k_step<PF_LOSS_SPATIAL><<<grid, kStepWarps * 32, 0, st>>>(a);
  return (int)cudaGetLastError();
}
