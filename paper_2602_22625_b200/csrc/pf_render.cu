// K3 forward and K4 backward render kernels (16x16 tiles, one thread per pixel).
//
// Reference semantics (pkg/src/primfit/_kernels.py):
//   forward_nosave / fill_entries (76-136, 183-255): per pixel, walk the tile's
//   z-ascending list; inverse affine -> texel coords; skip outside the template
//   box; m = bilinear(alpha); skip m < eps_skip; a = alpha_max*sig(nu)*m;
//   C += T*a*c; T *= 1-a; out = C + T*bg, alpha = 1 - T.  No alpha clamp.
//   backward_tiles (258-363): per pixel, reverse sweep over the saved entries
//   with the relative suffix colour S and back-product B (no division by 1-a).
//
// B200 design:
//   forward  - the tile's primitive records (96 B each) are staged into shared
//              memory with cp.async, double-buffered in chunks of 128; each
//              pixel keeps T and C in float64 registers.  The saved state is NOT
//              the reference's CSR (count pass + fill pass): each contributing
//              entry stores (list position j, incoming transmittance T_j) at a
//              fixed slot 256*bin_off[t] + k*256 + pixel (k = per-pixel ordinal),
//              so one pass suffices and the layout is coalesced across a warp.
//              T_j is saved exactly as the reference's Tbuf (_kernels.py:294-297),
//              which keeps the backward exact at alpha == 1.
//              With loss_kind != NONE the MSE / spatial loss, dL/dI (and dL/dA)
//              and per-tile loss partials are fused in; the last block reduces
//              the partials in fixed order (deterministic loss value).
//   backward - each warp iterates its pixels' saved entries back to front,
//              selecting the next list position with __reduce_max_sync, so it
//              only visits entries that touch at least one of its 32 pixels.
//              Active lanes compute the 8 gradients in float64; a 9-shuffle
//              __shfl_xor transpose-butterfly reduces them across the warp and 8
//              lanes issue one float64 atomicAdd each (RED.E.ADD.F64).
#include "../../include/primfit_b200.h"
#include "pf_common.cuh"

namespace pf {

constexpr int kChunk = 128;  // records per cp.async stage (12 KB)

struct FwdArgs {
  const RecF* recf;
  const double* tex;  // planar [4][texels]
  int texels;
  const int32_t* bin_off;
  const int32_t* bin_idx;
  const int32_t* status;
  int W, H, ntx, ty_begin;
  double eps_skip, mu_blend;
  double bg0, bg1, bg2;
  const float* bg_img;
  uint16_t* ent_j;
  double* ent_T;
  int32_t* ent_n;
  float* img;
  float* alpha;
  const float* target;
  const float* target_alpha;
  double alpha_w, inv_3P, inv_P;
  float* dI;
  float* dA;
  double* part;
  uint32_t* counter;
  double* sums;
};

template <int NV>
__device__ __forceinline__ void block_sum(double (&v)[NV], double (*red)[NV]) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int k = 0; k < NV; ++k) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v[k] += __shfl_xor_sync(kFull, v[k], o);
  }
  if (lane == 0) {
#pragma unroll
    for (int k = 0; k < NV; ++k) red[warp][k] = v[k];
  }
  __syncthreads();
  if (threadIdx.x == 0) {
#pragma unroll
    for (int k = 0; k < NV; ++k) {
      double s = 0.0;
      for (int w = 0; w < (int)(blockDim.x >> 5); ++w) s += red[w][k];
      v[k] = s;
    }
  }
}

template <bool SAVE, int LOSS, bool MU>
__global__ void __launch_bounds__(kTilePix) k_forward(FwdArgs a) {
  __shared__ __align__(16) RecF srec[2][kChunk];
  __shared__ double red[kTilePix / 32][3];
  __shared__ bool am_last;

  if (a.status && a.status[1]) return;  // bin overflow: nothing valid to render (block-uniform)

  const int tb = blockIdx.x;
  const int tx = tb % a.ntx, ty = a.ty_begin + tb / a.ntx;
  const int x = tx * kTile + (threadIdx.x & (kTile - 1));
  const int y = ty * kTile + (threadIdx.x / kTile);
  const bool valid = x < a.W && y < a.H;
  const double xx = (double)x, yy = (double)y;

  const int b0 = a.bin_off[tb];
  const int L = a.bin_off[tb + 1] - b0;
  const double* plane_a = a.tex + 3 * (size_t)a.texels;

  double T = 1.0, C0 = 0.0, C1 = 0.0, C2 = 0.0;
  int nsave = 0;
  size_t e = (size_t)b0 * kTilePix + threadIdx.x;

  auto stage_chunk = [&](int stg, int start) {
    const int cnt = min(kChunk, L - start);
    char* dst = reinterpret_cast<char*>(srec[stg]);
    const char* src = reinterpret_cast<const char*>(a.recf);
    for (int pc = threadIdx.x; pc < cnt * 6; pc += kTilePix) {
      const int r = pc / 6, q = pc - r * 6;
      const int i = __ldg(a.bin_idx + b0 + start + r);
      cp_async16(dst + r * 96 + q * 16, src + (size_t)i * 96 + q * 16);
    }
    cp_async_commit();
  };

  if (L > 0) stage_chunk(0, 0);
  int stg = 0;
  for (int start = 0; start < L; start += kChunk) {
    const bool more = start + kChunk < L;
    if (more) {
      stage_chunk(stg ^ 1, start + kChunk);
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncthreads();
    const int cnt = min(kChunk, L - start);
    if (valid) {
      for (int jj = 0; jj < cnt; ++jj) {
        const RecF& r = srec[stg][jj];
        double U, V;
        if (!texel_coords(r, xx, yy, U, V)) continue;
        const Cell c = make_cell(U, V);
        const double m = bilinear(plane_a, r.base, r.wt, r.ht, c);
        if (m < a.eps_skip) continue;
        const double aa = __dmul_rn(r.sa, m);
        double cr = r.c0, cg = r.c1, cb = r.c2;
        if (MU) {
          cr = __dadd_rn(cr, __dmul_rn(a.mu_blend, bilinear(a.tex, r.base, r.wt, r.ht, c)));
          cg = __dadd_rn(cg, __dmul_rn(a.mu_blend,
                                       bilinear(a.tex + a.texels, r.base, r.wt, r.ht, c)));
          cb = __dadd_rn(cb, __dmul_rn(a.mu_blend,
                                       bilinear(a.tex + 2 * (size_t)a.texels, r.base, r.wt,
                                                r.ht, c)));
        }
        if (SAVE) {
          a.ent_j[e] = (uint16_t)(start + jj);
          a.ent_T[e] = T;
          e += kTilePix;
          ++nsave;
        }
        const double Ta = __dmul_rn(T, aa);
        C0 = __dadd_rn(C0, __dmul_rn(Ta, cr));
        C1 = __dadd_rn(C1, __dmul_rn(Ta, cg));
        C2 = __dadd_rn(C2, __dmul_rn(Ta, cb));
        T = __dmul_rn(T, __dsub_rn(1.0, aa));
      }
    }
    __syncthreads();
    stg ^= 1;
  }

  double loss_v[3] = {0.0, 0.0, 0.0};
  if (valid) {
    const size_t pix = (size_t)y * a.W + x;
    double g0 = a.bg0, g1 = a.bg1, g2 = a.bg2;
    if (a.bg_img) {
      g0 = a.bg_img[pix * 3 + 0];
      g1 = a.bg_img[pix * 3 + 1];
      g2 = a.bg_img[pix * 3 + 2];
    }
    const double I0 = __dadd_rn(C0, __dmul_rn(T, g0));
    const double I1 = __dadd_rn(C1, __dmul_rn(T, g1));
    const double I2 = __dadd_rn(C2, __dmul_rn(T, g2));
    const double Ia = 1.0 - T;
    a.img[pix * 3 + 0] = (float)I0;
    a.img[pix * 3 + 1] = (float)I1;
    a.img[pix * 3 + 2] = (float)I2;
    a.alpha[pix] = (float)Ia;
    if (SAVE) a.ent_n[pix] = nsave;
    if (LOSS != PF_LOSS_NONE) {
      // loss_mse (fit.py:112-116) / loss_spatial (fit.py:128-151)
      const double r0 = I0 - (double)a.target[pix * 3 + 0];
      const double r1 = I1 - (double)a.target[pix * 3 + 1];
      const double r2 = I2 - (double)a.target[pix * 3 + 2];
      loss_v[0] = r0 * r0 + r1 * r1 + r2 * r2;
      if (LOSS == PF_LOSS_MSE) {
        const double k = 2.0 * a.inv_3P;
        a.dI[pix * 3 + 0] = (float)(k * r0);
        a.dI[pix * 3 + 1] = (float)(k * r1);
        a.dI[pix * 3 + 2] = (float)(k * r2);
      } else {
        const double ta = (double)a.target_alpha[pix];
        const double mk = ta > 0.0 ? 1.0 : 0.0;
        const double m0 = r0 * mk, m1 = r1 * mk, m2 = r2 * mk;
        loss_v[1] = m0 * m0 + m1 * m1 + m2 * m2;
        const double ad = Ia - ta;
        loss_v[2] = ad * ad;
        const double k = 2.0 * a.inv_3P;
        a.dI[pix * 3 + 0] = (float)(k * m0);
        a.dI[pix * 3 + 1] = (float)(k * m1);
        a.dI[pix * 3 + 2] = (float)(k * m2);
        a.dA[pix] = (float)(a.alpha_w * 2.0 * ad * a.inv_P);
      }
    }
  }

  if (LOSS != PF_LOSS_NONE) {
    block_sum<3>(loss_v, red);
    if (threadIdx.x == 0) {
      a.part[tb * 3 + 0] = loss_v[0];
      a.part[tb * 3 + 1] = loss_v[1];
      a.part[tb * 3 + 2] = loss_v[2];
      __threadfence();
      const unsigned t = atomicAdd(a.counter, 1u);
      am_last = (t == gridDim.x - 1);
    }
    __syncthreads();
    if (am_last) {
      // last block: fixed-order reduction of all tile partials
      __threadfence();
      double v[3] = {0.0, 0.0, 0.0};
      for (int k = threadIdx.x; k < (int)gridDim.x; k += blockDim.x) {
        v[0] += __ldcg(a.part + k * 3 + 0);
        v[1] += __ldcg(a.part + k * 3 + 1);
        v[2] += __ldcg(a.part + k * 3 + 2);
      }
      __syncthreads();
      block_sum<3>(v, red);
      if (threadIdx.x == 0) {
        a.sums[0] = v[0];
        a.sums[1] = LOSS == PF_LOSS_MSE ? v[0] : v[1];
        a.sums[2] = v[2];
        *a.counter = 0u;
      }
    }
  }
}

struct BwdArgs {
  const RecF* recf;
  const RecB* recb;
  const double* tex;
  int texels;
  const int32_t* bin_off;
  const int32_t* bin_idx;
  const int32_t* status;
  const uint16_t* ent_j;
  const double* ent_T;
  const int32_t* ent_n;
  const float* dI;
  const float* dA;
  double bg0, bg1, bg2;
  const float* bg_img;
  double mu_blend;
  int W, H, ntx, ty_begin;
  double* grads;
};

// Sum 8 values over the warp with a transpose butterfly (9 shuffles instead of
// 40): afterwards lane l holds the warp total of value ((l >> 2) & 7).
__device__ __forceinline__ double warp_reduce8(const double (&g)[8]) {
  const int lane = threadIdx.x & 31;
  double w[4];
  const bool h16 = lane & 16;
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const double send = h16 ? g[q] : g[q + 4];
    const double keep = h16 ? g[q + 4] : g[q];
    w[q] = keep + __shfl_xor_sync(kFull, send, 16);
  }
  double x2[2];
  const bool h8 = lane & 8;
#pragma unroll
  for (int q = 0; q < 2; ++q) {
    const double send = h8 ? w[q] : w[q + 2];
    const double keep = h8 ? w[q + 2] : w[q];
    x2[q] = keep + __shfl_xor_sync(kFull, send, 8);
  }
  const bool h4 = lane & 4;
  double y = (h4 ? x2[1] : x2[0]) + __shfl_xor_sync(kFull, h4 ? x2[0] : x2[1], 4);
  y += __shfl_xor_sync(kFull, y, 2);
  y += __shfl_xor_sync(kFull, y, 1);
  return y;
}

template <bool MU, bool HAS_DA>
__global__ void __launch_bounds__(kTilePix) k_backward(BwdArgs a) {
  if (a.status && a.status[1]) return;
  const int tb = blockIdx.x;
  const int tx = tb % a.ntx, ty = a.ty_begin + tb / a.ntx;
  const int x = tx * kTile + (threadIdx.x & (kTile - 1));
  const int y = ty * kTile + (threadIdx.x / kTile);
  const bool valid = x < a.W && y < a.H;
  const int lane = threadIdx.x & 31;
  const double xx = (double)x, yy = (double)y;
  const int b0 = a.bin_off[tb];
  const double* plane_a = a.tex + 3 * (size_t)a.texels;

  const size_t pix = valid ? (size_t)y * a.W + x : 0;
  int k = valid ? a.ent_n[pix] - 1 : -1;
  size_t e = (size_t)b0 * kTilePix + threadIdx.x + (size_t)(k > 0 ? k : 0) * kTilePix;
  unsigned key = 0;
  double Tk = 0.0;
  if (k >= 0) {
    key = (unsigned)a.ent_j[e] + 1u;
    Tk = a.ent_T[e];
  }
  double dI0 = 0.0, dI1 = 0.0, dI2 = 0.0, dA = 0.0;
  double g0 = a.bg0, g1 = a.bg1, g2 = a.bg2;
  if (valid) {
    dI0 = a.dI[pix * 3 + 0];
    dI1 = a.dI[pix * 3 + 1];
    dI2 = a.dI[pix * 3 + 2];
    if (HAS_DA) dA = a.dA[pix];
    if (a.bg_img) {
      g0 = a.bg_img[pix * 3 + 0];
      g1 = a.bg_img[pix * 3 + 1];
      g2 = a.bg_img[pix * 3 + 2];
    }
  }
  double S0 = 0.0, S1 = 0.0, S2 = 0.0, B = 1.0;

  while (true) {
    const unsigned jm = __reduce_max_sync(kFull, key);
    if (jm == 0u) break;
    const bool act = key == jm;
    const int i = __ldg(a.bin_idx + b0 + (int)(jm - 1u));
    double g[8];
#pragma unroll
    for (int c = 0; c < 8; ++c) g[c] = 0.0;
    if (act) {
      const RecF r = a.recf[i];
      const RecB rb = a.recb[i];
      double U, V;
      texel_coords(r, xx, yy, U, V);
      const Cell c = make_cell(U, V);
      double gU, gV;
      const double m = bilinear_grad(plane_a, r.base, r.wt, r.ht, c, gU, gV);
      const double aa = __dmul_rn(r.sa, m);
      double ck0 = r.c0, ck1 = r.c1, ck2 = r.c2;
      if (MU) {
        ck0 = __dadd_rn(ck0, __dmul_rn(a.mu_blend, bilinear(a.tex, r.base, r.wt, r.ht, c)));
        ck1 = __dadd_rn(ck1, __dmul_rn(a.mu_blend,
                                       bilinear(a.tex + a.texels, r.base, r.wt, r.ht, c)));
        ck2 = __dadd_rn(ck2, __dmul_rn(a.mu_blend, bilinear(a.tex + 2 * (size_t)a.texels,
                                                            r.base, r.wt, r.ht, c)));
      }
      // _kernels.py:319-359
      const double gg = dI0 * (ck0 - S0 - g0 * B) + dI1 * (ck1 - S1 - g1 * B) +
                        dI2 * (ck2 - S2 - g2 * B) + dA * B;
      const double dalpha = Tk * gg;
      g[4] = dalpha * rb.sd * m;
      if (rb.one_minus_mu > 0.0) {
        const double wc = Tk * aa * rb.one_minus_mu;
        g[5] = dI0 * wc * rb.cd0;
        g[6] = dI1 * wc * rb.cd1;
        g[7] = dI2 * wc * rb.cd2;
      }
      const double dm = dalpha * r.sa;
      const double hw = 0.5 * (double)(r.wt - 1), hh = 0.5 * (double)(r.ht - 1);
      const double mu_u = gU * hw, mu_v = gV * hh;
      const double u = U / hw - 1.0, v = V / hh - 1.0;
      g[0] = dm * (mu_u * rb.gxu + mu_v * rb.gxv);
      g[1] = dm * (mu_u * rb.gyu + mu_v * rb.gyv);
      g[2] = dm * (mu_u * (-u * rb.inv_s) + mu_v * (-v * rb.inv_s));
      g[3] = dm * (mu_u * (v * rb.q) + mu_v * (-u * rb.inv_q));
      const double om = 1.0 - aa;
      S0 = aa * ck0 + om * S0;
      S1 = aa * ck1 + om * S1;
      S2 = aa * ck2 + om * S2;
      B *= om;
      --k;
      if (k >= 0) {
        e -= kTilePix;
        key = (unsigned)a.ent_j[e] + 1u;
        Tk = a.ent_T[e];
      } else {
        key = 0;
      }
    }
    const unsigned ball = __ballot_sync(kFull, act);
    double* gp = a.grads + (size_t)i * 8;
    if ((ball & (ball - 1u)) == 0u) {
      if (act) {
#pragma unroll
        for (int c = 0; c < 8; ++c)
          if (g[c] != 0.0) atomicAdd(gp + c, g[c]);
      }
    } else {
      const double tot = warp_reduce8(g);
      if ((lane & 3) == 0 && tot != 0.0) atomicAdd(gp + (lane >> 2), tot);
    }
  }
}

}  // namespace pf

using namespace pf;

extern "C" int pf_forward(const void* rec, int n, const double* tex, int texels,
                          const int32_t* bin_off, const int32_t* bin_idx, const int32_t* status,
                          int W, int H, int ty_begin, int ty_end, double eps_skip,
                          double mu_blend, double bg_r, double bg_g, double bg_b,
                          const float* bg_img, uint16_t* ent_j, double* ent_T, int32_t* ent_n,
                          float* img, float* alpha, int loss_kind, const float* target,
                          const float* target_alpha, double alpha_w, double inv_3P, double inv_P,
                          float* dI, float* dA, double* part, uint32_t* counter, double* sums,
                          void* stream) {
  if (W < 1 || H < 1 || n < 0 || !bin_off || !img || !alpha) return PF_ERR_ARG;
  const int ntx = div_up(W, kTile), nty = div_up(H, kTile);
  if (ty_begin < 0 || ty_end > nty || ty_begin > ty_end) return PF_ERR_ARG;
  const bool save = ent_j != nullptr;
  if (save && (!ent_T || !ent_n)) return PF_ERR_ARG;
  if (loss_kind != PF_LOSS_NONE) {
    if (!target || !dI || !part || !counter || !sums) return PF_ERR_ARG;
    if (loss_kind == PF_LOSS_SPATIAL && (!target_alpha || !dA)) return PF_ERR_ARG;
    if (loss_kind != PF_LOSS_MSE && loss_kind != PF_LOSS_SPATIAL) return PF_ERR_ARG;
  }
  const int n_tiles = (ty_end - ty_begin) * ntx;
  if (n_tiles == 0) return PF_OK;
  FwdArgs a;
  a.recf = (const RecF*)rec;
  a.tex = tex;
  a.texels = texels;
  a.bin_off = bin_off;
  a.bin_idx = bin_idx;
  a.status = status;
  a.W = W;
  a.H = H;
  a.ntx = ntx;
  a.ty_begin = ty_begin;
  a.eps_skip = eps_skip;
  a.mu_blend = mu_blend;
  a.bg0 = bg_r;
  a.bg1 = bg_g;
  a.bg2 = bg_b;
  a.bg_img = bg_img;
  a.ent_j = ent_j;
  a.ent_T = ent_T;
  a.ent_n = ent_n;
  a.img = img;
  a.alpha = alpha;
  a.target = target;
  a.target_alpha = target_alpha;
  a.alpha_w = alpha_w;
  a.inv_3P = inv_3P;
  a.inv_P = inv_P;
  a.dI = dI;
  a.dA = dA;
  a.part = part;
  a.counter = counter;
  a.sums = sums;
  cudaStream_t st = (cudaStream_t)stream;
  const bool mu = mu_blend > 0.0;
#define PF_FWD(SV, LS, MUV) k_forward<SV, LS, MUV><<<n_tiles, kTilePix, 0, st>>>(a)
#define PF_FWD_MU(SV, LS) \
  if (mu) PF_FWD(SV, LS, true); else PF_FWD(SV, LS, false)
  if (save) {
    if (loss_kind == PF_LOSS_MSE) { PF_FWD_MU(true, PF_LOSS_MSE); }
    else if (loss_kind == PF_LOSS_SPATIAL) { PF_FWD_MU(true, PF_LOSS_SPATIAL); }
    else { PF_FWD_MU(true, PF_LOSS_NONE); }
  } else {
    if (loss_kind == PF_LOSS_MSE) { PF_FWD_MU(false, PF_LOSS_MSE); }
    else if (loss_kind == PF_LOSS_SPATIAL) { PF_FWD_MU(false, PF_LOSS_SPATIAL); }
    else { PF_FWD_MU(false, PF_LOSS_NONE); }
  }
#undef PF_FWD_MU
#undef PF_FWD
  return (int)cudaGetLastError();
}

extern "C" int pf_backward(const void* rec, int n, const double* tex, int texels,
                           const int32_t* bin_off, const int32_t* bin_idx, const int32_t* status,
                           const uint16_t* ent_j, const double* ent_T, const int32_t* ent_n,
                           const float* dI, const float* dA, double bg_r, double bg_g,
                           double bg_b, const float* bg_img, double mu_blend, int W, int H,
                           int ty_begin, int ty_end, double* grads, void* stream) {
  if (W < 1 || H < 1 || n < 0 || !bin_off || !ent_j || !ent_T || !ent_n || !dI || !grads)
    return PF_ERR_ARG;
  const int ntx = div_up(W, kTile), nty = div_up(H, kTile);
  if (ty_begin < 0 || ty_end > nty || ty_begin > ty_end) return PF_ERR_ARG;
  const int n_tiles = (ty_end - ty_begin) * ntx;
  if (n_tiles == 0) return PF_OK;
  BwdArgs a;
  a.recf = (const RecF*)rec;
  a.recb = (const RecB*)((const char*)rec + sizeof(RecF) * (size_t)n);
  a.tex = tex;
  a.texels = texels;
  a.bin_off = bin_off;
  a.bin_idx = bin_idx;
  a.status = status;
  a.ent_j = ent_j;
  a.ent_T = ent_T;
  a.ent_n = ent_n;
  a.dI = dI;
  a.dA = dA;
  a.bg0 = bg_r;
  a.bg1 = bg_g;
  a.bg2 = bg_b;
  a.bg_img = bg_img;
  a.mu_blend = mu_blend;
  a.W = W;
  a.H = H;
  a.ntx = ntx;
  a.ty_begin = ty_begin;
  a.grads = grads;
  cudaStream_t st = (cudaStream_t)stream;
  const bool mu = mu_blend > 0.0;
  if (mu) {
    if (dA) k_backward<true, true><<<n_tiles, kTilePix, 0, st>>>(a);
    else k_backward<true, false><<<n_tiles, kTilePix, 0, st>>>(a);
  } else {
    if (dA) k_backward<false, true><<<n_tiles, kTilePix, 0, st>>>(a);
    else k_backward<false, false><<<n_tiles, kTilePix, 0, st>>>(a);
  }
  return (int)cudaGetLastError();
}
