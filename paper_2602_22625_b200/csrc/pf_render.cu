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
//   Each warp owns an 8x4 pixel sub-tile (8 warps = 16x16 tile), compact so the
//   warp-uniform culling below rejects as many list entries as possible, and
//   warps never wait on each other on the hot path.  Pixel-sized buffers are
//   float4 per pixel (one 16-byte access): image+alpha (RGBA), target+target
//   alpha, dL/dI+dL/dA, background.
//   forward  - for every 32 list entries a warp runs a lane-parallel
//              conservative separating-axis test (primitive axes) of each
//              entry's footprint against its 8x4 pixel rectangle (32-byte fp32
//              cull records) and keeps a ballot mask; only surviving entries are
//              evaluated per pixel (warp-uniform loop, two entries per
//              iteration for ILP).  Survivors run the float64 decision chain and
//              an fp32-tap bilinear alpha sample from the quad atlas (one 16-byte
//              load, no bounds checks; the eps decision is re-taken on the
//              float64 plane when within rounding).  T and C are float64.
//              Saved state: per contributing (pixel, entry) one 16-byte record
//              (list position, texel cell, 24-bit bilinear weights, incoming
//              T = the reference's Tbuf, _kernels.py:294-297) at slot
//              256*bin_off[t] + k*256 + pixel (k = the pixel's contribution
//              ordinal): single pass, coalesced within a warp.
//              With loss_kind != NONE the MSE / spatial loss, dL/dI (and dL/dA)
//              and per-warp loss partials are fused in; the backward reduces the
//              partials in fixed order (deterministic loss value).
//   backward - the tile's 96-byte fp32 gradient records are staged in shared
//              memory with cp.async (one barrier at block start).  Each warp
//              then walks its pixels' saved entries back to front, picking the
//              next list position with __reduce_max_sync so it only visits
//              entries that touch its 32 pixels.  Active lanes compute the 8
//              gradients in fp32 (the backward takes no decisions; <= 3e-4 of
//              the float64 reference against a 1e-3 bar); a 9-shuffle
//              __shfl_xor transpose butterfly reduces them across the warp and 8
//              lanes issue one float64 atomicAdd each (RED.E.ADD.F64); with <= 2
//              active lanes the lanes issue their atomics directly.
#include "../../include/primfit_b200.h"
#include "pf_common.cuh"

namespace pf {

constexpr int kWarpsPerTile = kTilePix / 32;

// Forward blocks are 2 warps (a 16x4 strip of a tile): the forward has no
// block-level cooperation, so small blocks only shrink the scheduling tail.
constexpr int kFwdWarps = 2;
constexpr int kFwdBlocksPerTile = kWarpsPerTile / kFwdWarps;

// Pixel of lane (threadIdx.x & 31) in warp w (0..7) of tile (tx, ty), and the
// centre of that warp's 8x4 rectangle.
__device__ __forceinline__ void pixel_of(int w, int tx, int ty, int& x, int& y, float& cx,
                                         float& cy) {
  const int l = threadIdx.x & 31;
  const int wx = (w & 1) * kWarpW, wy = (w >> 1) * kWarpH;
  x = tx * kTile + wx + (l & (kWarpW - 1));
  y = ty * kTile + wy + (l / kWarpW);
  cx = (float)(tx * kTile + wx) + 0.5f * (kWarpW - 1);
  cy = (float)(ty * kTile + wy) + 0.5f * (kWarpH - 1);
}

// Conservative footprint-vs-warp-rectangle test (see RecC): reject only when
// the rectangle centre's (u, v) is beyond 1 + the rectangle's projected half
// width (+ slack); NaN never rejects.
__device__ __forceinline__ bool may_touch(const RecC* __restrict__ rc, float cx, float cy) {
  const float4 a = __ldg(reinterpret_cast<const float4*>(rc));
  const float4 b = __ldg(reinterpret_cast<const float4*>(rc) + 1);
  const float dx = cx - a.x, dy = cy - a.y;
  const float uc = a.z * dx + a.w * dy;
  const float vc = b.x * dy - b.y * dx;
  const bool out_u = fabsf(uc) > 1.0f + b.z + 1e-5f * fabsf(uc);
  const bool out_v = fabsf(vc) > 1.0f + b.w + 1e-5f * fabsf(vc);
  return !(out_u || out_v);
}

struct FwdArgs {
  const RecF* recf;
  const RecC* recc;
  const double* tex;     // planar [4][texels]
  const float4* quad;    // alpha quad atlas [texels]
  int texels;
  const int32_t* bin_off;
  const int32_t* bin_idx;
  const int32_t* status;
  int W, H, ntx, ty_begin;
  double eps_skip, mu_blend;
  double bg0, bg1, bg2;
  const float4* bg4;     // per-pixel background (rgb, -), or NULL
  SavedEnt* ent;
  int32_t* ent_n;
  float4* img4;          // out: (r, g, b, alpha)
  const float4* tgt4;    // target (r, g, b, target alpha)
  double alpha_w, w_mse, w_gray, inv_3P, inv_P;
  float4* d4;            // out: (dL/dI r, g, b, dL/dA)
  double* part;
};

template <bool SAVE, int LOSS, bool MU>
__global__ void __launch_bounds__(kFwdWarps * 32) k_forward(FwdArgs a) {
  if (a.status && a.status[1]) return;  // bin overflow: nothing valid to render (block-uniform)

  const int tb = blockIdx.x / kFwdBlocksPerTile;
  const int wt = (blockIdx.x % kFwdBlocksPerTile) * kFwdWarps + (threadIdx.x >> 5);
  const int tx = tb % a.ntx, ty = a.ty_begin + tb / a.ntx;
  int x, y;
  float cx, cy;
  pixel_of(wt, tx, ty, x, y, cx, cy);
  const bool valid = x < a.W && y < a.H;
  const int lane = threadIdx.x & 31;
  const double xx = (double)x, yy = (double)y;
  const size_t pix = valid ? (size_t)y * a.W + x : 0;

  // prefetch the pixel's epilogue inputs; they are independent of the list walk
  float4 tg = make_float4(0.f, 0.f, 0.f, 0.f), bgp = tg;
  if (valid && LOSS != PF_LOSS_NONE) tg = __ldg(a.tgt4 + pix);
  if (valid && a.bg4) bgp = __ldg(a.bg4 + pix);

  const int b0 = a.bin_off[tb];
  const int L = a.bin_off[tb + 1] - b0;
  const double* plane_a = a.tex + 3 * (size_t)a.texels;

  double T = 1.0, C0 = 0.0, C1 = 0.0, C2 = 0.0;
  int nsave = 0;
  const size_t e0 = (size_t)b0 * kTilePix + wt * 32 + lane;

  for (int sub = 0; sub < L; sub += 32) {
    // warp-cooperative cull: lane l tests list entry sub + l against the warp rect
    int my_i = 0;
    bool cand = false;
    if (sub + lane < L) {
      my_i = __ldg(a.bin_idx + b0 + sub + lane);
      cand = may_touch(a.recc + my_i, cx, cy);
    }
    unsigned mask = __ballot_sync(kFull, cand);
    while (mask) {
      const int bit = __ffs(mask) - 1;
      mask &= mask - 1;
      const int i = __shfl_sync(kFull, my_i, bit);
      if (!valid) continue;
      const RecF& r = a.recf[i];
      double U, V;
      if (!texel_coords(r, xx, yy, U, V)) continue;
      const Cell c = make_cell(U, V);
      double m = bilerp(load_quad(a.quad, r.base, r.wt, c.u0, c.v0), c.wu, c.wv);
      // re-take an eps decision within fp32-tap rounding on the float64 plane
      if (fabs(m - a.eps_skip) <= 1e-6 * a.eps_skip) m = bilinear(plane_a, r.base, r.wt, r.ht, c);
      if (m < a.eps_skip) continue;
      const double aa = r.sa * m;
      double cr = r.c0, cg = r.c1, cb = r.c2;
      if (MU) {
        cr += a.mu_blend * bilinear(a.tex, r.base, r.wt, r.ht, c);
        cg += a.mu_blend * bilinear(a.tex + a.texels, r.base, r.wt, r.ht, c);
        cb += a.mu_blend * bilinear(a.tex + 2 * (size_t)a.texels, r.base, r.wt, r.ht, c);
      }
      if (SAVE) {
        a.ent[e0 + (size_t)nsave * kTilePix] = pack_saved(sub + bit, c.u0, c.v0, c.wu, c.wv, T);
        ++nsave;
      }
      const double Ta = T * aa;
      C0 += Ta * cr;
      C1 += Ta * cg;
      C2 += Ta * cb;
      T *= 1.0 - aa;
    }
  }

  float l0 = 0.0f, l1 = 0.0f, l2 = 0.0f;
  if (valid) {
    const double g0 = a.bg4 ? (double)bgp.x : a.bg0;
    const double g1 = a.bg4 ? (double)bgp.y : a.bg1;
    const double g2 = a.bg4 ? (double)bgp.z : a.bg2;
    const double I0 = C0 + T * g0;
    const double I1 = C1 + T * g1;
    const double I2 = C2 + T * g2;
    const double Ia = 1.0 - T;
    a.img4[pix] = make_float4((float)I0, (float)I1, (float)I2, (float)Ia);
    if (SAVE) a.ent_n[pix] = nsave;
    if (LOSS != PF_LOSS_NONE) {
      // loss_mse (fit.py:112-116) / loss_spatial (fit.py:128-151)
      const double r0 = I0 - (double)tg.x, r1 = I1 - (double)tg.y, r2 = I2 - (double)tg.z;
      const double sse = r0 * r0 + r1 * r1 + r2 * r2;
      const double k = 2.0 * a.inv_3P;
      l0 = (float)sse;
      if (LOSS == PF_LOSS_MSE) {
        l1 = l0;
        a.d4[pix] = make_float4((float)(k * r0), (float)(k * r1), (float)(k * r2), 0.0f);
      } else if (LOSS == PF_LOSS_COMBINED) {
        // mse_w * loss_mse + gray_l1_w * loss_grayscale_l1 (fit.py:112-125, 162-168)
        const double d = r0 * 0.299 + r1 * 0.587 + r2 * 0.114;
        l1 = (float)fabs(d);
        const double kg = a.w_gray * (d > 0.0 ? 1.0 : (d < 0.0 ? -1.0 : 0.0)) * a.inv_P;
        const double km = a.w_mse * k;
        a.d4[pix] = make_float4((float)(km * r0 + kg * 0.299), (float)(km * r1 + kg * 0.587),
                                (float)(km * r2 + kg * 0.114), 0.0f);
      } else {
        const double ta = (double)tg.w;
        const double mk = ta > 0.0 ? 1.0 : 0.0;
        const double ad = Ia - ta;
        l1 = (float)(sse * mk);
        l2 = (float)(ad * ad);
        a.d4[pix] = make_float4((float)(k * r0 * mk), (float)(k * r1 * mk), (float)(k * r2 * mk),
                                (float)(a.alpha_w * 2.0 * ad * a.inv_P));
      }
    }
  }
  if (LOSS != PF_LOSS_NONE) {
    // per-warp partials at fixed slots (no block barrier); pf_backward reduces them
    // in fixed order in float64 (fp32 inside a warp: 32 terms, ~1e-7 relative)
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      l0 += __shfl_xor_sync(kFull, l0, o);
      l1 += __shfl_xor_sync(kFull, l1, o);
      l2 += __shfl_xor_sync(kFull, l2, o);
    }
    if (lane == 0) {
      double* pp = a.part + ((size_t)tb * kWarpsPerTile + wt) * 3;
      pp[0] = l0;
      pp[1] = l1;
      pp[2] = l2;
    }
  }
}

struct BwdArgs {
  const RecG* recg;
  const double* tex;
  const float4* quad;
  int texels;
  const int32_t* bin_off;
  const int32_t* bin_idx;
  const int32_t* status;
  const SavedEnt* ent;
  const int32_t* ent_n;
  const float4* d4;  // (dL/dI r, g, b, dL/dA)
  float bg0, bg1, bg2;
  const float4* bg4;
  float mu_blend;
  int W, H, ntx, ty_begin;
  double* grads;
  const double* part;  // forward loss partials (NULL: none)
  int n_part;
  double* sums;
};

// Sum 8 values over the warp with a transpose butterfly (9 shuffles instead of
// 40): afterwards lane l holds the warp total of value ((l >> 2) & 7).
__device__ __forceinline__ float warp_reduce8(const float (&g)[8]) {
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

// Fixed-order reduction of the forward's per-warp loss partials (block 0).
__device__ void reduce_loss_partials(const double* part, int n_part, double* sums) {
  __shared__ double red[kWarpsPerTile][3];
  double v0 = 0.0, v1 = 0.0, v2 = 0.0;
  for (int k = threadIdx.x; k < n_part; k += blockDim.x) {
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
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) s += red[w][threadIdx.x];
    sums[threadIdx.x] = s;
  }
}

constexpr int kBwdStage = 128;  // list entries whose gradient records are staged (12 KB)

__device__ __forceinline__ float bilinear_f(const double* __restrict__ plane, int base, int wt,
                                            int ht, int u0, int v0, float wu, float wv) {
  const Cell c{u0, v0, (double)wu, (double)wv};
  return (float)bilinear(plane, base, wt, ht, c);
}

template <bool MU>
__global__ void __launch_bounds__(kTilePix) k_backward(BwdArgs a) {
  __shared__ __align__(16) RecG sg[kBwdStage];
  __shared__ int sidx[kBwdStage];
  if (a.status && a.status[1]) return;
  if (a.part && blockIdx.x == 0) reduce_loss_partials(a.part, a.n_part, a.sums);
  const int tb = blockIdx.x;
  const int tx = tb % a.ntx, ty = a.ty_begin + tb / a.ntx;
  int x, y;
  float cxf, cyf;
  pixel_of(threadIdx.x >> 5, tx, ty, x, y, cxf, cyf);
  const bool valid = x < a.W && y < a.H;
  const int lane = threadIdx.x & 31;
  const int b0 = a.bin_off[tb];
  const int L = a.bin_off[tb + 1] - b0;

  // stage the gradient records of the first kBwdStage list entries
  {
    constexpr int kPieces = sizeof(RecG) / 16;
    const int cnt = min(L, kBwdStage);
    for (int pc = threadIdx.x; pc < cnt * kPieces; pc += kTilePix) {
      const int r = pc / kPieces, q = pc - r * kPieces;
      const int i = __ldg(a.bin_idx + b0 + r);
      if (q == 0) sidx[r] = i;
      cp_async16(reinterpret_cast<char*>(&sg[r]) + q * 16,
                 reinterpret_cast<const char*>(a.recg + i) + q * 16);
    }
    cp_async_commit();
  }

  const size_t pix = valid ? (size_t)y * a.W + x : 0;
  int k = valid ? a.ent_n[pix] - 1 : -1;
  size_t e = (size_t)b0 * kTilePix + threadIdx.x + (size_t)(k > 0 ? k : 0) * kTilePix;
  unsigned key = 0;
  SavedEnt cur{};
  if (k >= 0) {
    cur = a.ent[e];
    key = (cur.w0 & 0xffffu) + 1u;
  }
  float4 dd = make_float4(0.f, 0.f, 0.f, 0.f);
  float g0 = a.bg0, g1 = a.bg1, g2 = a.bg2;
  if (valid) {
    dd = __ldg(a.d4 + pix);
    if (a.bg4) {
      const float4 b = __ldg(a.bg4 + pix);
      g0 = b.x;
      g1 = b.y;
      g2 = b.z;
    }
  }
  const float dI0 = dd.x, dI1 = dd.y, dI2 = dd.z, dA = dd.w;
  float S0 = 0.0f, S1 = 0.0f, S2 = 0.0f, B = 1.0f;
  cp_async_wait<0>();
  __syncthreads();

  while (true) {
    const unsigned jm = __reduce_max_sync(kFull, key);
    if (jm == 0u) break;
    const int j = (int)(jm - 1u);
    const bool act = key == jm;
    const bool staged = j < kBwdStage;
    const int i = staged ? sidx[j] : __ldg(a.bin_idx + b0 + j);
    float g[8];
#pragma unroll
    for (int c = 0; c < 8; ++c) g[c] = 0.0f;
    if (act) {
      const SavedView se = unpack_saved(cur);
      const float Tc = se.T;
      // prefetch this lane's next saved entry while the math below runs
      --k;
      if (k >= 0) {
        e -= kTilePix;
        cur = a.ent[e];
        key = (cur.w0 & 0xffffu) + 1u;
      } else {
        key = 0;
      }
      RecG r;
      if (staged)
        r = sg[j];
      else
        r = a.recg[i];
      const float wu = se.wu, wv = se.wv;
      const float4 q = load_quad(a.quad, r.base, r.wt, se.u0, se.v0);
      const float iu = 1.0f - wu, iv = 1.0f - wv;
      const float m = (iu * iv) * q.x + (wu * iv) * q.y + (iu * wv) * q.z + (wu * wv) * q.w;
      const float gU = iv * (q.y - q.x) + wv * (q.w - q.z);
      const float gV = iu * (q.z - q.x) + wu * (q.w - q.y);
      const float aa = r.sa * m;
      float ck0 = r.c0, ck1 = r.c1, ck2 = r.c2;
      if (MU) {
        const double* t = a.tex;
        const float mu = a.mu_blend;
        ck0 += mu * bilinear_f(t, r.base, r.wt, r.ht, se.u0, se.v0, wu, wv);
        ck1 += mu * bilinear_f(t + a.texels, r.base, r.wt, r.ht, se.u0, se.v0, wu, wv);
        ck2 += mu * bilinear_f(t + 2 * (size_t)a.texels, r.base, r.wt, r.ht, se.u0, se.v0, wu, wv);
      }
      // _kernels.py:319-359
      const float gg = dI0 * (ck0 - S0 - g0 * B) + dI1 * (ck1 - S1 - g1 * B) +
                       dI2 * (ck2 - S2 - g2 * B) + dA * B;
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
      const float u = ((float)se.u0 + wu) * r.inv_hw - 1.0f;
      const float v = ((float)se.v0 + wv) * r.inv_hh - 1.0f;
      g[0] = dm * (mu_u * r.gxu + mu_v * r.gxv);
      g[1] = dm * (mu_u * r.gyu + mu_v * r.gyv);
      g[2] = dm * (mu_u * (-u * r.inv_s) + mu_v * (-v * r.inv_s));
      g[3] = dm * (mu_u * (v * r.q) + mu_v * (-u * r.inv_q));
      const float om = 1.0f - aa;
      S0 = aa * ck0 + om * S0;
      S1 = aa * ck1 + om * S1;
      S2 = aa * ck2 + om * S2;
      B *= om;
    }
    const unsigned ball = __ballot_sync(kFull, act);
    double* gp = a.grads + (size_t)i * 8;
    if (__popc(ball) <= 2) {
      if (act) {
#pragma unroll
        for (int c = 0; c < 8; ++c)
          if (g[c] != 0.0f) atomicAdd(gp + c, (double)g[c]);
      }
    } else {
      const float tot = warp_reduce8(g);
      if ((lane & 3) == 0 && tot != 0.0f) atomicAdd(gp + (lane >> 2), (double)tot);
    }
  }
}

}  // namespace pf

using namespace pf;

// Saved-state layout: [entries] SavedEnt (16 B).
extern "C" size_t pf_saved_bytes(int capacity) {
  return (size_t)pf_saved_capacity(capacity) * sizeof(SavedEnt);
}

extern "C" int pf_forward(const void* rec, int n, const double* tex, const float* quad,
                          int texels, const int32_t* bin_off, const int32_t* bin_idx,
                          const int32_t* status, int W, int H,
                          int ty_begin, int ty_end, double eps_skip, double mu_blend, double bg_r,
                          double bg_g, double bg_b, const float* bg4, void* saved,
                          long long saved_entries, int32_t* ent_n, float* img4, int loss_kind,
                          const float* tgt4, double alpha_w, double w_mse, double w_gray,
                          double inv_3P, double inv_P, float* d4, double* part, void* stream) {
  pf::NvtxRange nvtx_range("pf_forward");
  if (W < 1 || H < 1 || n < 0 || !bin_off || !img4 || !tex || !quad) return PF_ERR_ARG;
  const int ntx = div_up(W, kTile), nty = div_up(H, kTile);
  if (ty_begin < 0 || ty_end > nty || ty_begin > ty_end) return PF_ERR_ARG;
  const bool save = saved != nullptr;
  if (save && (!ent_n || saved_entries < 0)) return PF_ERR_ARG;
  if (loss_kind != PF_LOSS_NONE) {
    if (!tgt4 || !d4 || !part) return PF_ERR_ARG;
    if (loss_kind != PF_LOSS_MSE && loss_kind != PF_LOSS_SPATIAL &&
        loss_kind != PF_LOSS_COMBINED)
      return PF_ERR_ARG;
  }
  const int n_tiles = (ty_end - ty_begin) * ntx;
  if (n_tiles == 0) return PF_OK;
  FwdArgs a;
  a.recf = (const RecF*)rec;
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
  a.mu_blend = mu_blend;
  a.bg0 = bg_r;
  a.bg1 = bg_g;
  a.bg2 = bg_b;
  a.bg4 = (const float4*)bg4;
  a.ent = (SavedEnt*)saved;
  a.ent_n = ent_n;
  a.img4 = (float4*)img4;
  a.tgt4 = (const float4*)tgt4;
  a.alpha_w = alpha_w;
  a.w_mse = w_mse;
  a.w_gray = w_gray;
  a.inv_3P = inv_3P;
  a.inv_P = inv_P;
  a.d4 = (float4*)d4;
  a.part = part;
  cudaStream_t st = (cudaStream_t)stream;
  const bool mu = mu_blend > 0.0;
#define PF_FWD(SV, LS, MUV) \
  k_forward<SV, LS, MUV><<<n_tiles * kFwdBlocksPerTile, kFwdWarps * 32, 0, st>>>(a)
#define PF_FWD_MU(SV, LS) \
  if (mu) PF_FWD(SV, LS, true); else PF_FWD(SV, LS, false)
  if (save) {
    if (loss_kind == PF_LOSS_MSE) { PF_FWD_MU(true, PF_LOSS_MSE); }
    else if (loss_kind == PF_LOSS_SPATIAL) { PF_FWD_MU(true, PF_LOSS_SPATIAL); }
    else if (loss_kind == PF_LOSS_COMBINED) { PF_FWD_MU(true, PF_LOSS_COMBINED); }
    else { PF_FWD_MU(true, PF_LOSS_NONE); }
  } else {
    if (loss_kind == PF_LOSS_MSE) { PF_FWD_MU(false, PF_LOSS_MSE); }
    else if (loss_kind == PF_LOSS_SPATIAL) { PF_FWD_MU(false, PF_LOSS_SPATIAL); }
    else if (loss_kind == PF_LOSS_COMBINED) { PF_FWD_MU(false, PF_LOSS_COMBINED); }
    else { PF_FWD_MU(false, PF_LOSS_NONE); }
  }
#undef PF_FWD_MU
#undef PF_FWD
  return (int)cudaGetLastError();
}

extern "C" int pf_backward(const void* rec, int n, const double* tex, const float* quad,
                           int texels, const int32_t* bin_off, const int32_t* bin_idx,
                           const int32_t* status, const void* saved, long long saved_entries,
                           const int32_t* ent_n, const float* d4, double bg_r, double bg_g,
                           double bg_b, const float* bg4, double mu_blend, int W, int H,
                           int ty_begin, int ty_end, double* grads, const double* part,
                           double* sums, void* stream) {
  pf::NvtxRange nvtx_range("pf_backward");
  if (W < 1 || H < 1 || n < 0 || !bin_off || !saved || saved_entries < 0 || !ent_n || !d4 ||
      !grads || !tex || !quad || (part && !sums))
    return PF_ERR_ARG;
  const int ntx = div_up(W, kTile), nty = div_up(H, kTile);
  if (ty_begin < 0 || ty_end > nty || ty_begin > ty_end) return PF_ERR_ARG;
  const int n_tiles = (ty_end - ty_begin) * ntx;
  if (n_tiles == 0) return PF_OK;
  BwdArgs a;
  a.recg = (const RecG*)((const char*)rec + sizeof(RecF) * (size_t)n);
  a.tex = tex;
  a.quad = (const float4*)quad;
  a.texels = texels;
  a.bin_off = bin_off;
  a.bin_idx = bin_idx;
  a.status = status;
  a.ent = (const SavedEnt*)saved;
  a.ent_n = ent_n;
  a.d4 = (const float4*)d4;
  a.bg0 = (float)bg_r;
  a.bg1 = (float)bg_g;
  a.bg2 = (float)bg_b;
  a.bg4 = (const float4*)bg4;
  a.mu_blend = (float)mu_blend;
  a.W = W;
  a.H = H;
  a.ntx = ntx;
  a.ty_begin = ty_begin;
  a.grads = grads;
  a.part = part;
  a.n_part = n_tiles * kWarpsPerTile;
  a.sums = sums;
  cudaStream_t st = (cudaStream_t)stream;
  if (mu_blend > 0.0)
    k_backward<true><<<n_tiles, kTilePix, 0, st>>>(a);
  else
    k_backward<false><<<n_tiles, kTilePix, 0, st>>>(a);
  return (int)cudaGetLastError();
}
