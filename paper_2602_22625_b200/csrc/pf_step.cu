// K34: the fit step's render -> loss -> backward as ONE persistent kernel.
//
// Reference: the loop body of run_loop (pkg/src/primfit/fit.py:486-492):
//   out, saved = render_forward(scene, bins, bg, save=True)   raster.py:290-363
//   value, dI, dA = evaluate_loss(loss_spec, out.color, out.alpha)  fit.py:112-151
//   grads = backward(scene, saved, dI, dA)                    grad.py:134-187
// Both losses the fit uses (MSE, spatial) are pixel-local: dL/dI and dL/dA of
// a pixel depend only on that pixel's colour and alpha.  So the thread that
// composites a pixel already holds everything its backward needs, and the
// saved contribution lists never leave the SM.
//
// Layout per CTA (persistent, one per SM; 3 warp groups of 1 producer + 8
// consumer warps; tiles from a longest-first ticket stream, see pf_bin's classes):
//   shared  the zero-padded alpha atlas (float64 when it fits next to the groups,
//           else float32, else read from the global fp32 plane through L1),
//           per group a 2-slot ring of stage buffers -- ST (32 or 64) step +
//           cull records (RecS 224 B + RecC 32 B per list entry) and the tile's
//           target (+ background) rows, all by TMA bulk copies under mbarriers --
//           and a 5-deep per-pixel contribution stack (deeper entries spill to
//           HBM at a slot unique to (tile entry, pixel)).
//   forward  per consumer warp (8x4 pixels): lane-parallel fp32 footprint cull of
//           32 list entries, then per surviving entry the centred affine float64
//           texel map (2 DFMA per axis; the reference's exact op order re-runs
//           only inside a guard band around the box edges / the eps threshold),
//           4 shared taps, float64 bilinear and eps test -- identical decisions
//           to _kernels.py:183-255 -- fp32 compositing (T, colour, alpha as
//           sum T a) and a 20-byte stack push (list position, incoming T, m,
//           dm/dU, dm/dV).
//   loss     pixel-local loss, dL/dI, dL/dA in registers (MSE in fp32); per-warp
//           partial sums written at a fixed slot (folded in fixed order by the
//           Adam launch, so the loss value is deterministic).
//   backward back-to-front walk over the stack (list position picked with
//           __reduce_max_sync), records from shared memory, template coordinates
//           u, v from the float64 affine map; warp transpose-butterfly reduction
//           and float64 RED atomics into grads.
// mu_blend > 0 (colour from the texture) keeps the two-kernel path.
//
// Slot mode (template SLOT, the fit loop): the tile lists come from K1's slot
// scatter instead of pf_bin; a prologue run by every warp z-sorts each tile's
// list (warp bitonic sorts in registers; long / overflowed lists through a
// gather + rank sort), builds the longest-first classes, gives each producer a
// CTA-local first tile, and arrives on a grid barrier that the producers wait
// on only before their first global ticket.  No fence instruction anywhere in
// this file's kernel: a fence makes ptxas emit the gradient REDs as returning
// ATOMs (+10 %); ordering uses acquire / release atomics instead.
// LOSS == PF_LOSS_EXTERN: dL/dI, dL/dA per pixel are staged in place of the
// target (the autograd Function's backward; forward recomputed on chip).
#include <cstdlib>
#include <type_traits>

#include "../../include/primfit_b200.h"
#include "pf_bins.cuh"
#include "pf_common.cuh"

namespace pf {

namespace {

constexpr int kCW = kTilePix / 32;                      // consumer warps per group (one tile)
// list entries staged per tile: ST = 32, or 64 for long-list scenes (template
// parameter of k_step; pf_fit_step's `stage` hint picks it)
#ifndef PF_NBUF
#define PF_NBUF 2
#endif
constexpr int kNBuf = PF_NBUF;                          // stage buffers per group (ring)
constexpr int kSlotArena = 128;  // spill entries per group for slot-mode in-place lists (L <= 128)
#ifndef PF_KS
#define PF_KS 5
#endif
#ifndef PF_F32_LERP
// fp32 bilinear alpha / eps decision / dm-dU, dm-dV in the fit step with fp32
// atlas taps (the float64 chain only inside the guard bands); measured +1.4 % at
// c3 with the fp32 shared atlas, +4 % at c5 (global atlas) over the float64 path
// with the fp64 shared atlas.  0 restores the float64 path (A/B).
#define PF_F32_LERP 1
#endif
constexpr int kKS = PF_KS;                              // contribution-stack depth in smem
constexpr uint32_t kEntBytes = sizeof(RecS) + sizeof(RecC);
// CTA shape for G groups: warps [0, 8G) consume (group = warp / 8), warps
// [8G, 9G) produce, padded to whole warpgroups so the producers' warpgroup can
// hand registers to the consumers' (setmaxnreg)
__host__ __device__ constexpr int step_warps(int G) { return (9 * G + 3) / 4 * 4; }
__host__ __device__ constexpr int step_threads(int G) { return 32 * step_warps(G); }
// registers per thread: launch budget, producer warpgroup after dec, consumers after inc
__host__ __device__ constexpr int step_regs(int G) { return (65536 / step_threads(G)) / 8 * 8; }
// (the pool setmaxnreg.inc draws from is what the launch allocated)
constexpr int kProdRegs = 24;
__host__ __device__ constexpr int step_cons_regs(int G) {
  return ((step_regs(G) * step_threads(G) - 32 * (step_warps(G) - 8 * G) * kProdRegs) /
          (256 * G)) / 8 * 8;
}
static_assert(step_cons_regs(3) == 80 && step_cons_regs(2) == 112, "register split");
// one stage buffer: ST RecS + ST RecC + the tile's target (+ background) pixels
__host__ __device__ constexpr size_t buf_rec_bytes(int st) { return (size_t)st * kEntBytes; }
constexpr size_t kBufPix = (size_t)kTilePix * sizeof(float4);
constexpr size_t kStackLevel = (size_t)kTilePix * (sizeof(float4) + sizeof(float));
__host__ __device__ constexpr size_t buf_bytes(bool bg, int st) {
  return buf_rec_bytes(st) + kBufPix * (bg ? 2 : 1);
}
// per group: kNBuf stage buffers + a kKS-deep contribution stack per consumer thread
__host__ __device__ constexpr size_t group_bytes(bool bg, int st) {
  return kNBuf * buf_bytes(bg, st) + kKS * kStackLevel;
}

struct StepArgs {
  const RecF* recf;
  const RecS* recs;
  const RecC* recc;
  const double* tex;
  const float* apad;     // zero-padded fp32 alpha plane (global copy)
  const double* apad64;  // the same plane in float64 (shared-memory copy source)
  int pad_texels;
  int texels;
  const int32_t* bin_off;
  const int32_t* bin_idx;
  const int32_t* status;
  int W, H, ntx, ty_begin, n_tiles;
  double eps_skip;
  double eps_band;       // eps re-check band (see warp_tile)
  float eps_f, eps_band_f;  // the same for the fp32 bilinear path (PF_F32_LERP)
  float k2_3P;           // (float)(2 / (3 P)): fp32 MSE gradient scale
  double bg0, bg1, bg2;
  float bgf0, bgf1, bgf2;  // the same as float (backward)
  const float4* bg4;
  float4* img4;          // optional (r, g, b, alpha)
  const float4* tgt4;
  double alpha_w, w_mse, w_gray, inv_3P, inv_P;
  double* part;          // [n_tiles * 8][3] per-warp loss partials
  float4* spill;         // [slot][2] for stack depth >= kKS
  double* grads;
  unsigned* ctr;         // [2]: tile ticket, finished producers (self-resetting)
  unsigned csleep, psleep;  // back-off (ns) of consumer / producer barrier waits
  const int32_t* classes;  // pf_bin's tile classes (counts + lists) or NULL: tile = ticket
  int32_t* classes_rw;
  int32_t* tile_cost;      // [n_tiles] measured work of each tile (next step's classes)
  unsigned long long* prof;  // diagnostics (PF_STEP_PROF=1): [warp slot][6], else NULL
  unsigned long long* tl;    // diagnostics timeline or NULL
  // slot mode (sb.cnt != NULL): the tile lists are K1's slot scatter, sorted here
  // by the producers (see SlotBins); no pf_bin launch precedes this kernel
  SlotBins sb;
  const int4* rect;      // K1's band-clipped rects per z rank (dirty-step validation)
  uint32_t* done;        // Adam iteration counter words (advanced here in slot mode)
  int32_t* status_rw;    // [2] published K, error flag (slot mode)
};

// Warp bitonic sort, ascending, of 32 keys (k0 at element lane) or 64 (k1 at
// element lane + 32): the producer's per-tile list sort in slot mode.
__device__ __forceinline__ uint32_t bitonic_xchg(uint32_t v, int e, int kk, int j) {
  const uint32_t p = __shfl_xor_sync(kFull, v, j);
  return (((e & kk) == 0) == ((e & j) == 0)) ? min(v, p) : max(v, p);
}
__device__ __forceinline__ void sort_keys(uint32_t& k0, uint32_t& k1, bool two) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int kk = 2; kk <= 32; kk <<= 1) {
#pragma unroll
    for (int j = kk >> 1; j > 0; j >>= 1) {
      k0 = bitonic_xchg(k0, lane, kk, j);
      if (two) k1 = bitonic_xchg(k1, lane + 32, kk, j);
    }
  }
  if (two) {
    const uint32_t lo = min(k0, k1), hi = max(k0, k1);
    k0 = lo;
    k1 = hi;
#pragma unroll
    for (int j = 16; j > 0; j >>= 1) {
      k0 = bitonic_xchg(k0, lane, 64, j);
      k1 = bitonic_xchg(k1, lane + 32, 64, j);
    }
  }
}

// 128 keys, four per lane (element lane + 32 r): the prologue's medium path
__device__ __forceinline__ void sort_keys4(uint32_t (&k)[4]) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int kk = 2; kk <= 128; kk <<= 1) {
#pragma unroll
    for (int j = kk >> 1; j > 0; j >>= 1) {
      if (j >= 32) {
        const int rj = j >> 5;
#pragma unroll
        for (int r = 0; r < 4; ++r) {
          if ((r & rj) == 0) {  // (r, r | rj): same lane, elements 32 j apart
            const bool up = ((lane + 32 * r) & kk) == 0;
            const uint32_t x = k[r], y = k[r | rj];
            k[r] = up ? min(x, y) : max(x, y);
            k[r | rj] = up ? max(x, y) : min(x, y);
          }
        }
      } else {
#pragma unroll
        for (int r = 0; r < 4; ++r) k[r] = bitonic_xchg(k[r], lane + 32 * r, kk, j);
      }
    }
  }
}

__device__ __forceinline__ unsigned atom_add_acq_rel(unsigned* p, unsigned v) {
  unsigned old;
  asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
  return old;
}

__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

// ---- mbarrier / bulk-copy primitives (PTX)
__device__ __forceinline__ uint32_t su32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void cp_async4(void* smem, const void* gmem) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(su32(smem)), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() {
  asm volatile("cp.async.wait_all;" ::: "memory");
}

__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(b)) : "memory");
}
__device__ __forceinline__ void mbar_arrive_tx(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(b)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ bool mbar_try(uint64_t* b, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n .reg .pred p;\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
      " selp.u32 %0, 1, 0, p;\n}"
      : "=r"(ok)
      : "r"(su32(b)), "r"(parity)
      : "memory");
  return ok != 0;
}
#ifdef PF_SUSPEND_WAIT  // (A/B variant: measured equal to the nanosleep back-off)
// try_wait with a suspend-time hint: the warp is parked by the hardware until
// the phase completes (or the hint elapses), no polling loop in the issue slots
__device__ __forceinline__ bool mbar_try_suspend(uint64_t* b, uint32_t parity, uint32_t ns) {
  uint32_t ok;
  asm volatile(
      "{\n .reg .pred p;\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n"
      " selp.u32 %0, 1, 0, p;\n}"
      : "=r"(ok)
      : "r"(su32(b)), "r"(parity), "r"(ns)
      : "memory");
  return ok != 0;
}
#endif
// wait with an explicit back-off (the waiting warp leaves the issue slots alone)
__device__ __forceinline__ void mbar_wait_sleep(uint64_t* b, uint32_t parity, unsigned ns) {
#ifdef PF_SUSPEND_WAIT
  (void)ns;
  while (!mbar_try_suspend(b, parity, PF_SUSPEND_WAIT)) {
  }
#else
  while (!mbar_try(b, parity)) __nanosleep(ns);
#endif
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          su32(dst)),
      "l"(src), "r"(bytes), "r"(su32(bar))
      : "memory");
}

__device__ __forceinline__ bool cull_touch(const RecC& rc, float cx, float cy) {
  const float dx = cx - rc.px, dy = cy - rc.py;
  const float uc = rc.au * dx + rc.bu * dy;
  const float vc = rc.av * dy - rc.bv * dx;
  const bool out_u = fabsf(uc) > 1.0f + rc.eu + 1e-5f * fabsf(uc);
  const bool out_v = fabsf(vc) > 1.0f + rc.ev + 1e-5f * fabsf(vc);
  return !(out_u || out_v);
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

// fp32 -> fp64 on the integer ALU for a non-negative finite float (alpha taps
// are in [0, 1]); denormals flush to 0.  Keeps F2F off the (quarter-rate)
// conversion pipe, which bounds this kernel otherwise.
__device__ __forceinline__ double f32_to_f64_alu(uint32_t b) {
  const uint32_t hi = (b >> 3) + 0x38000000u, lo = b << 29;
  return (b & 0x7f800000u) ? __hiloint2double((int)hi, (int)lo) : 0.0;
}

// (the float64 and fp32 accessors are each unused in one PF_F32_LERP variant)
#pragma nv_diag_suppress 177
// Padded alpha atlas access, float64 result: shared fp64 copy (LDS.64),
// shared fp32 copy, or the global fp32 plane.
struct AtlasS64 {
  uint32_t base;
  __device__ __forceinline__ double operator()(int i) const {
    double v;
    asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(base + 8u * (uint32_t)i));
    return v;
  }
  __device__ __forceinline__ float f(int i) const { return (float)(*this)(i); }
};
struct AtlasS32 {
  uint32_t base;
  __device__ __forceinline__ double operator()(int i) const {
    uint32_t v;
    asm volatile("ld.shared.b32 %0, [%1];" : "=r"(v) : "r"(base + 4u * (uint32_t)i));
    return f32_to_f64_alu(v);
  }
  __device__ __forceinline__ float f(int i) const {
    uint32_t v;
    asm volatile("ld.shared.b32 %0, [%1];" : "=r"(v) : "r"(base + 4u * (uint32_t)i));
    return __uint_as_float(v);
  }
};
struct AtlasG32 {
  const uint32_t* p;
  __device__ __forceinline__ double operator()(int i) const { return f32_to_f64_alu(__ldg(p + i)); }
  __device__ __forceinline__ float f(int i) const { return __uint_as_float(__ldg(p + i)); }
};

// floor(U) and U - floor(U) for 0 <= U < 2^31 with two DADDs (round-down add of
// 1.5 * 2^52 leaves floor(U) in the low mantissa bits) -- no conversion pipe.
__device__ __forceinline__ void cell_of(double U, int& u0, double& wu) {
  constexpr double kMagic = 6755399441055744.0;
  const double t = __dadd_rd(U, kMagic);
  u0 = __double2loint(t);
  wu = U - (t - kMagic);
}

// Record access for one tile: staged (shared) entries, plus -- for lists longer
// than ST -- the remaining entries straight from HBM/L2.
struct StagedRecs {
  const RecS* s;
  const RecC* c;
  __device__ __forceinline__ const RecS& rec(int j) const { return s[j]; }
  __device__ __forceinline__ const RecC& cull(int j) const { return c[j]; }
};
template <int ST>
struct MixedRecs {
  const RecS* s;
  const RecC* c;
  const RecS* gs;
  const RecC* gc;
  const int32_t* idx;  // bin_idx + b0
  __device__ __forceinline__ const RecS& rec(int j) const {
    return j < ST ? s[j] : gs[__ldcg(idx + j)];
  }
  __device__ __forceinline__ const RecC& cull(int j) const {
    return j < ST ? c[j] : gc[__ldcg(idx + j)];
  }
};

// One consumer warp's share (8x4 pixels) of one tile: forward, loss, backward.
template <int LOSS, typename RECS, typename ATL>
__device__ __forceinline__ void warp_tile(const StepArgs& a, const RECS& R, const ATL& atl,
                                          const float4* tgs, const float4* bgs, float4* stA,
                                          float* stB, int tile, int b0, int L, int txy, int w) {
  const int lane = threadIdx.x & 31;
  const int ct = w * 32 + lane;  // consumer thread (pixel) index within the tile
  const int tx = txy & 0xffff, ty = txy >> 16;
  const int wx = (w & 1) * kWarpW, wy = (w >> 1) * kWarpH;
  const int x = tx * kTile + wx + (lane & (kWarpW - 1));
  const int y = ty * kTile + wy + (lane / kWarpW);
  const float cx = (float)(tx * kTile + wx) + 0.5f * (kWarpW - 1);
  const float cy = (float)(ty * kTile + wy) + 0.5f * (kWarpH - 1);
  const bool valid = x < a.W && y < a.H;
  const double xx = (double)x, yy = (double)y;
  const size_t pix = valid ? (size_t)y * a.W + x : 0;
  const size_t slot0 = (size_t)b0 * kTilePix + ct;
  const int tp_ = (wy + lane / kWarpW) * kTile + wx + (lane & (kWarpW - 1));  // pixel in tile
  const double* plane_a = a.tex + 3 * (size_t)a.texels;

  // ---- forward (k_forward semantics, _kernels.py:183-255)
  // compositing state in fp32: ~1e-7 relative on the image against the 1e-5 bar
  // (every decision was taken in float64 above it)
  // alpha = 1 - T is accumulated as sum T*a (all terms positive: relative
  // accuracy also where T is close to 1)
  float T = 1.0f, Aacc = 0.0f, C0 = 0.0f, C1 = 0.0f, C2 = 0.0f;
  int ns = 0;
  int work = 2;  // this rect's work units (candidates + 2 x backward steps): tile cost
  for (int sub = 0; sub < L; sub += 32) {
    const int jl = sub + lane;
    const bool cand = jl < L && cull_touch(R.cull(jl), cx, cy);
    unsigned mask = __ballot_sync(kFull, cand);
    work += __popc(mask);
    if (!valid) mask = 0u;  // divergent only in a partial last tile row / column
    while (mask) {
      const int bit = __ffs(mask) - 1;
      mask &= mask - 1;
      const int j = sub + bit;
      const RecS& r = R.rec(j);
      // centred texel coordinates: |U - hw| against hw -/+ delta decides
      // inside / outside / guard band (exact reference chain) per axis
      const double Uc = fma(r.au, xx, fma(r.bu, yy, r.cu));
      const double Vc = fma(r.av, xx, fma(r.bv, yy, r.cv));
      const double aU = fabs(Uc), aV = fabs(Vc);
      if (aU > r.out_u || aV > r.out_v) continue;
      const bool exact = !(aU < r.in_u && aV < r.in_v);
      double U = Uc + r.hwd, V = Vc + r.hhd;
      if (exact && !texel_coords(a.recf[r.gidx], xx, yy, U, V)) continue;
      int u0, v0;
      double wu, wv;
      cell_of(U, u0, wu);
      cell_of(V, v0, wv);
      int tp = r.pbase + v0 * r.wp + u0;
#if PF_F32_LERP
      // the common case in fp32: bilinear alpha from fp32 taps, eps decision
      // outside a 1e-6 band around eps (>> the fp32 error), dm/dU, dm/dV; the
      // cell and weights come from the float64 U, V (exact cell choice)
      float wuf = (float)wu, wvf = (float)wv;
      float f00 = atl.f(tp), f01 = atl.f(tp + 1), f10 = atl.f(tp + r.wp), f11 = atl.f(tp + r.wp + 1);
      const float lf0 = fmaf(wuf, f01 - f00, f00), lf1 = fmaf(wuf, f11 - f10, f10);
      float mf = fmaf(wvf, lf1 - lf0, lf0);
      if (exact || fabsf(mf - a.eps_f) <= a.eps_band_f) {
        // rare: the reference's exact chain for the decision and the value
        const RecF& f = a.recf[r.gidx];
        if (!exact) (void)texel_coords(f, xx, yy, U, V);
        const Cell c = make_cell(U, V);
        const double m = bilinear(plane_a, f.base, f.wt, f.ht, c);
        if (m < a.eps_skip) continue;
        mf = (float)m;
        wuf = (float)c.wu;
        wvf = (float)c.wv;
        tp = r.pbase + c.v0 * r.wp + c.u0;
        f00 = atl.f(tp);
        f01 = atl.f(tp + 1);
        f10 = atl.f(tp + r.wp);
        f11 = atl.f(tp + r.wp + 1);
      } else if (mf < a.eps_f) {
        continue;
      }
      const float gUf = fmaf(wvf, (f11 - f10) - (f01 - f00), f01 - f00);
      const float gVf = fmaf(wuf, (f11 - f01) - (f10 - f00), f10 - f00);
      const float4 ea = make_float4(__int_as_float(j), T, mf, gUf);
      const float eb = gVf;
#else
      double t00 = atl(tp), t01 = atl(tp + 1), t10 = atl(tp + r.wp), t11 = atl(tp + r.wp + 1);
      const double l0 = fma(wu, t01 - t00, t00), l1 = fma(wu, t11 - t10, t10);
      double m = fma(wv, l1 - l0, l0);
      if (exact || fabs(m - a.eps_skip) <= a.eps_band) {
        // rare: the reference's exact chain for the decision and the value
        const RecF& f = a.recf[r.gidx];
        if (!exact) (void)texel_coords(f, xx, yy, U, V);
        const Cell c = make_cell(U, V);
        m = bilinear(plane_a, f.base, f.wt, f.ht, c);
        wu = c.wu;
        wv = c.wv;
        tp = r.pbase + c.v0 * r.wp + c.u0;
        t00 = atl(tp);
        t01 = atl(tp + 1);
        t10 = atl(tp + r.wp);
        t11 = atl(tp + r.wp + 1);
      }
      if (m < a.eps_skip) continue;
      // dm/dU, dm/dV (_kernels.py:61-73) -- alpha channel only (Appendix A.3)
      const double gU = fma(wv, (t11 - t10) - (t01 - t00), t01 - t00);
      const double gV = fma(wu, (t11 - t01) - (t10 - t00), t10 - t00);
      const float mf = (float)m;
      const float4 ea = make_float4(__int_as_float(j), T, mf, (float)gU);
      const float eb = (float)gV;
#endif
      if (LOSS == PF_LOSS_RENDER) {
        // (forward only: no contribution stack)
      } else if (ns < kKS) {
        stA[ns * kTilePix + ct] = ea;
        stB[ns * kTilePix + ct] = eb;
      } else {
        float4* sp = a.spill + 2 * (slot0 + (size_t)(ns - kKS) * kTilePix);
        sp[0] = ea;
        sp[1] = make_float4(eb, 0.f, 0.f, 0.f);
      }
      ++ns;
      const float aa = r.saf * mf;
      const float Ta = T * aa;
      C0 += Ta * r.c0f;
      C1 += Ta * r.c1f;
      C2 += Ta * r.c2f;
      Aacc += Ta;
      T *= 1.0f - aa;
    }
  }

  // ---- loss (fit.py:112-151), pixel-local
  const float4 bgp = bgs ? bgs[tp_] : make_float4(0.f, 0.f, 0.f, 0.f);
  const float g0 = a.bg4 ? bgp.x : a.bgf0;
  const float g1 = a.bg4 ? bgp.y : a.bgf1;
  const float g2 = a.bg4 ? bgp.z : a.bgf2;
  if (LOSS == PF_LOSS_RENDER) {
    // render only (the autograd forward): the image, no loss, no backward
    if (valid) a.img4[pix] = make_float4(fmaf(T, g0, C0), fmaf(T, g1, C1), fmaf(T, g2, C2), Aacc);
    if (a.tile_cost && lane == 0) atomicMax(a.tile_cost + tile, work);
    return;
  }
  const float4 tg = tgs[tp_];
  float dI0 = 0.f, dI1 = 0.f, dI2 = 0.f, dA = 0.f;
  float l0 = 0.f, l1 = 0.f, l2 = 0.f;
#ifndef PF_LOSS32
#define PF_LOSS32 1
#endif
  if (LOSS == PF_LOSS_EXTERN) {
    // gradients from upstream (the autograd backward): the staged rows hold
    // (dL/dI r, g, b, dL/dA) per pixel; no loss here
    if (valid) {
      dI0 = tg.x;
      dI1 = tg.y;
      dI2 = tg.z;
      dA = tg.w;
    }
  } else if (valid && PF_LOSS32 && LOSS == PF_LOSS_MSE) {
    // MSE in fp32 end to end: the image is stored as fp32 and the per-warp
    // partials are fp32 sums already; (I - t) to ~1 ulp of I (< 1e-7)
    const float I0 = fmaf(T, g0, C0), I1 = fmaf(T, g1, C1), I2 = fmaf(T, g2, C2);
    if (a.img4) a.img4[pix] = make_float4(I0, I1, I2, Aacc);
    const float r0 = I0 - tg.x, r1 = I1 - tg.y, r2 = I2 - tg.z;
    l0 = fmaf(r0, r0, fmaf(r1, r1, r2 * r2));
    l1 = l0;
    const float k = a.k2_3P;
    dI0 = k * r0;
    dI1 = k * r1;
    dI2 = k * r2;
  } else if (valid) {
    const double I0 = (double)C0 + (double)T * (a.bg4 ? (double)bgp.x : a.bg0);
    const double I1 = (double)C1 + (double)T * (a.bg4 ? (double)bgp.y : a.bg1);
    const double I2 = (double)C2 + (double)T * (a.bg4 ? (double)bgp.z : a.bg2);
    const double Ia = (double)Aacc;
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
    } else if (LOSS == PF_LOSS_COMBINED) {
      // mse_w * loss_mse + gray_l1_w * loss_grayscale_l1 (fit.py:112-125, 162-168)
      const double d = r0 * 0.299 + r1 * 0.587 + r2 * 0.114;
      l1 = (float)fabs(d);
      const double kg = a.w_gray * (d > 0.0 ? 1.0 : (d < 0.0 ? -1.0 : 0.0)) * a.inv_P;
      const double km = a.w_mse * k;
      dI0 = (float)(km * r0 + kg * 0.299);
      dI1 = (float)(km * r1 + kg * 0.587);
      dI2 = (float)(km * r2 + kg * 0.114);
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
  if (LOSS != PF_LOSS_EXTERN) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    l0 += __shfl_xor_sync(kFull, l0, o);
    if (LOSS != PF_LOSS_MSE) {  // MSE: l1 == l0, l2 == 0
      l1 += __shfl_xor_sync(kFull, l1, o);
      l2 += __shfl_xor_sync(kFull, l2, o);
    }
  }
  }
  if (LOSS == PF_LOSS_MSE) l1 = l0;
  if (LOSS != PF_LOSS_EXTERN && lane == 0) {
    double* pp = a.part + ((size_t)tile * kCW + w) * 3;
    pp[0] = l0;
    pp[1] = l1;
    pp[2] = l2;
  }

  // ---- backward (_kernels.py:258-363), back to front over the stack
  float S0 = 0.f, S1 = 0.f, S2 = 0.f, B = 1.f;
  int k = ns - 1;
  float4 ea = make_float4(0.f, 0.f, 0.f, 0.f);
  float eb = 0.f;
  unsigned key = 0;
  auto fetch = [&](int d) {
    if (d < kKS) {
      ea = stA[d * kTilePix + ct];
      eb = stB[d * kTilePix + ct];
    } else {
      const float4* sp = a.spill + 2 * (slot0 + (size_t)(d - kKS) * kTilePix);
      ea = sp[0];
      eb = sp[1].x;
    }
    key = (unsigned)__float_as_int(ea.x) + 1u;
  };
  if (k >= 0) fetch(k);
  while (true) {
    const unsigned jm = __reduce_max_sync(kFull, key);
    if (jm == 0u) break;
    work += 2;
    const bool act = key == jm;
    const unsigned ball = __ballot_sync(kFull, act);
    const RecS& r = R.rec((int)jm - 1);
    float g[8];
#pragma unroll
    for (int c = 0; c < 8; ++c) g[c] = 0.0f;
    if (act) {
      const float Tc = ea.y, m = ea.z, gU = ea.w, gV = eb;
      if (--k >= 0) fetch(k); else key = 0;
      // normalised template coordinates u = (U - hw) / hw, v = (V - hh) / hh from
      // the centred affine map in float64 (an fp32 dx = x - px loses ~ulp(x) / s:
      // 1e-3 of the rotation gradient on a 4K canvas)
      const double Uc = fma(r.au, xx, fma(r.bu, yy, r.cu));
      const double Vc = fma(r.av, xx, fma(r.bv, yy, r.cv));
      const float u = (float)Uc * r.inv_hw;
      const float v = (float)Vc * r.inv_hh;
      const float aa = r.saf * m;
      const float gg = dI0 * (r.c0f - S0 - g0 * B) + dI1 * (r.c1f - S1 - g1 * B) +
                       dI2 * (r.c2f - S2 - g2 * B) + dA * B;
      const float dalpha = Tc * gg;
      g[4] = dalpha * r.sd * m;
      {
        // colour logits (the fused path runs with mu_blend == 0: 1 - mu = 1)
        const float wc = Tc * aa;
        g[5] = dI0 * wc * r.cd0;
        g[6] = dI1 * wc * r.cd1;
        g[7] = dI2 * wc * r.cd2;
      }
      const float dm = dalpha * r.saf;
      const float mu_u = gU * r.hw, mu_v = gV * r.hh;
      g[0] = dm * (mu_u * r.gxu + mu_v * r.gxv);
      g[1] = dm * (mu_u * r.gyu + mu_v * r.gyv);
      g[2] = dm * (mu_u * (-u * r.inv_s) + mu_v * (-v * r.inv_s));
      g[3] = dm * (mu_u * (v * r.q) + mu_v * (-u * r.inv_q));
      const float om = 1.0f - aa;
      S0 = aa * r.c0f + om * S0;
      S1 = aa * r.c1f + om * S1;
      S2 = aa * r.c2f + om * S2;
      B *= om;
    }
    double* gp = a.grads + (size_t)r.gidx * 8;
#ifndef PF_DIRECT_MAX
#define PF_DIRECT_MAX 2  // entries with at most this many lanes skip the warp reduction
#endif
    if (__popc(ball) <= PF_DIRECT_MAX) {
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
  // the tile's cost for the next step's longest-first schedule: max over its rects
  if (a.tile_cost && lane == 0) atomicMax(a.tile_cost + tile, work);
}

}  // namespace

// Slot-mode prologue of pf_fit_step (every warp of every CTA, before the role
// split): each tile's slot list -- K1's arrival-order scatter, see SlotBins --
// becomes the z-sorted list of bin_tiles (raster.py:227-265), written back in
// place (list base tile * m) or, for long / overflowed lists, into the pool
// (base n_tiles * m + pool offset); a dirty step (host edits re-scattered by
// pf_preprocess_sync) first drops entries whose primitive no longer covers the
// tile and duplicates.  The tile then joins its cost class (cost measured by the
// previous step, else its length) with the CSR-shaped entry (tile, list base,
// L, tx | ty << 16) the producers read, and its count is zeroed for the next
// K1.  A grid barrier (all CTAs are resident: one per SM) ends the phase.
constexpr int kSortRound = 1024;  // tiles per CTA and round (scratch: 20 B each)
constexpr bool kDiag = PF_DIAG != 0;  // (pf_common.cuh: 0 in the product library)
#ifndef PF_PROLOGUE_MARKS
#define PF_PROLOGUE_MARKS 1  // (diagnostics, PF_STEP_PROF only: phase times of the prologue)
#endif
template <int G>
__device__ __forceinline__ void slot_prologue(const StepArgs& a, unsigned char* scratch,
                                              int4* first) {
  const SlotBins& sb = a.sb;
  unsigned long long* const prof_ = kDiag ? a.prof : nullptr;
  unsigned long long* const tl_ = kDiag ? a.tl : nullptr;
  __shared__ int s_ccnt[kTileClasses], s_cbase[kTileClasses];
  __shared__ unsigned s_k;
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5, nwarps = blockDim.x >> 5;
  const unsigned lt_mask = (1u << lane) - 1u;
  const bool dirty = __ldcg(sb.ctl + kSlotDirty) != 0u;
  const int nslot = sb.n_tiles * sb.m;
  int4* ent = reinterpret_cast<int4*>(scratch);
  int* cls = reinterpret_cast<int*>(ent + kSortRound);
  int32_t* cost = a.classes_rw + tile_cost_offset(a.n_tiles);
  int4* clists = reinterpret_cast<int4*>(a.classes_rw + kTileClasses);
  const int per = (a.n_tiles + gridDim.x - 1) / gridDim.x;
  const int c0 = min(a.n_tiles, (int)blockIdx.x * per), c1 = min(a.n_tiles, c0 + per);
  unsigned kacc = 0;
  if (t == 0) s_k = 0u;
  auto covers = [&](uint32_t z, int txy) {
    if (z == ~0u) return false;
    const int4 r = __ldcg(a.rect + z);
    const int tx = txy & 0xffff, ty = txy >> 16;
    return r.y <= ty && ty <= r.w && (r.x & 0xffff) <= tx && tx <= (r.x >> 16);
  };
  for (int r0 = c0; r0 < c1; r0 += kSortRound) {
    const int nr = min(kSortRound, c1 - r0);
    if (t < kTileClasses) s_ccnt[t] = 0;
    __syncthreads();
    // a warp's tiles in batches of kB: every batch's slot rows land in shared
    // memory by async copies (and the counts / costs in lanes 0..kB-1) before the
    // first sort; the per-tile processing is a rolled loop (one copy of the sort
    // code: this phase runs once per launch, instruction-cache misses dominate
    // an unrolled version)
#ifndef PF_SORT_BATCH
#define PF_SORT_BATCH 4
#endif
    constexpr int kB = PF_SORT_BATCH;
    uint32_t* kbuf = reinterpret_cast<uint32_t*>(cls + kSortRound) + warp * (kB * 64);
    for (int ib = warp; ib < nr; ib += nwarps * kB) {
      int qraw = 0, qw = 0;
      if (lane < kB && ib + lane * nwarps < nr) {
        qraw = __ldcg(sb.cnt + r0 + ib + lane * nwarps);
        qw = __ldcg(cost + r0 + ib + lane * nwarps);
      }
#pragma unroll
      for (int q = 0; q < kB; ++q) {
        const int i = ib + q * nwarps;
        if (i < nr) {
          const uint32_t* sl = sb.slot + (size_t)(r0 + i) * sb.m;
          if (lane < sb.m) cp_async4(kbuf + q * 64 + lane, sl + lane);
          if (lane + 32 < sb.m) cp_async4(kbuf + q * 64 + 32 + lane, sl + 32 + lane);
        }
      }
      cp_async_wait_all();
      __syncwarp();
      if (PF_PROLOGUE_MARKS && prof_ && t == 0 && ib == warp && blockIdx.x < 256)
        prof_[6 * 148 * 32 + 65536 * 8 + 512 + 4 * blockIdx.x + 0] = gtimer();
#pragma unroll 1
      for (int q = 0; q < kB; ++q) {
        const int i = ib + q * nwarps;
        if (i >= nr) break;  // (warp-uniform)
        const int tile = r0 + i;
        const int txy = (tile % a.ntx) | ((a.ty_begin + tile / a.ntx) << 16);
        uint32_t* sl = sb.slot + (size_t)tile * sb.m;
        int raw = __shfl_sync(kFull, qraw, q);
        const int wq = __shfl_sync(kFull, qw, q);
        uint32_t k0 = lane < sb.m ? kbuf[q * 64 + lane] : ~0u;
        uint32_t k1 = lane + 32 < sb.m ? kbuf[q * 64 + 32 + lane] : ~0u;
        int L = 0, b0 = tile * sb.m;
        if (raw <= 64 && raw <= sb.m) {
          if (lane >= raw) k0 = ~0u;
          if (lane + 32 >= raw) k1 = ~0u;
          if (dirty) {
            if (!covers(k0, txy)) k0 = ~0u;
            if (!covers(k1, txy)) k1 = ~0u;
          }
#pragma unroll 1
          for (int pass = 0; pass < (dirty ? 2 : 1); ++pass) {
            sort_keys(k0, k1, raw > 32);
            if (pass == 0 && dirty) {
              // duplicates are adjacent after the sort: drop all but the first, re-sort
              const uint32_t p0 = __shfl_up_sync(kFull, k0, 1);
              const uint32_t l0 = __shfl_sync(kFull, k0, 31);
              const uint32_t q1 = __shfl_up_sync(kFull, k1, 1);
              const bool d0 = lane > 0 && k0 == p0;
              const bool d1 = lane == 0 ? k1 == l0 : k1 == q1;
              if (d0) k0 = ~0u;
              if (d1) k1 = ~0u;
            }
          }
          L = __popc(__ballot_sync(kFull, k0 != ~0u)) + __popc(__ballot_sync(kFull, k1 != ~0u));
          if (lane < L) sl[lane] = k0;
          if (lane + 32 < L) sl[lane + 32] = k1;
        } else if (raw <= 128 && raw <= sb.m && !dirty) {
          // medium path (c2-like long lists): 128 keys in registers, sorted in place
          uint32_t k4[4];
#pragma unroll
          for (int r = 0; r < 4; ++r) {
            const int e = lane + 32 * r;
            k4[r] = e < raw ? __ldcg(sl + e) : ~0u;
          }
          sort_keys4(k4);
          L = raw;
#pragma unroll
          for (int r = 0; r < 4; ++r)
            if (lane + 32 * r < L) sl[lane + 32 * r] = k4[r];
        } else {
          // general path (long or overflowed lists; rare): gather the slots and
          // the tile's overflow entries into scratch, keep valid first
          // occurrences, rank by z into the pool
          int gb = 0;
          if (lane == 0) gb = (int)atomicAdd(sb.ctl + kSlotGather, 2u * (uint32_t)raw);
          gb = __shfl_sync(kFull, gb, 0);
          if (gb + 2 * raw > sb.gat_cap) {
            if (lane == 0) sb.ctl[kSlotErr] = 1u;
            raw = 0;
          }
          uint32_t* g1 = sb.gat + gb;
          uint32_t* g2 = g1 + raw;
          const int n_in = min(raw, sb.m);
          for (int k = lane; k < n_in; k += 32) g1[k] = __ldcg(sl + k);
          int pos = n_in;
          if (raw > sb.m) {
            const int novf = min((int)__ldcg(sb.ctl + kSlotOvf), sb.ovf_cap);
            for (int o0 = 0; o0 < novf && pos < raw; o0 += 32) {
              const int o = o0 + lane;
              const int2 e = o < novf ? __ldcg(sb.ovf + o) : make_int2(-1, 0);
              const bool hit = e.x == tile;
              const unsigned hm = __ballot_sync(kFull, hit);
              const int at = pos + __popc(hm & lt_mask);
              if (hit && at < raw) g1[at] = (uint32_t)e.y;
              pos = min(raw, pos + __popc(hm));
            }
          }
          __syncwarp();
          for (int q0 = 0; q0 < pos; q0 += 32) {
            const int k = q0 + lane;
            const uint32_t key = k < pos ? __ldcg(g1 + k) : ~0u;
            bool keep = key != ~0u && (!dirty || covers(key, txy));
            if (dirty && keep)
              for (int j = 0; j < k; ++j)
                if (__ldcg(g1 + j) == key) {
                  keep = false;
                  break;
                }
            if (k < pos) g2[k] = keep ? key : ~0u;
            L += __popc(__ballot_sync(kFull, keep));
          }
          __syncwarp();
          int pb = 0;
          if (lane == 0) pb = (int)atomicAdd(sb.ctl + kSlotPool, (uint32_t)L);
          pb = __shfl_sync(kFull, pb, 0);
          if (pb + L > sb.pool_cap) {
            if (lane == 0) sb.ctl[kSlotErr] = 1u;
            L = 0;
          }
          for (int q0 = 0; q0 < pos && L > 0; q0 += 32) {
            const int k = q0 + lane;
            const uint32_t key = k < pos ? __ldcg(g2 + k) : ~0u;
            if (key != ~0u) {
              int rk = 0;
              for (int j = 0; j < pos; ++j) rk += __ldcg(g2 + j) < key;
              sb.pool[pb + rk] = key;
            }
          }
          b0 = nslot + pb;
        }
        if (lane == 0) {
          sb.cnt[tile] = 0;  // (read above by this lane) ready for the next K1
          cost[tile] = 0;
          const int4 e = make_int4(tile, b0, L, txy);
          ent[i] = e;
          if (r0 == c0 && i < G) {
            // the CTA's first G tiles are its producers' first tiles: they start
            // on CTA-local lists right away, while other CTAs still finish (no
            // grid barrier before the first copies); they stay out of the global
            // classes (choosing the heaviest G instead measured the same)
            first[i] = e;
            cls[i] = -1;
          } else {
            const int cl = tile_class(wq > 0 ? wq : L);
            cls[i] = cl | (atomicAdd(&s_ccnt[cl], 1) << 8);
          }
          kacc += (unsigned)L;
        }
      }
    }
    __syncthreads();
    if (PF_PROLOGUE_MARKS && prof_ && t == 0 && blockIdx.x < 256)
      prof_[6 * 148 * 32 + 65536 * 8 + 512 + 4 * blockIdx.x + 1] = gtimer();
    if (t < kTileClasses) s_cbase[t] = s_ccnt[t] ? atomicAdd(a.classes_rw + t, s_ccnt[t]) : 0;
    __syncthreads();
    for (int i = t; i < nr; i += blockDim.x) {
      if (cls[i] < 0) continue;
      const int cl = cls[i] & 0xff, rank = cls[i] >> 8;
      clists[(size_t)cl * a.n_tiles + s_cbase[cl] + rank] = ent[i];
    }
    __syncthreads();
  }
  if (PF_PROLOGUE_MARKS && prof_ && t == 0 && blockIdx.x < 256)
    prof_[6 * 148 * 32 + 65536 * 8 + 512 + 4 * blockIdx.x + 2] = gtimer();
  if (lane == 0 && kacc) atomicAdd(&s_k, kacc);
  tl_mark(tl_, 14, 1);
  __syncthreads();
  // arrive on the grid barrier: this CTA's lists and class entries are complete
  // (the producers wait for every CTA before their first global ticket)
  if (t == 0) {
    if (s_k) atomicAdd(sb.ctl + kSlotK, s_k);
    atom_add_acq_rel(a.ctr + 2, 1u);
  }
}

// Persistent, warp-specialised.  One CTA per SM; G groups of one producer warp
// and 8 consumer warps (one 8x4 pixel sub-tile each).  Warps [0, 8G) consume
// (group = warp / 8), warps [8G, 9G) produce, padded to whole warpgroups: the
// producer / padding warpgroup drops to 24 registers (setmaxnreg) so that the
// consumer warpgroups run at 80 (G = 3).
//   producer  takes a tile ticket, reads the tile's list, then (once the ring
//             slot is free) TMA bulk-copies the list's step + cull records and
//             the tile's target (+ background) rows into an nbuf-deep ring of
//             stage buffers (mbarrier full/empty handshake, expect_tx bytes).
//   consumers forward -> loss -> backward out of shared memory only; no
//             block-wide barrier after the prologue, so warps drift freely.
// The padded alpha atlas is loaded into shared memory once per CTA: float64
// (ATL == 2) when it fits, else float32 (ATL == 1); ATL == 0 reads the global
// fp32 plane.
template <int LOSS, int ATL, int G, bool BG, int ST, bool SLOT>
__global__ void __launch_bounds__(step_threads(G), 1) k_step(StepArgs a) {
  extern __shared__ __align__(128) unsigned char sm[];
  // diagnostics pointers (PF_STEP_PROF / PF_TIMELINE); a PF_DIAG=0 build drops them
  unsigned long long* const prof_ = kDiag ? a.prof : nullptr;
  unsigned long long* const tl_ = kDiag ? a.tl : nullptr;
  __shared__ __align__(8) uint64_t full[G][kNBuf], empty[G][kNBuf];
  __shared__ int4 hdr[G][kNBuf];

  tl_mark(tl_, 1, 0);
  const int t = threadIdx.x;
  const int lane = t & 31, warp = t >> 5;
  constexpr bool has_bg = BG;
  constexpr size_t gbytes = group_bytes(BG, ST), bbytes = buf_bytes(BG, ST);
  unsigned char* satl = sm + G * gbytes;
  using Atl = typename std::conditional<
      ATL == 2, AtlasS64, typename std::conditional<ATL == 1, AtlasS32, AtlasG32>::type>::type;
  Atl atl;
  if constexpr (ATL == 0) atl.p = reinterpret_cast<const uint32_t*>(a.apad);
  else atl.base = su32(satl);
  // the atlas arrives asynchronously (TMA bulk copy, atl_bar); consumers wait for
  // it before their first tile, so the copy overlaps the first tickets
  __shared__ __align__(8) uint64_t atl_bar;
  // slot mode: the atlas copy goes out after the prologue's list loads (they are
  // on the critical path, the atlas is needed only by the first tile; measured
  // -0.5 us to the grid barrier at c3)
#ifdef PF_ATLAS_EARLY
  constexpr bool atl_late = false;  // (A/B)
#else
  constexpr bool atl_late = SLOT;
#endif
  auto issue_atlas = [&]() {
    if (ATL != 0) {
      const uint32_t bytes = (uint32_t)a.pad_texels * (ATL == 2 ? 8u : 4u);
      const char* src = reinterpret_cast<const char*>(ATL == 2 ? (const void*)a.apad64
                                                               : (const void*)a.apad);
      mbar_arrive_tx(&atl_bar, bytes);
      // chunks of <= 32 KB, issued from a staggered start across CTAs
      constexpr uint32_t kChunk = 32768;
      const uint32_t nch = (bytes + kChunk - 1) / kChunk;
      for (uint32_t k = 0; k < nch; ++k) {
        const uint32_t q = (k + blockIdx.x) % nch;
        const uint32_t off = q * kChunk, len = min(kChunk, bytes - off);
        bulk_g2s(satl + off, src + off, len, &atl_bar);
      }
    } else {
      mbar_arrive(&atl_bar);
    }
  };
  if (t == 0) {
    mbar_init(&atl_bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    if (!atl_late) issue_atlas();
  }
  if (t < G * kNBuf) {
    mbar_init(&full[t / kNBuf][t % kNBuf], 1);
    mbar_init(&empty[t / kNBuf][t % kNBuf], kCW);
  }
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  pdl_wait();  // bins, classes and records of this step are complete from here on
  tl_mark(tl_, 1, 1);
  constexpr bool slot_mode = SLOT;  // (a template parameter: consumer registers)
  // (no fences in this kernel: any fence makes ptxas turn every gradient RED
  // into a returning ATOM -- 10 % of the kernel's time)
  __shared__ unsigned s_adv;
  if (slot_mode && blockIdx.x == 0 && t == 0) {
    // (no pf_bin in slot mode) the Adam step before this one is complete: advance
    // the iteration counter the next Adam launch reads before its own wait.
    // Returning atomics, their values consumed before the block barrier that
    // precedes this CTA's trigger: performed at L2 before the dependent launches.
    unsigned adv = 0u;
    if (atomicExch(a.done + 2, 0u) != 0u) adv = atomicAdd(a.done + 1, 1u) + 1u;
    s_adv = adv;
  }
  __syncthreads();
  // after the wait (so a dependent that starts early knows K2 -- and by induction
  // the previous Adam step -- has completed): the Adam kernel may start loading
  // its inputs that this kernel does not write
  pdl_trigger();
  if (slot_mode ? __ldcg(a.sb.ctl + kSlotErr) != 0u : a.status[1] != 0) {
    // bin overflow (grid-uniform): lists are not valid; leave clean counters
    if (blockIdx.x == 0 && a.classes && t < kTileClasses) a.classes_rw[t] = 0;
    if (slot_mode && blockIdx.x == 0 && t == 0) a.status_rw[1] = 1;
    return;
  }
  __shared__ int4 s_first[G];  // slot mode: each producer's CTA-local first tile
  if (SLOT && t < G) s_first[t] = make_int4(-1, 0, 0, 0);
  if constexpr (SLOT) {
    __syncthreads();
    const unsigned long long pro0 = prof_ ? gtimer() : 0;
    slot_prologue<G>(a, sm, s_first);
    if (prof_ && t == 0 && blockIdx.x < 256) {  // (diagnostics: prologue span per CTA)
      unsigned long long* pp = prof_ + 6 * 148 * 32 + 65536 * 8 + 2 * blockIdx.x;
      pp[0] = pro0;
      pp[1] = gtimer();
    }
    if (atl_late && t == 0) issue_atlas();
  }

  const bool consumer = warp < G * kCW;
  const int g = consumer ? warp / kCW : warp - G * kCW;
  const int wg = consumer ? warp % kCW : kCW;
  unsigned char* gs = sm + g * gbytes;
  float4* stA = reinterpret_cast<float4*>(gs + kNBuf * bbytes);
  float* stB = reinterpret_cast<float*>(stA + kKS * kTilePix);
  auto buf_rec = [&](int b) { return reinterpret_cast<RecS*>(gs + b * bbytes); };
  auto buf_cull = [&](int b) {
    return reinterpret_cast<RecC*>(gs + b * bbytes + ST * sizeof(RecS));
  };
  auto buf_tgt = [&](int b) {
    return reinterpret_cast<float4*>(gs + b * bbytes + buf_rec_bytes(ST));
  };
  auto buf_bg = [&](int b) {
    return reinterpret_cast<float4*>(gs + b * bbytes + buf_rec_bytes(ST) + kBufPix);
  };

  unsigned long long p_wait = 0, p_work = 0, p_n = 0, p_first = 0, p_t0 = prof_ ? gtimer() : 0;
  auto finish = [&]() {
    tl_mark(tl_, 1, 3);
    if (prof_ && lane == 0) {
      unsigned long long* o = prof_ + ((size_t)blockIdx.x * blockDim.x / 32 + warp) * 6;
      o[0] = p_wait;
      o[1] = p_work;
      o[2] = p_n;
      o[3] = p_t0;
      o[4] = gtimer();
      o[5] = (unsigned long long)(wg == kCW) | (p_first << 1);
    }
  };
  // Register hand-over (warpgroup-uniform: warps [8G, ...) are whole
  // warpgroups): the producer / padding warpgroup shrinks, the consumer
  // warpgroups grow.  The two roles never re-join, so each is allocated
  // against its own limit.
  if (!consumer) {
    asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(kProdRegs));
    if (g >= G) return;  // padding warp
    // ---------------- producer warp
    // Dynamic schedule: a global ticket t is mapped to a tile through the
    // per-class tile lists (pf_bin's, or the slot-mode prologue's; classes by
    // cost, heaviest first: longest-processing-time order, so the tail of the
    // launch is made of light tiles).  The next tile's ticket and list are
    // fetched right after the current tile's copies go out, overlapping the wait
    // for the next free ring slot.  (Everything here may have been written by
    // this launch's prologue in slot mode: L2 loads, not the nc path.)
    int cls_pre = 0;  // lane l < kTileClasses: tiles in classes heaviest..l (inclusive)
    auto load_classes = [&]() {
      const int c = lane < kTileClasses ? __ldcg(a.classes + (kTileClasses - 1 - lane)) : 0;
      cls_pre = c;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(kFull, cls_pre, o);
        if (lane >= o) cls_pre += y;
      }
    };
    // (slot mode: the class counts are complete only after the grid barrier)
    if (!SLOT && a.classes) load_classes();
    // list base: CSR bin_idx, or (slot mode) the slot + pool lists
    const int32_t* lists = SLOT ? reinterpret_cast<const int32_t*>(a.sb.slot) : a.bin_idx;
    // tickets: the first one of each producer is static (blockIdx, group), later
    // ones come from the global counter (offset by the static range)
    int ticket_k = 0;
    int tile = a.n_tiles, b0 = 0, L = 0, txy = 0, i0 = 0, i1 = 0;
    auto next_tile = [&]() {
      int t = blockIdx.x * G + g;
      if constexpr (SLOT) {
        if (ticket_k == 0) {
          ticket_k = 1;
          const int4 f = s_first[g];  // CTA-local first tile (no ticket)
          if (f.x >= 0) {
            tile = f.x;
            b0 = f.y;
            L = f.z;
            txy = f.w;
            return;
          }
        }
        if (ticket_k == 1) {
          // first global ticket: every CTA's lists and classes are complete
          if (lane == 0)
            while (ld_acquire(a.ctr + 2) < gridDim.x) __nanosleep(64);
          __syncwarp();
          load_classes();
          ticket_k = 2;
        }
        if (lane == 0) t = (int)atomicAdd(a.ctr, 1u);
        t = __shfl_sync(kFull, t, 0);
      } else if (ticket_k++ > 0) {
        if (lane == 0) t = (int)atomicAdd(a.ctr, 1u) + (int)gridDim.x * G;
        t = __shfl_sync(kFull, t, 0);
      }
      tile = a.n_tiles;
      if (t >= a.n_tiles) return;
      if (a.classes) {
        const unsigned below = __ballot_sync(kFull, lane < kTileClasses && cls_pre <= t);
        const int ci = __popc(below);  // rank of the class holding ticket t
        const int before = __shfl_sync(kFull, cls_pre, max(ci - 1, 0));
        const int idx = t - (ci > 0 ? before : 0);
        // (ci == kTileClasses: counts do not cover t -- never with complete lists)
        if (ci < kTileClasses) {
          const int4 e = __ldcg(reinterpret_cast<const int4*>(a.classes + kTileClasses) +
                                (size_t)(kTileClasses - 1 - ci) * a.n_tiles + idx);
          tile = e.x;
          b0 = e.y;
          L = e.z;
          txy = e.w;
        }
      } else {
        tile = t;
        b0 = __ldg(a.bin_off + tile);
        L = __ldg(a.bin_off + tile + 1) - b0;
        txy = (tile % a.ntx) | ((a.ty_begin + tile / a.ntx) << 16);
      }
    };
    auto load_list = [&]() {
      if (tile < a.n_tiles) i0 = lane < L ? __ldcg(lists + b0 + lane) : 0;
      if (ST > 32 && tile < a.n_tiles) i1 = lane + 32 < L ? __ldcg(lists + b0 + lane + 32) : 0;
    };
    int buf = 0;
    uint32_t eph = 0;  // parity of the empty barrier we wait on next, per slot (bit b)
    // one fetch site: the next tile's ticket and list are fetched right after the
    // previous tile's copies went out, before waiting for its ring slot
#pragma unroll 1
    for (int k = 0;; ++k) {
      const unsigned long long cp = prof_ ? clock64() : 0;
      next_tile();
      load_list();
      if (prof_) {  // producer "work" = ticket + list fetch
        p_work += clock64() - cp;
        ++p_n;
      }
      if (k >= kNBuf) {
        const unsigned long long c0 = prof_ ? clock64() : 0;
        mbar_wait_sleep(&empty[g][buf], (eph >> buf) & 1u, a.psleep);
        if (prof_) p_wait += clock64() - c0;
        eph ^= 1u << buf;
      }
      if (tile >= a.n_tiles) {
        int last = 0;
        if (lane == 0) {
          hdr[g][buf] = make_int4(-1, 0, 0, 0);
          mbar_arrive(&full[g][buf]);
          last = atomicAdd(a.ctr + 1, 1u) == gridDim.x * G - 1;
        }
        // the last producer out resets the ticket and (every producer read them
        // at its start) the class counts for the next step; slot mode: publishes
        // K, resets the per-step slot words and the prologue's grid barrier
        if (__shfl_sync(kFull, last, 0)) {
          if (lane == 0) {
            atomicExch(a.ctr, 0u);
            atomicExch(a.ctr + 1, 0u);
            if (SLOT) {
              atomicExch(a.ctr + 2, 0u);  // the prologue's grid barrier
              a.status_rw[0] = (int32_t)atomicExch(a.sb.ctl + kSlotK, 0u);
              a.status_rw[1] = __ldcg(a.sb.ctl + kSlotErr) != 0u ? 1 : 0;
              a.sb.ctl[kSlotPool] = 0u;
              a.sb.ctl[kSlotGather] = 0u;
              a.sb.ctl[kSlotOvf] = 0u;
              a.sb.ctl[kSlotDirty] = 0u;
            }
          }
          // (a render-only pass leaves them: the backward pass on the same lists
          // schedules from them next)
          if (LOSS != PF_LOSS_RENDER && a.classes && lane < kTileClasses) a.classes_rw[lane] = 0;
        }
        break;
      }
      const int nst = min(L, ST);
      const int tx = txy & 0xffff, ty = txy >> 16;
      const int vw = min(kTile, a.W - tx * kTile);
      const int vh = min(kTile, a.H - ty * kTile);
      const uint32_t row_bytes = (uint32_t)vw * sizeof(float4);
      constexpr uint32_t kTgtRows = LOSS == PF_LOSS_RENDER ? 0u : 1u;  // (no target to stage)
      if (lane == 0) {
        hdr[g][buf] = make_int4(tile, b0, L, txy);
        mbar_arrive_tx(&full[g][buf], (uint32_t)nst * kEntBytes +
                                          (uint32_t)vh * row_bytes * ((has_bg ? 1u : 0u) + kTgtRows));
      }
      __syncwarp();
      if (lane < nst) {
        bulk_g2s(buf_rec(buf) + lane, a.recs + i0, sizeof(RecS), &full[g][buf]);
        bulk_g2s(buf_cull(buf) + lane, a.recc + i0, sizeof(RecC), &full[g][buf]);
      }
      if (ST > 32 && lane + 32 < nst) {  // (ST = 64: two entries per lane)
        bulk_g2s(buf_rec(buf) + lane + 32, a.recs + i1, sizeof(RecS), &full[g][buf]);
        bulk_g2s(buf_cull(buf) + lane + 32, a.recc + i1, sizeof(RecC), &full[g][buf]);
      }
      if (lane < vh) {
        const size_t row = (size_t)(ty * kTile + lane) * a.W + (size_t)tx * kTile;
        if (kTgtRows) bulk_g2s(buf_tgt(buf) + lane * kTile, a.tgt4 + row, row_bytes, &full[g][buf]);
        if (has_bg) bulk_g2s(buf_bg(buf) + lane * kTile, a.bg4 + row, row_bytes, &full[g][buf]);
      }
      buf = buf + 1 == kNBuf ? 0 : buf + 1;
    }
    finish();
  } else {
    asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(step_cons_regs(G)));
    // ---------------- consumer warps
    int buf = 0;
    uint32_t fph = 0;
    mbar_wait_sleep(&atl_bar, 0, 100);  // the shared-memory atlas has landed
    for (;;) {
      const unsigned long long c0 = prof_ ? clock64() : 0;
      mbar_wait_sleep(&full[g][buf], (fph >> buf) & 1u, a.csleep);
      const unsigned long long c1 = prof_ ? clock64() : 0;
      if (prof_) {
        p_wait += c1 - c0;
        if (p_n == 0) p_first = c1 - c0;
      }
      fph ^= 1u << buf;
      const int4 h = hdr[g][buf];
      if (h.x < 0) break;
      const RecS* rs = buf_rec(buf);
      const RecC* rc = buf_cull(buf);
      const float4* tgs = buf_tgt(buf);
      const float4* bgs = has_bg ? buf_bg(buf) : nullptr;
      // spill entry base: the CSR offset; slot mode: the group's arena for a list
      // in the tile's own slots, its pool range for a general-path list
      int sbase = h.y;
      if constexpr (SLOT) {
        const int nslot = a.sb.n_tiles * a.sb.m;
        sbase = h.y >= nslot ? (int)gridDim.x * G * kSlotArena + (h.y - nslot)
                             : (int)(blockIdx.x * G + g) * kSlotArena;
      }
      if (h.z <= ST) {
        warp_tile<LOSS>(a, StagedRecs{rs, rc}, atl, tgs, bgs, stA, stB, h.x, sbase, h.z, h.w, wg);
      } else {
        const int32_t* lst = (SLOT ? reinterpret_cast<const int32_t*>(a.sb.slot) : a.bin_idx) + h.y;
        warp_tile<LOSS>(a, MixedRecs<ST>{rs, rc, a.recs, a.recc, lst}, atl, tgs, bgs,
                        stA, stB, h.x, sbase, h.z, h.w, wg);
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[g][buf]);
      if (prof_) {
        const unsigned long long dt = clock64() - c1;
        p_work += dt;
        ++p_n;
        if (lane == 0 && h.x < 65536)
          prof_[6 * 148 * 32 + (size_t)h.x * kCW + wg] = dt | ((unsigned long long)(gtimer() & 0xffffffffu) << 32);
      }
      buf = buf + 1 == kNBuf ? 0 : buf + 1;
    }
    finish();
  }
}

// Fixed-order fold of pf_fit_step's per-warp loss partials into sums[3], used
// before a cross-rank allreduce (single-rank steps fold inside
// pf_adam_preprocess instead).  Many blocks: block b folds the contiguous chunk
// [b*chunk, (b+1)*chunk) (strided by thread, warp butterfly, warps in order) into
// bsum[b]; the last block to finish folds bsum[0..nb) the same way.  The order
// depends on n_part only, never on timing: deterministic.  (One block over all
// partials took 60 us at c5: a serial step on the multi-GPU critical path.)
constexpr int kFoldThreads = 256;
__device__ __forceinline__ void fold3_block(double& v0, double& v1, double& v2,
                                            double (*red)[3]) {
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
}

__global__ void __launch_bounds__(kFoldThreads) k_fold(const double* __restrict__ part,
                                                       int n_part, int chunk, double* bsum,
                                                       unsigned* ctr, double* sums) {
  __shared__ double red[kFoldThreads / 32][3];
  __shared__ bool last;
  pdl_wait();     // the fit step's partials (launched as its programmatic dependent)
  pdl_trigger();  // (the next node -- the allreduce or Adam -- waits for this grid)
  const int t = threadIdx.x;
  const int c0 = blockIdx.x * chunk, c1 = min(n_part, c0 + chunk);
  double v0 = 0.0, v1 = 0.0, v2 = 0.0;
  for (int k = c0 + t; k < c1; k += kFoldThreads) {
    v0 += part[3 * (size_t)k + 0];
    v1 += part[3 * (size_t)k + 1];
    v2 += part[3 * (size_t)k + 2];
  }
  fold3_block(v0, v1, v2, red);
  if (t < 3) {
    double s = 0.0;
    for (int w = 0; w < kFoldThreads / 32; ++w) s += red[w][t];
    bsum[3 * blockIdx.x + t] = s;
    __threadfence();  // (the block sums before the ticket)
  }
  __syncthreads();
  if (t == 0) last = atomicAdd(ctr, 1u) == gridDim.x - 1;
  __syncthreads();
  if (!last) return;
  __threadfence();
  v0 = v1 = v2 = 0.0;
  for (int b = t; b < (int)gridDim.x; b += kFoldThreads) {
    v0 += __ldcg(bsum + 3 * b + 0);
    v1 += __ldcg(bsum + 3 * b + 1);
    v2 += __ldcg(bsum + 3 * b + 2);
  }
  __syncthreads();  // (red reused)
  fold3_block(v0, v1, v2, red);
  if (t < 3) {
    double s = 0.0;
    for (int w = 0; w < kFoldThreads / 32; ++w) s += red[w][t];
    sums[t] = s;
  }
  if (t == 0) *ctr = 0u;  // self-resetting for the next launch / graph replay
}

static int fold_blocks(int n_part) {
  const int nb = (n_part + 511) / 512;
  return nb < 1 ? 1 : (nb > 4 * 148 ? 4 * 148 : nb);
}

}  // namespace pf

using namespace pf;

extern "C" size_t pf_fold_scratch_bytes(int n_part) {
  return n_part < 0 ? 0 : (size_t)fold_blocks(n_part) * 3 * sizeof(double) + 16;
}

extern "C" int pf_fold_loss(const double* part, int n_part, double* sums, void* scratch,
                            void* stream) {
  if (!part || !sums || !scratch || n_part < 0) return PF_ERR_ARG;
  const int nb = fold_blocks(n_part);
  const int chunk = n_part > 0 ? (n_part + nb - 1) / nb : 1;
  double* bsum = static_cast<double*>(scratch);
  unsigned* ctr = reinterpret_cast<unsigned*>(bsum + 3 * (size_t)nb);
  return (int)launch_pdl(k_fold, nb, kFoldThreads, 0, (cudaStream_t)stream, part, n_part, chunk,
                         bsum, ctr, sums);
}

// (capacity entries for CSR offsets / the slot-mode pool, plus the slot-mode
// per-group arenas of kSlotArena entries: one CTA of 3 groups per SM)
extern "C" size_t pf_step_spill_bytes(int capacity) {
  const size_t entries = (size_t)(capacity > 0 ? capacity : 1) + 64 +
                         (size_t)dev_attrs().sms * 3 * kSlotArena;
  return entries * kTilePix * 2 * sizeof(float4);
}

static unsigned long long* g_prof_buf = nullptr;
static int g_prof_slots = 0;

// Diagnostics only (not part of the documented ABI): copy the last profiled
// pf_fit_step's per-warp counters to the host (synchronous).
extern "C" int pf_step_prof_dump(unsigned long long* host, int max_slots) {
  if (!g_prof_buf) return 0;
  const int n = g_prof_slots < max_slots ? g_prof_slots : max_slots;
  cudaDeviceSynchronize();
  cudaMemcpy(host, g_prof_buf, sizeof(unsigned long long) * 6 * n, cudaMemcpyDeviceToHost);
  return n;
}

extern "C" int pf_step_prof_prologue(unsigned long long* host, int n_ctas) {
  if (!g_prof_buf) return 0;
  cudaDeviceSynchronize();
  cudaMemcpy(host, g_prof_buf + 6 * 148 * 32 + 65536 * 8, sizeof(unsigned long long) * 2 * n_ctas,
             cudaMemcpyDeviceToHost);
  // then 4 phase marks per CTA (batch landed, tiles sorted, classes, end)
  cudaMemcpy(host + 2 * n_ctas, g_prof_buf + 6 * 148 * 32 + 65536 * 8 + 512,
             sizeof(unsigned long long) * 4 * n_ctas, cudaMemcpyDeviceToHost);
  return n_ctas;
}

extern "C" int pf_step_prof_tiles(unsigned long long* host, int n_tiles) {
  if (!g_prof_buf) return 0;
  cudaDeviceSynchronize();
  cudaMemcpy(host, g_prof_buf + 6 * 148 * 32, sizeof(unsigned long long) * 8 * (size_t)n_tiles,
             cudaMemcpyDeviceToHost);
  return n_tiles;
}

extern "C" int pf_fit_step(const void* rec, int n, const double* tex, const float* apad,
                           const double* apad64, int pad_texels, int texels, const int32_t* bin_off,
                           const int32_t* bin_idx, const int32_t* status, int W, int H,
                           int ty_begin, int ty_end, double eps_skip, double bg_r, double bg_g,
                           double bg_b, const float* bg4, int loss_kind, const float* tgt4,
                           double alpha_w, double w_mse, double w_gray, double inv_3P,
                           double inv_P, void* spill, float* img4,
                           double* part, double* grads, uint32_t* counters,
                           const int32_t* tile_classes, int stage, void* scratch,
                           size_t scratch_bytes, int capacity, void* slots, int slot_m,
                           void* stream) {
  pf::NvtxRange nvtx_range("pf_fit_step");
  const bool render = loss_kind == PF_LOSS_RENDER;  // forward only: no target / partials / grads
  if (W < 1 || H < 1 || n < 0 || !status || !tex || !apad || (!render && (!tgt4 || !part || !grads)) ||
      (render && !img4) || !spill || !counters || pad_texels < 0 || (pad_texels & 3))
    return PF_ERR_ARG;
  if (!slots && (!bin_off || !bin_idx)) return PF_ERR_ARG;
  if (slots && (slot_m < 1 || !tile_classes || !scratch || capacity < 0)) return PF_ERR_ARG;
  if (loss_kind != PF_LOSS_MSE && loss_kind != PF_LOSS_SPATIAL && loss_kind != PF_LOSS_COMBINED &&
      loss_kind != PF_LOSS_EXTERN && !render)
    return PF_ERR_ARG;
  if ((loss_kind == PF_LOSS_EXTERN || render) && slots) return PF_ERR_ARG;  // (CSR lists only)
  const int ntx = div_up(W, kTile), nty = div_up(H, kTile);
  if (ty_begin < 0 || ty_end > nty || ty_begin > ty_end) return PF_ERR_ARG;
  const int n_tiles = (ty_end - ty_begin) * ntx;
  if (n_tiles == 0) return PF_OK;
  StepArgs a;
  a.recf = (const RecF*)rec;
  a.recc = (const RecC*)((const char*)rec + (sizeof(RecF) + sizeof(RecG)) * (size_t)n);
  a.recs = (const RecS*)((const char*)rec + (sizeof(RecF) + sizeof(RecG) + sizeof(RecC)) * (size_t)n);
  a.tex = tex;
  a.apad = apad;
  a.apad64 = apad64;
  a.pad_texels = pad_texels;
  a.texels = texels;
  a.bin_off = bin_off;
  a.bin_idx = bin_idx;
  a.status = status;
  a.W = W;
  a.H = H;
  a.ntx = ntx;
  a.ty_begin = ty_begin;
  a.n_tiles = n_tiles;
  a.eps_skip = eps_skip;
  // eps re-check band: fp32 taps (<= 6e-8 relative) + affine U, V (<= 1e-10 texel)
  a.eps_band = 1e-6 * eps_skip + 1e-9;
  a.eps_f = (float)eps_skip;
  a.eps_band_f = (float)(1e-6 + 1e-6 * eps_skip);  // >> fp32 taps + lerp error (~2e-7)
  a.k2_3P = (float)(2.0 * inv_3P);
  a.bg0 = bg_r;
  a.bg1 = bg_g;
  a.bg2 = bg_b;
  a.bgf0 = (float)bg_r;
  a.bgf1 = (float)bg_g;
  a.bgf2 = (float)bg_b;
  a.bg4 = (const float4*)bg4;
  a.img4 = (float4*)img4;
  a.tgt4 = (const float4*)tgt4;
  a.alpha_w = alpha_w;
  a.w_mse = w_mse;
  a.w_gray = w_gray;
  a.inv_3P = inv_3P;
  a.inv_P = inv_P;
  a.part = part;
  a.spill = (float4*)spill;
  a.grads = grads;
  a.ctr = counters;
  const Diag& dg = diag();
  a.csleep = dg.csleep;
  a.psleep = dg.psleep;
  a.classes = dg.step_nolpt ? nullptr : tile_classes;
  a.classes_rw = const_cast<int32_t*>(a.classes);
  a.tile_cost = tile_classes ? const_cast<int32_t*>(tile_classes) + tile_cost_offset(n_tiles)
                             : nullptr;
  a.prof = nullptr;
  a.tl = pf_timeline_ptr();
  a.sb = SlotBins{};
  a.rect = nullptr;
  a.done = nullptr;
  a.status_rw = const_cast<int32_t*>(status);
  if (slots) {
    if (scratch_bytes < carve(nullptr, n, capacity, n_tiles).total) return PF_ERR_SCRATCH;
    const BinScratch bs = carve(scratch, n, capacity, n_tiles);
    a.sb = slot_carve(slots, n_tiles, slot_m, capacity);
    a.rect = bs.rect;
    a.done = bs.done;
    if (dg.step_nolpt || !a.classes) return PF_ERR_ARG;  // slot mode needs K1's classes
  }
  static unsigned long long* prof_buf = nullptr;
  if (dg.step_prof) {
    if (!prof_buf)
      cudaMalloc(&prof_buf, sizeof(unsigned long long) * (6 * 148 * 32 + 65536 * 8 + 512 + 1024));
    a.prof = prof_buf;
  }
  g_prof_buf = prof_buf;
  cudaStream_t st = (cudaStream_t)stream;
  const DevAttrs da = dev_attrs();
  const int sms = da.sms, optin = da.optin;
  const size_t budget = (size_t)optin - 1024;  // static smem (barriers, headers)
  // three groups per CTA; the atlas goes to shared memory as float64 when it
  // fits, else float32, else stays global; stage depth 64 on the caller's hint
  // (long tile lists), else 32
  constexpr int G = 3;
  const int ST = stage >= 64 ? 64 : 32;
  const bool no64 = dg.step_atl32;
  const bool bg = bg4 != nullptr;
  const size_t gb = group_bytes(bg, ST);
  const size_t a32 = (size_t)pad_texels * sizeof(float), a64 = 2 * a32;
  // atlas placement at the chosen group count: fp64 in shared memory when it
  // fits, else fp32, else the global fp32 plane through L1 -- never fewer groups
  // (measured at c5, 4 templates: 3 groups + global atlas 422 us/step against
  // 2 groups + shared fp32 atlas 485 us)
  int atl = 0;
  if (!dg.step_atl0) {  // (diagnostics: force the global plane)
    // (the fp32 bilinear path reads fp32 taps: the fp64 copy would only add
    // conversions)
    if (!PF_F32_LERP && apad64 && !no64 && G * gb + a64 <= budget) atl = 2;
    else if (G * gb + a32 <= budget) atl = 1;
  }
  const size_t smem = G * gb + (atl == 2 ? a64 : atl == 1 ? a32 : 0);
  void (*kern)(StepArgs);
#if PF_F32_LERP
#define PF_PICK4(LS, SS, SL)                                                                    \
  kern = bg ? (atl == 1 ? k_step<LS, 1, 3, true, SS, SL> : k_step<LS, 0, 3, true, SS, SL>)     \
            : (atl == 1 ? k_step<LS, 1, 3, false, SS, SL> : k_step<LS, 0, 3, false, SS, SL>);
#else
#define PF_PICK4(LS, SS, SL)                                                                    \
  kern = bg ? (atl == 2   ? k_step<LS, 2, 3, true, SS, SL>                                      \
               : atl == 1 ? k_step<LS, 1, 3, true, SS, SL>                                      \
                          : k_step<LS, 0, 3, true, SS, SL>)                                     \
            : (atl == 2   ? k_step<LS, 2, 3, false, SS, SL>                                     \
               : atl == 1 ? k_step<LS, 1, 3, false, SS, SL>                                     \
                          : k_step<LS, 0, 3, false, SS, SL>);
#endif
#define PF_PICK3(LS, SS)    \
  if (slots) {              \
    PF_PICK4(LS, SS, true)  \
  } else {                  \
    PF_PICK4(LS, SS, false) \
  }
#define PF_PICK(LS)      \
  if (ST == 64) {        \
    PF_PICK3(LS, 64)     \
  } else {               \
    PF_PICK3(LS, 32)     \
  }
  if (loss_kind == PF_LOSS_MSE) {
    PF_PICK(PF_LOSS_MSE)
  } else if (loss_kind == PF_LOSS_EXTERN) {
    if (ST == 64) {
      PF_PICK4(PF_LOSS_EXTERN, 64, false)
    } else {
      PF_PICK4(PF_LOSS_EXTERN, 32, false)
    }
  } else if (render) {
    if (ST == 64) {
      PF_PICK4(PF_LOSS_RENDER, 64, false)
    } else {
      PF_PICK4(PF_LOSS_RENDER, 32, false)
    }
  } else if (loss_kind == PF_LOSS_COMBINED) {
    PF_PICK(PF_LOSS_COMBINED)
  } else {
    PF_PICK(PF_LOSS_SPATIAL)
  }
#undef PF_PICK4
#undef PF_PICK3
#undef PF_PICK
  if (const cudaError_t e = ensure_dyn_smem((const void*)kern, smem)) return (int)e;
  const int grid = min(sms, max(1, (n_tiles + G - 1) / G));
  g_prof_slots = grid * step_warps(G);
  return (int)launch_pdl(kern, grid, step_threads(G), smem, st, a);
}
