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
#include <cstdlib>
#include <utility>
#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>  // header-only NVTX3: a no-op unless a tool (nsys, ncu) injects

namespace pf {

// NVTX range over one C-ABI entry point (host side: the launch call it names;
// nsys / ncu --nvtx show each stage by name).
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange&) = delete;
  NvtxRange& operator=(const NvtxRange&) = delete;
};

constexpr int kTile = 16;                 // render tile edge (16x16 pixels / block)
constexpr int kTilePix = kTile * kTile;   // 256 threads per render block
constexpr unsigned kFull = 0xffffffffu;

// Forward record: everything the per-pair forward math reads (128 bytes).
struct __align__(16) RecF {
  double px, py;          // centre (canvas px; pixel centres at integer coords)
  double ct, st;          // cos / sin of rotation
  double inv_s, inv_sq;   // RN(1/s), RN(1/(s q)) -- exact-quotient division (div_rn)
  double s, sq;           // scale, scale * aspect   (v divisor, _kernels.py:112)
  double wm1, hm1;        // (double)(wt - 1), (double)(ht - 1)
  double sa;              // alpha_max * sigmoid(opacity_logit)
  double c0, c1, c2;      // (1 - mu_blend) * sigmoid(color_logit)
  int32_t base, wt, ht, tid;  // template atlas slot
};
static_assert(sizeof(RecF) == 128, "RecF must be 128 bytes");

// Gradient record (80 bytes, fp32): everything the backward reads per
// primitive.  The backward takes no decision (the saved entries fix which
// pairs contribute), so fp32 suffices for the 1e-3 gradient bar (measured
// ~1e-5 against the float64 reference); it is staged in shared memory.
struct __align__(16) RecG {
  float sa, c0, c1, c2;       // alpha_max*sig, (1-mu)*sigmoid(c)
  float sd, cd0, cd1, cd2;    // alpha_max*sig*(1-sig), sc*(1-sc)
  float gxu, gxv, gyu, gyv;   // -ct/s, st/(s q), -st/s, -ct/(s q)
  float inv_s, q, inv_q, hw;  // 1/s, aspect, 1/aspect, 0.5 (wt - 1)
  float hh, inv_hw, inv_hh, omm;  // 0.5 (ht - 1), 1/hw, 1/hh, 1 - mu_blend
  int32_t base, wt, ht, pad;  // template atlas slot
};
static_assert(sizeof(RecG) == 96, "RecG must be 96 bytes");

// Cull record (32 bytes, fp32): just what the warp-level footprint test needs,
// so testing 32 list entries costs two 16-byte loads per lane.
//   u(c) ~= au*dx + bu*dy,  v(c) ~= av*dy - bv*dx  (dx = c.x - px, dy = c.y - py)
//   eu, ev: the warp rectangle's projected half widths in (u, v) units plus the
//   rounding slack of the fp32 centre (conservative; never rejects a hit).
struct __align__(16) RecC {
  float px, py, au, bu;
  float av, bv, eu, ev;
};
static_assert(sizeof(RecC) == 32, "RecC must be 32 bytes");

// Step record (224 bytes): everything pf_fit_step reads per list entry, staged
// in shared memory once per tile by TMA bulk copies.
//   forward  texel coordinates as one affine map per axis, centred on the box:
//              U - hw = au*x + bu*y + cu,  V - hh = av*x + bv*y + cv   (float64)
//            -- the reference's per-pair chain (_kernels.py:106-114) folded into
//            per-primitive coefficients.  They differ from the reference's U, V
//            by < 1e-10 texel; `delta` (>= 1e4 x that bound) is the guard band:
//            |U - hw| < hw - delta (both axes) is inside for the reference too,
//            > hw + delta is outside; anything between re-takes the inside test
//            with the reference's exact op order (texel_coords on RecF), so
//            every inside/outside decision matches the reference.
//            Opacity / colours in float64 for the compositing; pbase/wp address
//            the zero-padded alpha plane.
//   backward fp32 gradient coefficients (as RecG) and gidx = the row of grads.
struct __align__(16) RecS {
  double au, bu, cu, av, bv, cv;
  double sa, c0, c1, c2;        // alpha_max*sig, (1-mu)*sigmoid(c)
  double hwd, hhd;              // (wt - 1) / 2, (ht - 1) / 2
  double in_u, out_u;           // hw - delta, hw + delta
  double in_v, out_v;           // hh - delta, hh + delta
  int32_t pbase, wp;            // padded-atlas base, padded row stride (wt + 1)
  int32_t gidx, pad_i;          // primitive index (row of params / grads)
  float sd, cd0, cd1, cd2;      // alpha_max*sig*(1-sig), sc*(1-sc)
  float gxu, gxv, gyu, gyv;     // -ct/s, st/(s q), -st/s, -ct/(s q)
  float inv_s, q, inv_q, hw;    // 1/s, aspect, 1/aspect, 0.5 (wt - 1)
  float hh, omm, saf, inv_hw;   // 0.5 (ht - 1), 1 - mu_blend, (float)sa, 1 / hw
  float c0f, c1f, c2f, inv_hh;  // (float)c, 1 / hh
};
static_assert(sizeof(RecS) == 224, "RecS must be 224 bytes");

// Tile cost classes for pf_fit_step's longest-first schedule.  pf_bin's
// optional tile_classes buffer: int32 [kTileClasses] counts, then
// [kTileClasses][n_tiles] int4 tile entries (tile, list offset, list length,
// tx | ty << 16), then [n_tiles] tile costs measured by the previous
// pf_fit_step (its rects' candidate + backward-step counts, max over the tile;
// 0 = unknown).  Class = cost / 4, or list length / 4 when the cost is
// unknown, capped at kTileClasses - 1.
constexpr int kTileClasses = 16;
__host__ __device__ inline size_t tile_cost_offset(int n_tiles) {
  return kTileClasses + 4 * (size_t)kTileClasses * n_tiles;
}
__host__ __device__ inline int tile_class(int L) { return L / 4 < kTileClasses - 1 ? L / 4 : kTileClasses - 1; }

// Warp sub-tile shape (8 warps cover a 16x16 tile) -- used by the cull record.
constexpr int kWarpW = 8, kWarpH = 4;

// Saved forward entry (16 bytes, one 128-bit store / load): list position j
// (16 bits), texel cell u0, v0 (16 bits each), bilinear weights wu, wv as
// 24-bit fixed point (2^-24 = fp32 resolution on [0, 1)) and the incoming
// transmittance T (the reference's Tbuf, _kernels.py:294-297) as fp32:
//   w0 = j | u0 << 16,  w1 = v0 | wu[23:8] << 16,  w2 = wu[7:0] | wv << 8,  w3 = T
struct __align__(16) SavedEnt {
  uint32_t w0, w1, w2;
  float T;
};

__device__ __forceinline__ uint32_t to_fix24(double w) {
  const double q = w * 16777216.0 + 0.5;
  return (uint32_t)(q >= 16777215.0 ? 16777215.0 : (q < 0.0 ? 0.0 : q));
}

__device__ __forceinline__ SavedEnt pack_saved(int j, int u0, int v0, double wu, double wv,
                                              double T) {
  const uint32_t qu = to_fix24(wu), qv = to_fix24(wv);
  SavedEnt s;
  s.w0 = (uint32_t)(j & 0xffff) | ((uint32_t)(u0 & 0xffff) << 16);
  s.w1 = (uint32_t)(v0 & 0xffff) | ((qu >> 8) << 16);
  s.w2 = (qu & 0xffu) | (qv << 8);
  s.T = (float)T;
  return s;
}

struct SavedView {
  int j, u0, v0;
  float wu, wv, T;
};

__device__ __forceinline__ SavedView unpack_saved(const SavedEnt& s) {
  SavedView v;
  v.j = (int)(s.w0 & 0xffffu);
  v.u0 = (int)(int16_t)(s.w0 >> 16);
  v.v0 = (int)(int16_t)(s.w1 & 0xffffu);
  const uint32_t qu = ((s.w1 >> 16) << 8) | (s.w2 & 0xffu);
  v.wu = (float)qu * (1.0f / 16777216.0f);
  v.wv = (float)(s.w2 >> 8) * (1.0f / 16777216.0f);
  v.T = s.T;
  return v;
}
static_assert(sizeof(SavedEnt) == 16, "SavedEnt must be 16 bytes");

// Stable two-branch logistic, _kernels.py:27-32, without the branch: both arms
// evaluate exp(-|x|) (exp(-x) for x >= 0, exp(x) below) and divide by 1 + e, so
// one exp and one division give the reference's value for every x (NaN, +-0,
// +-inf included) and divergent lanes do not run both arms.
__device__ __forceinline__ double sigmoid(double x) {
  const double e = exp(-fabs(x));
  return (x >= 0.0 ? 1.0 : e) / (1.0 + e);
}

// a / b given inv = RN(1/b): Markstein correction step.  The result is exact
// whenever a/b is representable (so lattice / box-edge hits land exactly where
// the reference's correctly rounded division puts them) and correctly rounded
// in all but vanishingly rare cases otherwise.  3 FP64 ops instead of DDIV.
__device__ __forceinline__ double div_rn(double a, double b, double inv) {
  const double q0 = a * inv;
  const double r = fma(-q0, b, a);
  return fma(r, inv, q0);
}

// Canvas pixel -> texel coordinates, reference op order (_kernels.py:109-115),
// no contraction.  Returns the inside-box predicate (inclusive at W-1).
__device__ __forceinline__ bool texel_coords(const RecF& r, double xx, double yy,
                                             double& U, double& V) {
  const double dx = __dsub_rn(xx, r.px);
  const double dy = __dsub_rn(yy, r.py);
  const double u = div_rn(__dadd_rn(__dmul_rn(r.ct, dx), __dmul_rn(r.st, dy)), r.s, r.inv_s);
  const double v = div_rn(__dadd_rn(__dmul_rn(-r.st, dx), __dmul_rn(r.ct, dy)), r.sq, r.inv_sq);
  U = __dmul_rn(__dmul_rn(__dadd_rn(u, 1.0), 0.5), r.wm1);
  V = __dmul_rn(__dmul_rn(__dadd_rn(v, 1.0), 0.5), r.hm1);
  return !(U < 0.0 || U > r.wm1 || V < 0.0 || V > r.hm1);
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

// Alpha "quad atlas": for texel (u, v) of a template, the four bilinear taps
// (a[v][u], a[v][u+1], a[v+1][u], a[v+1][u+1]) with the reference's zero
// padding already applied (_kernels.py:35-40), as fp32 (one 16-byte load per
// sample, no bounds checks).  Built once per atlas by pf_atlas_quad.  The fp32
// taps move m by <= 6e-8 relative; the one decision that depends on m
// (m < eps_skip) is re-taken on the float64 plane when m is within 1e-6 of eps.
__device__ __forceinline__ float4 load_quad(const float4* __restrict__ quad, int base, int wt,
                                            int u0, int v0) {
  return __ldg(quad + (size_t)base + v0 * wt + u0);
}

__device__ __forceinline__ double bilerp(const float4& t, double wu, double wv) {
  const double iu = 1.0 - wu, iv = 1.0 - wv;
  return (iu * iv) * (double)t.x + (wu * iv) * (double)t.y + (iu * wv) * (double)t.z +
         (wu * wv) * (double)t.w;
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

// Programmatic dependent launch (PDL): kernels of the fit step are launched
// with programmatic stream serialization, so a kernel's blocks may start while
// its predecessor drains.  Rules: (1) before pdl_wait() a kernel reads nothing
// its predecessor writes and writes nothing its predecessor reads; (2) every
// path calls pdl_wait() before exiting; (3) a kernel whose dependent reads
// data from EARLIER kernels before its own wait triggers only after its wait
// (then "dependent launched" implies "everything before me completed").
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

// Diagnostics timeline (PF_TIMELINE=1 builds the pointer; NULL otherwise):
// per kernel slot k, [4k] = min block start, [4k+1] = min PDL-wait return,
// [4k+2] = max PDL-wait return, [4k+3] = max block end (globaltimer ns).
__device__ __forceinline__ unsigned long long gtime_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
#ifndef PF_DIAG
#define PF_DIAG 1  // diagnostics code compiled in (the product library is built with 0)
#endif
__device__ __forceinline__ void tl_mark(unsigned long long* tl, int slot, int what) {
  if (!PF_DIAG) return;
  if (tl != nullptr && what == 2) {  // any lane-0 caller: min / max into the wait fields
    if ((threadIdx.x & 31) != 0) return;
    const unsigned long long t = gtime_ns();
    atomicMin(tl + 4 * slot + 1, t);
    atomicMax(tl + 4 * slot + 2, t);
    return;
  }
  if (tl == nullptr || (threadIdx.x & (what == 3 ? 31 : 0xffffffff)) != 0) return;
  const unsigned long long t = gtime_ns();
  if (what == 0 || what == 1) atomicMin(tl + 4 * slot + what, t);
  if (what == 1 || what == 3) atomicMax(tl + 4 * slot + (what == 1 ? 2 : 3), t);
}
unsigned long long* pf_timeline_ptr();

// ---- host-side launch helpers, per device (one process may drive several GPUs)
constexpr int kMaxDevices = 64;
struct DevAttrs {
  int sms, optin;  // SM count, opt-in shared memory per block
};
inline DevAttrs dev_attrs() {
  static DevAttrs cache[kMaxDevices] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  DevAttrs a = {0, 0};
  if (dev >= 0 && dev < kMaxDevices && cache[dev].sms > 0) return cache[dev];
  cudaDeviceGetAttribute(&a.sms, cudaDevAttrMultiProcessorCount, dev);
  cudaDeviceGetAttribute(&a.optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  if (dev >= 0 && dev < kMaxDevices) cache[dev] = a;  // (benign race: same values)
  return a;
}
// cudaFuncAttributeMaxDynamicSharedMemorySize >= smem for `kern` on the current
// device, set at most once per (device, kernel) and size increase.
cudaError_t ensure_dyn_smem(const void* kern, size_t smem);

// Diagnostics switches (A/B runs, profiling), read from the environment once per
// process -- never on the launch path.
struct Diag {
  bool no_pdl, step_nolpt, step_prof, step_atl32, step_atl0, timeline;
  unsigned csleep, psleep;
  int bin_ncb, bin_two_level;  // -1: not set
};
const Diag& diag();

template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl2(void (*kern)(KArgs...), dim3 grid, int block, size_t smem,
                               cudaStream_t st, Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = dim3((unsigned)block);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = diag().no_pdl ? 0 : 1;  // (A/B switch PF_NO_PDL)
  return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}
template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*kern)(KArgs...), int grid, int block, size_t smem,
                              cudaStream_t st, Args&&... args) {
  return launch_pdl2(kern, dim3((unsigned)grid), block, smem, st, std::forward<Args>(args)...);
}

}  // namespace pf
