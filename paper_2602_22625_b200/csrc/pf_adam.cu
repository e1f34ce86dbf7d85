#include <mutex>
// K5 fused Adam step + loss/psnr history + gradient zeroing.
//
// Reference: adam_step (pkg/src/primfit/fit.py:195-238):
//   m = b1*m + (1-b1)*g ; v = b2*v + (1-b2)*g^2 ; m_hat = m/(1-b1^t) ; v_hat = v/(1-b2^t)
//   p -= (lr*gain) * m_hat / (sqrt(v_hat) + eps)   for live (non-frozen) primitives only;
//   then the scale column is clipped to [s_min, s_max] for ALL rows (fit.py:235-237).
// Same operation order, no FMA contraction, bias corrections and lr taken from
// host-computed tables (lr_schedule, fit.py:174-186, and Python's own
// 1 - beta**t), so given identical gradients the update is bit-identical.
// psnr (fit.py:241-247) = 10*log10(1/mse), inf when mse == 0.
#include <math_constants.h>

#include <cstdlib>

#include "../../include/primfit_b200.h"
#include "pf_common.cuh"

namespace pf {

constexpr double kB1 = 0.9, kB2 = 0.999, kEps = 1e-8;

struct AdamArgs {
  double* params;
  double* grads;
  double* m;
  double* v;
  const uint8_t* frozen;
  double gains[8];
  int n;
  const double* lr_table;
  const double* bc1_table;
  const double* bc2_table;
  int32_t* iter;
  double lr, bc1, bc2;
  int clamp;
  double s_min, s_max;
  int zero_grads;
  const double* sums;
  int loss_kind;
  double alpha_w, inv_3P, inv_P;
  double* hist_loss;
  double* hist_psnr;
  uint32_t* counter;
};

__global__ void __launch_bounds__(256) k_adam(AdamArgs a) {
  __shared__ bool am_last;
  const int idx = blockIdx.x * blockDim.x + threadIdx.x;
  int it = 0;
  double lr = a.lr, bc1 = a.bc1, bc2 = a.bc2;
  if (a.iter) {
    it = *a.iter;
    lr = a.lr_table[it];
    bc1 = a.bc1_table[it];
    bc2 = a.bc2_table[it];
  }
  if (idx < a.n * 8) {
    const int prim = idx >> 3, col = idx & 7;
    const double g = a.grads[idx];
    if (a.zero_grads) a.grads[idx] = 0.0;
    double p = a.params[idx];
    const bool live = a.frozen == nullptr || a.frozen[prim] == 0;
    if (live) {
      const double mm = __dadd_rn(__dmul_rn(kB1, a.m[idx]), __dmul_rn(1.0 - kB1, g));
      const double vv =
          __dadd_rn(__dmul_rn(kB2, a.v[idx]), __dmul_rn(1.0 - kB2, __dmul_rn(g, g)));
      a.m[idx] = mm;
      a.v[idx] = vv;
      const double mh = __ddiv_rn(mm, bc1);
      const double vh = __ddiv_rn(vv, bc2);
      const double eff = __dmul_rn(lr, a.gains[col]);
      p = __dsub_rn(p, __ddiv_rn(__dmul_rn(eff, mh), __dadd_rn(__dsqrt_rn(vh), kEps)));
    }
    if (a.clamp && col == 2) p = fmin(fmax(p, a.s_min), a.s_max);
    a.params[idx] = p;
  }
  if (a.iter) {
    __syncthreads();
    if (threadIdx.x == 0) {
      __threadfence();
      const unsigned t = atomicAdd(a.counter, 1u);
      am_last = (t == gridDim.x - 1);
    }
    __syncthreads();
    if (am_last && threadIdx.x == 0) {
      if (a.sums) {
        const double mse = a.sums[0] * a.inv_3P;
        double loss = mse;
        if (a.loss_kind == PF_LOSS_SPATIAL)
          loss = a.sums[1] * a.inv_3P + a.alpha_w * (a.sums[2] * a.inv_P);
        if (a.hist_loss) a.hist_loss[it] = loss;
        if (a.hist_psnr) a.hist_psnr[it] = mse == 0.0 ? CUDART_INF : 10.0 * log10(1.0 / mse);
      }
      *a.iter = it + 1;
      *a.counter = 0u;
    }
  }
}

}  // namespace pf

using namespace pf;

extern "C" int pf_adam(double* params, double* grads, double* m, double* v, const uint8_t* frozen,
                       const double* gains8, int n, const double* lr_table,
                       const double* bc1_table, const double* bc2_table, int32_t* iter,
                       double lr, double bc1, double bc2, int clamp, double s_min, double s_max,
                       int zero_grads, const double* sums, int loss_kind, double alpha_w,
                       double inv_3P, double inv_P, double* hist_loss, double* hist_psnr,
                       uint32_t* counter, void* stream) {
  if (n < 0 || (n > 0 && (!params || !grads || !m || !v))) return PF_ERR_ARG;
  if (iter && (!lr_table || !bc1_table || !bc2_table || !counter)) return PF_ERR_ARG;
  AdamArgs a;
  a.params = params;
  a.grads = grads;
  a.m = m;
  a.v = v;
  a.frozen = frozen;
  for (int c = 0; c < 8; ++c) a.gains[c] = gains8 ? gains8[c] : 1.0;
  a.n = n;
  a.lr_table = lr_table;
  a.bc1_table = bc1_table;
  a.bc2_table = bc2_table;
  a.iter = iter;
  a.lr = lr;
  a.bc1 = bc1;
  a.bc2 = bc2;
  a.clamp = clamp;
  a.s_min = s_min;
  a.s_max = s_max;
  a.zero_grads = zero_grads;
  a.sums = sums;
  a.loss_kind = loss_kind;
  a.alpha_w = alpha_w;
  a.inv_3P = inv_3P;
  a.inv_P = inv_P;
  a.hist_loss = hist_loss;
  a.hist_psnr = hist_psnr;
  a.counter = counter;
  const int total = n * 8;
  const int blocks = div_up(total > 0 ? total : 1, 256);
  k_adam<<<blocks, 256, 0, (cudaStream_t)stream>>>(a);
  return (int)cudaGetLastError();
}

extern "C" int pf_abi_version(void) { return 8; }
extern "C" size_t pf_record_bytes(void) { return sizeof(RecF) + sizeof(RecG) + sizeof(RecC) + sizeof(RecS); }
extern "C" int pf_render_tile(void) { return kTile; }
extern "C" long long pf_saved_capacity(int capacity) {
  return (long long)capacity * (long long)kTilePix;
}

static pf::Diag read_diag() {
    using pf::Diag;
    auto flag = [](const char* k) { return getenv(k) != nullptr; };
    auto num = [](const char* k, int dflt) { const char* e = getenv(k); return e ? atoi(e) : dflt; };
    Diag v;
    v.no_pdl = flag("PF_NO_PDL");
    v.step_nolpt = flag("PF_STEP_NOLPT");
    v.step_prof = flag("PF_STEP_PROF");
    v.step_atl32 = flag("PF_STEP_ATL32");
    v.step_atl0 = flag("PF_STEP_ATL0");
    v.timeline = flag("PF_TIMELINE");
    v.csleep = (unsigned)num("PF_CSLEEP", 200);
    v.psleep = (unsigned)num("PF_PSLEEP", 500);
    v.bin_ncb = num("PF_BIN_NCB", -1);
    v.bin_two_level = num("PF_BIN_TWO_LEVEL", -1);
    return v;
}
static pf::Diag g_diag = read_diag();
const pf::Diag& pf::diag() { return g_diag; }
// Diagnostics only: re-read the PF_* switches (tests that flip them at run time).
extern "C" int pf_diag_reload(void) {
  g_diag = read_diag();
  return 0;
}

cudaError_t pf::ensure_dyn_smem(const void* kern, size_t smem) {
  struct Entry {
    int dev;
    const void* kern;
    size_t smem;
  };
  static Entry table[256];
  static int used = 0;
  static std::mutex mu;
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lock(mu);
  for (int i = 0; i < used; ++i) {
    Entry& e = table[i];
    if (e.dev == dev && e.kern == kern) {
      if (smem <= e.smem) return cudaSuccess;
      const cudaError_t r =
          cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      if (r == cudaSuccess) e.smem = smem;
      return r;
    }
  }
  const cudaError_t r =
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (r == cudaSuccess && used < 256) table[used++] = Entry{dev, kern, smem};
  return r;
}

// Diagnostics timeline buffer (see tl_mark in pf_common.cuh): allocated on the
// first call when PF_TIMELINE is set in the environment, else NULL.
static unsigned long long* g_tl = nullptr;
extern "C" int pf_timeline_reset();
unsigned long long* pf::pf_timeline_ptr() {
  static bool checked = false;
  if (!checked) {
    checked = true;
    if (diag().timeline) {
      cudaMalloc(&g_tl, sizeof(unsigned long long) * 64);
      pf_timeline_reset();
    }
  }
  return g_tl;
}

extern "C" int pf_timeline_reset() {
  if (!g_tl) return 0;
  unsigned long long h[64];
  for (int k = 0; k < 16; ++k) {
    h[4 * k] = ~0ull;
    h[4 * k + 1] = ~0ull;
    h[4 * k + 2] = 0;
    h[4 * k + 3] = 0;
  }
  cudaMemcpy(g_tl, h, sizeof(h), cudaMemcpyHostToDevice);
  return 1;
}

extern "C" int pf_timeline_dump(unsigned long long* host) {
  if (!g_tl) return 0;
  cudaDeviceSynchronize();
  cudaMemcpy(host, g_tl, sizeof(unsigned long long) * 64, cudaMemcpyDeviceToHost);
  return 1;
}
