// Cross-band gradient exchange: a fixed-order sum of the bands' float64
// gradient + loss buffers (8N + 4 doubles), written back to every
// band's buffer.
//
// Reference: there is no multi-device path in the reference; its backward sums
// per-tile partials sequentially in tile order (reduce_partials,
// pkg/src/primfit/grad.py:190-206).  The row-band split turns
// that sum into one sum over bands per step.  Summing the bands in a FIXED
// order (band 0 first) gives bit-identical buffers on every band, so the
// replicated Adam steps stay identical.
//
// The pointers are plain device addresses: the bands' buffers on one device
// (the in-process band group, tests and projections), or peer buffers mapped
// over NVLink (cudaIpcOpenMemHandle) when each band lives on its own GPU --
// then rank r passes [begin, end) = its 1/world slice and the kernel is the
// one-shot reduce-scatter + all-gather over peer loads / stores.
#include "../../include/primfit_b200.h"
#include "pf_common.cuh"

namespace pf {
namespace {

struct SumArgs {
  const double* src[PF_MAX_BANDS];
  double* dst[PF_MAX_BANDS];
  int nsrc, ndst;
  long long begin, end;
};

__global__ void __launch_bounds__(256) k_sum_bands(SumArgs a) {
  pdl_wait();
  pdl_trigger();  // the dependent (Adam) reads the sums only after its own wait
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long i = a.begin + (long long)blockIdx.x * blockDim.x + threadIdx.x; i < a.end;
       i += stride) {
    double s = a.src[0][i];
    for (int k = 1; k < a.nsrc; ++k) s += a.src[k][i];
    for (int k = 0; k < a.ndst; ++k) a.dst[k][i] = s;
  }
}

}  // namespace
}  // namespace pf

using namespace pf;

extern "C" int pf_sum_bands(const double* const* srcs, int nsrc, double* const* dsts, int ndst,
                            long long begin, long long end, void* stream) {
  if (!srcs || !dsts || nsrc < 1 || nsrc > PF_MAX_BANDS || ndst < 0 || ndst > PF_MAX_BANDS ||
      begin < 0 || end < begin)
    return PF_ERR_ARG;
  SumArgs a = {};
  for (int k = 0; k < nsrc; ++k) {
    if (!srcs[k]) return PF_ERR_ARG;
    a.src[k] = srcs[k];
  }
  for (int k = 0; k < ndst; ++k) {
    if (!dsts[k]) return PF_ERR_ARG;
    a.dst[k] = dsts[k];
  }
  a.nsrc = nsrc;
  a.ndst = ndst;
  a.begin = begin;
  a.end = end;
  if (end == begin) return PF_OK;
  const long long n = end - begin;
  const int grid = (int)(n / 256 + 1 < 1184 ? n / 256 + 1 : 1184);
  return (int)launch_pdl(k_sum_bands, grid, 256, 0, (cudaStream_t)stream, a);
}
