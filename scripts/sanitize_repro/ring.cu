// Minimal repro of k_step's producer / consumer ring (pf_step.cu) for
// compute-sanitizer: is the mbarrier-synchronised pattern itself reported?
//   one producer warp: waits `empty` (after the first kNBuf slots), writes the
//   slot header, arrive.expect_tx on `full`, bulk-copies data into the slot;
//   consumer warps: wait `full`, read header + data, __syncwarp, lane 0 arrives
//   on `empty`.  SETMAXNREG=1 adds the register hand-over of k_step.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 -lineinfo -DSETMAXNREG=<0|1> ring.cu
#include <cstdio>
#include <cstdint>
#ifndef SETMAXNREG
#define SETMAXNREG 1
#endif
#ifndef GROUPS
#define GROUPS 1
#endif
constexpr int kNBuf = 2, kCons = GROUPS == 1 ? 4 : 8, kItems = 64, kWords = 256;
constexpr int kG = GROUPS, kThreads = GROUPS == 1 ? 256 : 896;

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t c) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(c) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(b)) : "memory");
}
__device__ __forceinline__ void mbar_arrive_tx(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ bool mbar_try(uint64_t* b, uint32_t parity) {
  uint32_t ok;
  asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}"
               : "=r"(ok) : "r"(su32(b)), "r"(parity) : "memory");
  return ok != 0;
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               ::"r"(su32(dst)), "l"(src), "r"(bytes), "r"(su32(bar)) : "memory");
}

__global__ void __launch_bounds__(kThreads, 1) k_ring(const int* src, int* out) {
  __shared__ __align__(128) int bufs[kG][kNBuf][kWords];
  __shared__ __align__(8) uint64_t fulls[kG][kNBuf], emptys[kG][kNBuf];
  __shared__ int hdrs[kG][kNBuf];
  __shared__ __align__(8) uint64_t atl_bar;
  extern __shared__ __align__(128) unsigned char dyn[];
  const int t = threadIdx.x, warp = t >> 5, lane = t & 31;
  if (t == 0) {
    mbar_init(&atl_bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    mbar_arrive_tx(&atl_bar, 16384);
    bulk_g2s(dyn, src, 16384, &atl_bar);
  }
  if (t < kG * kNBuf) {
    mbar_init(&fulls[t / kNBuf][t % kNBuf], 1);
    mbar_init(&emptys[t / kNBuf][t % kNBuf], kCons);
  }
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  __syncthreads();
  const bool consumer = warp < kG * kCons;
  const int g = consumer ? warp / kCons : warp - kG * kCons;
  int (*buf)[kWords] = bufs[g < kG ? g : 0];
  uint64_t* full = fulls[g < kG ? g : 0];
  uint64_t* empty = emptys[g < kG ? g : 0];
  int* hdr = hdrs[g < kG ? g : 0];
  if (!consumer) {
#if SETMAXNREG
    asm volatile("setmaxnreg.dec.sync.aligned.u32 24;");
#endif
    if (g >= kG) return;
    uint32_t eph = 0;
    for (int k = 0; k <= kItems; ++k) {
      const int b = k % kNBuf;
      if (k >= kNBuf) {
        while (!mbar_try(&empty[b], (eph >> b) & 1u)) __nanosleep(100);
        eph ^= 1u << b;
      }
      if (lane == 0) {
        hdr[b] = k < kItems ? k : -1;
        if (k < kItems) {
          mbar_arrive_tx(&full[b], kWords * 4);
          bulk_g2s(buf[b], src + (size_t)k * kWords, kWords * 4, &full[b]);
        } else {
          mbar_arrive(&full[b]);
        }
      }
      __syncwarp();
    }
  } else {
#if SETMAXNREG
    asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(GROUPS == 1 ? 232 : 80));
#endif
    while (!mbar_try(&atl_bar, 0)) __nanosleep(100);
    uint32_t fph = 0;
    int acc = 0;
    for (int k = 0;; ++k) {
      const int b = k % kNBuf;
      while (!mbar_try(&full[b], (fph >> b) & 1u)) __nanosleep(100);
      fph ^= 1u << b;
      const int h = hdr[b];
      if (h < 0) break;
      for (int i = lane; i < kWords; i += 32) acc += buf[b][i] * (warp + 1) + h + dyn[i];
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[b]);
    }
    atomicAdd(out, acc);
  }
}

int main() {
  int *src, *out;
  cudaMalloc(&src, sizeof(int) * kItems * kWords);
  cudaMalloc(&out, sizeof(int));
  cudaMemset(src, 1, sizeof(int) * kItems * kWords);
  cudaMemset(out, 0, sizeof(int));
  cudaFuncSetAttribute(k_ring, cudaFuncAttributeMaxDynamicSharedMemorySize, 180000);
  k_ring<<<148, kThreads, 180000>>>(src, out);
  const cudaError_t e = cudaDeviceSynchronize();
  int h = 0;
  cudaMemcpy(&h, out, sizeof(int), cudaMemcpyDeviceToHost);
  printf("ring: %s, sum %d\n", cudaGetErrorString(e), h);
  return e != cudaSuccess;
}
