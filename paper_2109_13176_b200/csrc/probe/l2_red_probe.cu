// l2_red_probe.cu -- measurement tool (not part of the gvom ABI): the L2
// reduction ceiling the ray cast's miss counting runs against (SURVEY.md 8(d):
// "Microbenchmark it: red.global.add.u32 into 16 MB / 64 MB / 512 MB arrays.
// Report it beside the HBM fraction").
//
//   probe_red(bytes, pattern, n_ops, &ms): n_ops red.global.add.u32 into a
//   zeroed u32 array of `bytes` (power of two), timed with CUDA events.
//   pattern 0: every lane a random word (32 L2 requests per warp instruction);
//   pattern 1: the 32 lanes of a warp hit 32 words of one random 128-byte line
//              (one request per instruction, 32 atomic ALU ops);
//   pattern 2: runs of 4 lanes share a random word (the ray cast's merged
//              shape is one red per run: this counts one op per run head).
#include <cuda_runtime.h>
#include <stdint.h>

namespace {

__device__ __forceinline__ uint32_t mix(uint64_t x) {
  x ^= x >> 33;
  x *= 0xff51afd7ed558ccdull;
  x ^= x >> 33;
  x *= 0xc4ceb9fe1a85ec53ull;
  x ^= x >> 33;
  return (uint32_t)x;
}

__device__ __forceinline__ void red_add(uint32_t* p, uint32_t v) {
  asm volatile("red.relaxed.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

__global__ void __launch_bounds__(256) k_red_probe(uint32_t* __restrict__ a, uint32_t mask,
                                                   int pattern, int64_t n_iter, uint64_t seed) {
  const int lane = threadIdx.x & 31;
  const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t it = 0; it < n_iter; ++it) {
    const uint64_t key = seed + (uint64_t)(gw + it * nw);
    if (pattern == 0) {
      red_add(a + (mix(key * 32 + lane) & mask), 1u);
    } else if (pattern == 1) {
      const uint32_t line = mix(key) & (mask & ~31u);
      red_add(a + line + lane, 1u);
    } else {
      if ((lane & 3) == 0) red_add(a + (mix(key * 8 + (lane >> 2)) & mask), 4u);
    }
  }
}

}  // namespace

extern "C" __attribute__((visibility("default"))) int probe_red(int64_t bytes, int pattern,
                                                                 int64_t n_warp_iters, float* ms,
                                                                 int64_t* warp_insts) {
  uint32_t* a = nullptr;
  if (cudaMalloc(&a, (size_t)bytes) != cudaSuccess) return -1;
  cudaMemset(a, 0, (size_t)bytes);
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int blocks = sms * 8, threads = 256;
  const int64_t warps = (int64_t)blocks * threads / 32;
  const int64_t iters = (n_warp_iters + warps - 1) / warps;
  const uint32_t mask = (uint32_t)(bytes / 4 - 1);
  k_red_probe<<<blocks, threads>>>(a, mask, pattern, 4, 1);  // warm-up
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  k_red_probe<<<blocks, threads>>>(a, mask, pattern, iters, 12345);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  cudaEventElapsedTime(ms, e0, e1);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  const cudaError_t err = cudaGetLastError();
  cudaFree(a);
  *warp_insts = iters * warps;  // red instructions issued (one per warp iteration)
  return err == cudaSuccess ? 0 : -2;
}
