// Microbenchmark: global RED.ADD throughput by access pattern (tools/, not product).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o red_bench red_bench.cu
// Each thread issues ITERS reductions; the table is larger than L2 so the
// fills / write-backs of a count table that does not fit L2 are included.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

constexpr int ITERS = 16;

// pattern 0: lane-consecutive keys (a warp covers 32 consecutive entries)
// pattern 1: per-lane stride 8 keys (C2-like: 16 work-items x 2 lanes)
// pattern 2: random keys (hash)
template <typename T>
__global__ void red_kernel(T* tab, uint64_t n_keys, int pattern, uint64_t total) {
  const uint64_t tid = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const uint64_t nthreads = (uint64_t)gridDim.x * blockDim.x;
  for (int i = 0; i < ITERS; ++i) {
    const uint64_t e = (uint64_t)i * nthreads + tid;  // event index
    if (e >= total) break;
    uint64_t key;
    if (pattern == 0) key = e;
    else if (pattern == 1) key = ((e / 32) * 32) + ((e % 32) * 8) % 256 + (e % 256) / 32;
    else { uint64_t x = e * 0x9E3779B97F4A7C15ull; x ^= x >> 29; key = x; }
    key %= n_keys;
    atomicAdd(&tab[key], (T)1);
  }
}

// two REDs per event on the same word (count + flag)
__global__ void red2_kernel(unsigned* tab, uint64_t n_keys, uint64_t total) {
  const uint64_t tid = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const uint64_t nthreads = (uint64_t)gridDim.x * blockDim.x;
  for (int i = 0; i < ITERS; ++i) {
    const uint64_t e = (uint64_t)i * nthreads + tid;
    if (e >= total) break;
    const uint64_t key = e % n_keys;
    atomicAdd(&tab[key], 1u);
    atomicOr(&tab[key], 1u << 30);
  }
}

int main() {
  const uint64_t n_keys = 75497472;  // C2 table
  const uint64_t total = n_keys;
  void* tab;
  cudaMalloc(&tab, n_keys * 8);
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  const int threads = 256;
  const uint64_t blocks = (total + (uint64_t)threads * ITERS - 1) / ((uint64_t)threads * ITERS);
  for (int bits = 32; bits <= 64; bits += 32) {
    for (int pat = 0; pat < 3; ++pat) {
      float best = 1e9f;
      for (int rep = 0; rep < 5; ++rep) {
        cudaMemsetAsync(tab, 0, n_keys * (bits / 8));
        cudaEventRecord(a);
        if (bits == 32) red_kernel<unsigned><<<blocks, threads>>>((unsigned*)tab, n_keys, pat, total);
        else red_kernel<unsigned long long><<<blocks, threads>>>((unsigned long long*)tab, n_keys, pat, total);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b);
        if (ms < best) best = ms;
      }
      printf("RED.%d pattern %d: %.3f ms  %.1f G red/s\n", bits, pat, best, total / (best * 1e6));
    }
  }
  {
    float best = 1e9f;
    for (int rep = 0; rep < 5; ++rep) {
      cudaMemsetAsync(tab, 0, n_keys * 4);
      cudaEventRecord(a);
      red2_kernel<<<blocks, threads>>>((unsigned*)tab, n_keys, total);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b);
      if (ms < best) best = ms;
    }
    printf("RED.32 add+or pattern 0: %.3f ms  %.1f G events/s\n", best, total / (best * 1e6));
  }
  {
    float best = 1e9f;
    for (int rep = 0; rep < 5; ++rep) {
      cudaEventRecord(a);
      cudaMemsetAsync(tab, 0, n_keys * 8);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b);
      if (ms < best) best = ms;
    }
    printf("memset %llu MB: %.3f ms  %.0f GB/s\n", (unsigned long long)(n_keys * 8 >> 20), best, n_keys * 8 / (best * 1e6));
  }
  cudaError_t e = cudaGetLastError();
  printf("status: %s\n", cudaGetErrorString(e));
  return 0;
}
