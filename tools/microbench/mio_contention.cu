// Does warp-shuffle / shared-memory work compete with random global gathers
// for the L1 (tag) pipe?  Gathers from an L2-resident array with, per
// gather, K extra shuffles (MODE 1), K shared-memory atomics (MODE 2) or
// none (MODE 0).  Prints gathers/s.  Tooling for the K1W design.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mio mio_contention.cu
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  std::fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); std::exit(1);} } while (0)

__device__ __forceinline__ int ld_relaxed(const int* p) {
  int r;
  asm volatile("ld.relaxed.gpu.global.b32 %0, [%1];" : "=r"(r) : "l"(p) : "memory");
  return r;
}

template <int MODE, int K>
__global__ void __launch_bounds__(256) k(const int* __restrict__ idx, size_t n, const int* colors,
                                         unsigned* out) {
  __shared__ unsigned sm[256];
  sm[threadIdx.x] = 0;
  __syncthreads();
  unsigned acc = 0;
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i + 3 * stride < n; i += 4 * stride) {
    int c[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) c[u] = ld_relaxed(colors + __ldg(idx + i + u * stride));
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      unsigned x = 1u << (c[u] & 31);
      if (MODE == 1) {
#pragma unroll
        for (int s = 0; s < K; ++s) x |= __shfl_xor_sync(0xffffffffu, x, 1 << s);
      } else if (MODE == 2) {
#pragma unroll
        for (int s = 0; s < K; ++s) atomicOr(&sm[(threadIdx.x + 37 * s + (x & 7)) & 255], x);
      }
      acc |= x;
    }
  }
  if (MODE == 2) { __syncthreads(); acc |= sm[threadIdx.x]; }
  if (acc == 0x12345678u) out[0] = acc;
}

template <int MODE, int K>
void run(const int* idx, size_t n, const int* colors, unsigned* out, int grid) {
  cudaEvent_t a, b;
  CK(cudaEventCreate(&a)); CK(cudaEventCreate(&b));
  k<MODE, K><<<grid, 256>>>(idx, n, colors, out);
  CK(cudaEventRecord(a));
  for (int r = 0; r < 5; ++r) k<MODE, K><<<grid, 256>>>(idx, n, colors, out);
  CK(cudaEventRecord(b));
  CK(cudaEventSynchronize(b));
  float ms; CK(cudaEventElapsedTime(&ms, a, b));
  std::printf("mode %d K %d grid %d: %.1f G gathers/s\n", MODE, K, grid, 5.0 * n / (ms * 1e-3) / 1e9);
}

__global__ void fill_idx(int* idx, size_t n, int range) {
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    unsigned long long x = i * 0x9E3779B97F4A7C15ull; x ^= x >> 29; x *= 0xBF58476D1CE4E5B9ull; x ^= x >> 32;
    idx[i] = (int)(x % (unsigned long long)range);
  }
}

int main() {
  const size_t n = 1 << 26;
  const int range = 4 << 20;  // 16 MB of colours: L2-resident
  int *idx, *colors; unsigned* out;
  CK(cudaMalloc(&idx, n * 4)); CK(cudaMalloc(&colors, range * 4)); CK(cudaMalloc(&out, 4));
  fill_idx<<<1184, 256>>>(idx, n, range);
  CK(cudaMemset(colors, 0, range * 4));
  CK(cudaDeviceSynchronize());
  const int grid = 148 * 8;
  run<0, 0>(idx, n, colors, out, grid);
  run<1, 1>(idx, n, colors, out, grid);
  run<1, 2>(idx, n, colors, out, grid);
  run<1, 5>(idx, n, colors, out, grid);
  run<2, 1>(idx, n, colors, out, grid);
  run<2, 2>(idx, n, colors, out, grid);
  std::printf("done\n");
  return 0;
}
