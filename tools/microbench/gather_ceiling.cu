// Ceiling microbenchmarks for the RSOC tentative-color kernel (SURVEY.md §7 hard part 8).
//
//  (1) coalesced int4 streaming from HBM (the CSR `cols` stream)
//  (2) random 4-byte gathers into a colors array of varying size, with the
//      index stream itself read coalesced from HBM (exactly the K1 access
//      pattern: cols[e] streamed, colors[cols[e]] gathered)
//
// Standalone: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o gather_ceiling gather_ceiling.cu
// Prints one line per case: bytes moved / time, gathers per second.
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  std::fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); std::exit(1);} } while (0)

__device__ __forceinline__ uint64_t evict_first_policy() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}

__device__ __forceinline__ int4 ld_stream(const int4* a, uint64_t pol) {
  int4 r;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.s32 {%0,%1,%2,%3}, [%4], %5;"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(a), "l"(pol));
  return r;
}

__device__ __forceinline__ int ld_relaxed(const int* p) {
  int r;
  asm volatile("ld.relaxed.gpu.global.b32 %0, [%1];" : "=r"(r) : "l"(p) : "memory");
  return r;
}

__global__ void stream_kernel(const int4* __restrict__ a, size_t n4, unsigned* out) {
  const uint64_t pol = evict_first_policy();
  unsigned acc = 0;
  size_t stride = (size_t)gridDim.x * blockDim.x;
  size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  for (; i + 3 * stride < n4; i += 4 * stride) {
    int4 x0 = ld_stream(a + i, pol), x1 = ld_stream(a + i + stride, pol);
    int4 x2 = ld_stream(a + i + 2 * stride, pol), x3 = ld_stream(a + i + 3 * stride, pol);
    acc ^= x0.x ^ x0.y ^ x0.z ^ x0.w ^ x1.x ^ x1.y ^ x1.z ^ x1.w;
    acc ^= x2.x ^ x2.y ^ x2.z ^ x2.w ^ x3.x ^ x3.y ^ x3.z ^ x3.w;
  }
  for (; i < n4; i += stride) { int4 x = ld_stream(a + i, pol); acc ^= x.x ^ x.y ^ x.z ^ x.w; }
  if (acc == 0x12345678u) out[0] = acc;
}

// MODE 0: ld.relaxed.gpu  MODE 1: ld.global.cg  MODE 2: default (L1-cached) ld
template <int MODE>
__device__ __forceinline__ int gather1(const int* colors, int w) {
  if (MODE == 0) return ld_relaxed(colors + w);
  if (MODE == 1) return __ldcg(colors + w);
  return colors[w];
}

template <int MODE>
__global__ void gather_kernel(const int4* __restrict__ idx, size_t n4, const int* colors, unsigned* out) {
  const uint64_t pol = evict_first_policy();
  unsigned acc = 0;
  size_t stride = (size_t)gridDim.x * blockDim.x;
  size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  for (; i + stride < n4; i += 2 * stride) {
    int4 a = ld_stream(idx + i, pol), b = ld_stream(idx + i + stride, pol);
    int c0 = gather1<MODE>(colors, a.x), c1 = gather1<MODE>(colors, a.y);
    int c2 = gather1<MODE>(colors, a.z), c3 = gather1<MODE>(colors, a.w);
    int c4 = gather1<MODE>(colors, b.x), c5 = gather1<MODE>(colors, b.y);
    int c6 = gather1<MODE>(colors, b.z), c7 = gather1<MODE>(colors, b.w);
    acc |= (1u << (c0 & 31)) | (1u << (c1 & 31)) | (1u << (c2 & 31)) | (1u << (c3 & 31));
    acc |= (1u << (c4 & 31)) | (1u << (c5 & 31)) | (1u << (c6 & 31)) | (1u << (c7 & 31));
  }
  for (; i < n4; i += stride) {
    int4 a = ld_stream(idx + i, pol);
    acc |= (1u << (gather1<MODE>(colors, a.x) & 31)) | (1u << (gather1<MODE>(colors, a.y) & 31));
    acc |= (1u << (gather1<MODE>(colors, a.z) & 31)) | (1u << (gather1<MODE>(colors, a.w) & 31));
  }
  if (acc == 0x12345678u) out[0] = acc;
}

__global__ void fill_idx(int* idx, size_t n, uint32_t range, uint64_t seed) {
  size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  for (; i < n; i += (size_t)gridDim.x * blockDim.x) {
    uint64_t z = seed + i * 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    z ^= z >> 31;
    idx[i] = (int)((z >> 32) % range);
  }
}

__global__ void fill_colors(int* c, size_t n) {
  size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  for (; i < n; i += (size_t)gridDim.x * blockDim.x) c[i] = (int)(i % 29);
}

int main(int argc, char** argv) {
  int dev = 0;
  CK(cudaSetDevice(dev));
  cudaDeviceProp prop;
  CK(cudaGetDeviceProperties(&prop, dev));
  const int sms = prop.multiProcessorCount;
  std::printf("device %s sms %d l2 %d MB\n", prop.name, sms, prop.l2CacheSize >> 20);
  unsigned* out;
  CK(cudaMalloc(&out, 64));
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));

  // (1) streaming
  const size_t stream_bytes = size_t(4) << 30;
  int4* big;
  CK(cudaMalloc(&big, stream_bytes));
  CK(cudaMemset(big, 1, stream_bytes));
  for (int bps : {4, 8, 16}) {
    int grid = sms * bps;
    float best = 1e9f;
    for (int it = 0; it < 6; ++it) {
      CK(cudaEventRecord(e0));
      stream_kernel<<<grid, 256>>>(big, stream_bytes / 16, out);
      CK(cudaEventRecord(e1));
      CK(cudaEventSynchronize(e1));
      float ms;
      CK(cudaEventElapsedTime(&ms, e0, e1));
      if (it > 0 && ms < best) best = ms;
    }
    std::printf("stream int4 grid=%d: %.1f GB/s\n", grid, stream_bytes / (best * 1e-3) / 1e9);
  }

  // (2) gathers: index stream of 1 Gi... 256 Mi indices (1 GiB), colors of varying size
  const size_t nidx = size_t(256) << 20;
  int* idx = reinterpret_cast<int*>(big);  // reuse
  int* colors;
  const size_t max_colors = size_t(134217728);
  CK(cudaMalloc(&colors, max_colors * 4));
  fill_colors<<<sms * 8, 256>>>(colors, max_colors);
  for (size_t ncol : {size_t(1) << 20, size_t(4) << 20, size_t(16) << 20, size_t(32) << 20,
                      size_t(64) << 20, max_colors}) {
    fill_idx<<<sms * 8, 256>>>(idx, nidx, (uint32_t)ncol, 12345);
    CK(cudaDeviceSynchronize());
    for (int mode = 0; mode < 3; ++mode) {
      for (int bps : {8, 16}) {
        int grid = sms * bps;
        float best = 1e9f;
        for (int it = 0; it < 5; ++it) {
          CK(cudaEventRecord(e0));
          if (mode == 0) gather_kernel<0><<<grid, 256>>>((const int4*)idx, nidx / 4, colors, out);
          if (mode == 1) gather_kernel<1><<<grid, 256>>>((const int4*)idx, nidx / 4, colors, out);
          if (mode == 2) gather_kernel<2><<<grid, 256>>>((const int4*)idx, nidx / 4, colors, out);
          CK(cudaEventRecord(e1));
          CK(cudaEventSynchronize(e1));
          float ms;
          CK(cudaEventElapsedTime(&ms, e0, e1));
          if (it > 0 && ms < best) best = ms;
        }
        double gps = nidx / (best * 1e-3) / 1e9;
        std::printf("gather colors=%zu MB mode=%d grid=%d: %.1f Ggathers/s  algo %.1f GB/s (idx+gather 8 B)\n",
                    ncol * 4 >> 20, mode, grid, gps, gps * 8);
      }
    }
  }
  CK(cudaGetLastError());
  std::printf("done\n");
  return 0;
}
