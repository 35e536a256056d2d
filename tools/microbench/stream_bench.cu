// Microbenchmark: streaming the segmented-pull index layout (1 KB per
// 512-slot chunk, warp-interleaved chunks inside a persistent CTA per SM) —
// which load form and how many chunks in flight per warp reach HBM bandwidth.
//
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -o sb stream_bench.cu
#include <cstdio>
#include <cstdint>
#include <cstdlib>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { \
  fprintf(stderr, "CUDA %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__); exit(1);} } while (0)

constexpr int kChunkU4 = 64;  // 1 KB

template <int LD>
__device__ __forceinline__ void ld32(const uint4* p, uint4& a, uint4& b) {
  if (LD == 0) {
    asm volatile("ld.global.nc.L1::no_allocate.L2::evict_first.v8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
                 : "=r"(a.x), "=r"(a.y), "=r"(a.z), "=r"(a.w), "=r"(b.x), "=r"(b.y), "=r"(b.z), "=r"(b.w)
                 : "l"(p));
  } else if (LD == 1) {
    a = __ldg(p);
    b = __ldg(p + 1);
  } else if (LD == 2) {
    asm volatile("ld.global.v8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
                 : "=r"(a.x), "=r"(a.y), "=r"(a.z), "=r"(a.w), "=r"(b.x), "=r"(b.y), "=r"(b.z), "=r"(b.w)
                 : "l"(p));
  } else {
    asm("ld.global.nc.L1::no_allocate.L2::evict_first.v8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
        : "=r"(a.x), "=r"(a.y), "=r"(a.z), "=r"(a.w), "=r"(b.x), "=r"(b.y), "=r"(b.z), "=r"(b.w)
        : "l"(p));
  }
}

template <int LD, int DEPTH>
__global__ void __launch_bounds__(1024, 1) stream(const uint4* __restrict__ idx, int C, uint32_t* out) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, NW = blockDim.x >> 5;
  const int per = (C + gridDim.x - 1) / gridDim.x;
  const int c0 = blockIdx.x * per, c1 = min(C, c0 + per);
  uint32_t x = 0;
  uint4 a[DEPTH], b[DEPTH];
#pragma unroll
  for (int d = 0; d < DEPTH; ++d)
    if (c0 + warp + d * NW < c1) ld32<LD>(idx + (int64_t)(c0 + warp + d * NW) * kChunkU4 + 2 * lane, a[d], b[d]);
  for (int c = c0 + warp; c < c1; c += DEPTH * NW) {
#pragma unroll
    for (int d = 0; d < DEPTH; ++d) {
      const int cc = c + d * NW;
      if (cc < c1) {
        x ^= a[d].x ^ a[d].y ^ a[d].z ^ a[d].w ^ b[d].x ^ b[d].y ^ b[d].z ^ b[d].w;
        const int cn = cc + DEPTH * NW;
        if (cn < c1) ld32<LD>(idx + (int64_t)cn * kChunkU4 + 2 * lane, a[d], b[d]);
      }
    }
  }
  if (x == 0x12345678u) out[0] = x;
}

int main() {
  cudaDeviceProp prop;
  CK(cudaGetDeviceProperties(&prop, 0));
  const int sms = prop.multiProcessorCount;
  const int C = 127445 * 2;  // 2x config 2's chunk count: 261 MB
  uint4* idx;
  uint32_t* out;
  CK(cudaMalloc(&idx, (size_t)C * kChunkU4 * 16));
  CK(cudaMemset(idx, 1, (size_t)C * kChunkU4 * 16));
  CK(cudaMalloc(&out, 4));
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  int gmul = 1;
  auto run = [&](const char* name, auto kern, int threads) {
    float best = 1e30f;
    for (int r = 0; r < 5; ++r) {
      CK(cudaEventRecord(e0));
      kern<<<sms * gmul, threads>>>(idx, C, out);
      CK(cudaEventRecord(e1));
      CK(cudaEventSynchronize(e1));
      float ms;
      CK(cudaEventElapsedTime(&ms, e0, e1));
      best = ms < best ? ms : best;
    }
    CK(cudaGetLastError());
    printf("%-40s grid=%dxSM thr=%4d %8.2f us %8.1f GB/s\n", name, gmul, threads, best * 1e3, (double)C * 1024 / (best * 1e-3) / 1e9);
  };
  for (int gm : {1, 2, 4}) {
    gmul = gm;
    for (int thr : {256, 512, 1024}) {
      run("v8.nc.evict_first depth1", stream<0, 1>, thr);
      run("v8.nc.evict_first depth2", stream<0, 2>, thr);
      run("2x ldg.128 depth2", stream<1, 2>, thr);
    }
  }
  return 0;
}
