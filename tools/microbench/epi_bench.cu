// Microbenchmark: the PageRank vertex update (a3) as a stand-alone streaming
// kernel over n = 4M vertices (config 2): read acc[n] + outdeg[n], write
// contrib[n] (+ acc reset). Variants isolate what costs time: the reset
// store, the IEEE division, the fp64 dangling sum, and the grid size.
//
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -o eb epi_bench.cu
#include <cstdio>
#include <cstdint>
#include <cstdlib>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { \
  fprintf(stderr, "CUDA %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__); exit(1);} } while (0)

template <int V>  // 0 full, 1 no reset, 2 no division (mul by rcp), 3 copy only
__global__ void __launch_bounds__(256) epi(float* __restrict__ acc, const int* __restrict__ outdeg,
                                           float* __restrict__ out, int64_t n, double* dsum) {
  double dpart = 0.0;
  const int64_t nq = n / 4;
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < nq; q += (int64_t)gridDim.x * blockDim.x) {
    const float4 s4 = reinterpret_cast<const float4*>(acc)[q];
    if (V != 1 && V != 3) reinterpret_cast<float4*>(acc)[q] = make_float4(0.f, 0.f, 0.f, 0.f);
    if (V == 3) {
      reinterpret_cast<float4*>(out)[q] = s4;
      continue;
    }
    const int4 od4 = __ldg(reinterpret_cast<const int4*>(outdeg) + q);
    const float s[4] = {s4.x, s4.y, s4.z, s4.w};
    const int od[4] = {od4.x, od4.y, od4.z, od4.w};
    float c[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const float rn = 0.15f / n + 0.85f * s[k];
      if (V == 2) c[k] = od[k] > 0 ? rn * __frcp_rn((float)od[k]) : 0.f;
      else c[k] = od[k] > 0 ? rn / (float)od[k] : 0.f;
      if (od[k] == 0) dpart += (double)rn;
    }
    reinterpret_cast<float4*>(out)[q] = make_float4(c[0], c[1], c[2], c[3]);
  }
  // block reduction, one atomic per block (as k_pr_acc)
  __shared__ double sred[8];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) dpart += __shfl_xor_sync(0xffffffffu, dpart, o);
  if ((threadIdx.x & 31) == 0) sred[threadIdx.x >> 5] = dpart;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < 8; ++w) t += sred[w];
    if (t != 0.0) atomicAdd(dsum, t);
  }
}

__global__ void init(float* acc, int* od, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    acc[i] = 1e-7f * (i & 1023);
    od[i] = (int)((i * 2654435761u) >> 28) % 5;
  }
}

int main() {
  cudaDeviceProp prop;
  CK(cudaGetDeviceProperties(&prop, 0));
  const int sms = prop.multiProcessorCount;
  const int64_t n = 1 << 22;
  float *acc, *out;
  int* od;
  double* ds;
  CK(cudaMalloc(&acc, n * 4));
  CK(cudaMalloc(&out, n * 4));
  CK(cudaMalloc(&od, n * 4));
  CK(cudaMalloc(&ds, 8));
  init<<<sms * 8, 256>>>(acc, od, n);
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  // big buffer to flush L2 between runs
  char* flush;
  const size_t fb = 512ull << 20;
  CK(cudaMalloc(&flush, fb));
  const char* names[] = {"full", "no-reset", "rcp", "copy"};
  for (int v = 0; v < 4; ++v) {
    for (int per_sm : {2, 8, 16, 64}) {
      for (int cold = 0; cold < 2; ++cold) {
        const int grid = sms * per_sm;
        float best = 1e30f;
        for (int r = 0; r < 5; ++r) {
          if (cold) CK(cudaMemsetAsync(flush, r, fb));
          CK(cudaEventRecord(e0));
          if (v == 0) epi<0><<<grid, 256>>>(acc, od, out, n, ds);
          if (v == 1) epi<1><<<grid, 256>>>(acc, od, out, n, ds);
          if (v == 2) epi<2><<<grid, 256>>>(acc, od, out, n, ds);
          if (v == 3) epi<3><<<grid, 256>>>(acc, od, out, n, ds);
          CK(cudaEventRecord(e1));
          CK(cudaEventSynchronize(e1));
          float ms;
          CK(cudaEventElapsedTime(&ms, e0, e1));
          best = ms < best ? ms : best;
        }
        const double bytes = v == 3 ? 8.0 * n : (v == 1 ? 12.0 * n : 16.0 * n);
        printf("%-9s grid=%3d/SM %-4s %8.2f us  %7.1f GB/s\n", names[v], per_sm, cold ? "cold" : "warm", best * 1e3,
               bytes / (best * 1e-3) / 1e9);
      }
    }
  }
  return 0;
}
