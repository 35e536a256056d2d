// Microbenchmark: random 4-byte gather throughput on B200 (sm_100a).
//
// Question it answers: how many
// random fp32 gathers per SM-clock can the pull PageRank edge pass expect
// from (a) LDG through L1/L2, (b) ld.global.nc, (c) shared memory,
// (d) distributed shared memory in a cluster — against the 2.2 edges/clk/SM
// that 50% of the HBM roofline needs at config 2.
//
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -o gr gather_rates.cu
#include <cooperative_groups.h>
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <vector>
namespace cg = cooperative_groups;

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { \
  fprintf(stderr, "CUDA %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__); exit(1);} } while (0)

__host__ __device__ inline uint64_t mix64(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

// skew = 0: uniform in [0, 2^bits); skew = 1: each bit set with p = 0.24
// (the RMAT a=.57,b=.19,c=.19,d=.05 source marginal).
__global__ void gen_idx(uint32_t* idx, int64_t m, int bits, int skew, uint32_t limit) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m;
       i += (int64_t)gridDim.x * blockDim.x) {
    uint32_t v = 0;
    if (!skew) {
      v = (uint32_t)(mix64(i * 7919 + 17) >> 20) & ((1u << bits) - 1);
    } else {
      for (int b = 0; b < bits; ++b) {
        uint64_t h = mix64((uint64_t)i * 64 + b);
        double u = (h >> 11) * (1.0 / 9007199254740992.0);
        v = (v << 1) | (u < 0.24 ? 1u : 0u);
      }
    }
    idx[i] = v % limit;
  }
}

__global__ void init_x(float* x, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) x[i] = 1.0f + (i & 7);
}

template <int MODE>
__device__ __forceinline__ float ldx(const float* p) {
  float r;
  if (MODE == 0) r = *p;
  else if (MODE == 1) asm volatile("ld.global.nc.f32 %0, [%1];" : "=f"(r) : "l"(p));
  else asm volatile("ld.global.cg.f32 %0, [%1];" : "=f"(r) : "l"(p));
  return r;
}

// streaming idx (uint4) + gather x[idx]
template <int MODE>
__global__ void __launch_bounds__(512) gather_global(const uint4* __restrict__ idx4, int64_t m4,
                                                     const float* __restrict__ x, float* out) {
  float acc = 0.f;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m4;
       i += (int64_t)gridDim.x * blockDim.x) {
    uint4 v = __ldg(idx4 + i);
    acc += ldx<MODE>(x + v.x) + ldx<MODE>(x + v.y) + ldx<MODE>(x + v.z) + ldx<MODE>(x + v.w);
  }
  if (acc == -1.f) out[0] = acc;
}

// stream only
__global__ void __launch_bounds__(512) stream_only(const uint4* __restrict__ idx4, int64_t m4, float* out) {
  uint32_t acc = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m4;
       i += (int64_t)gridDim.x * blockDim.x) {
    uint4 v = __ldg(idx4 + i);
    acc ^= v.x ^ v.y ^ v.z ^ v.w;
  }
  if (acc == 0xFFFFFFFFu) out[0] = 1.f;
}

// shared-memory gather: x segment of SEG floats staged in smem; idx taken mod SEG
__global__ void __launch_bounds__(1024) gather_smem(const uint4* __restrict__ idx4, int64_t m4,
                                                    const float* __restrict__ x, int seg, float* out) {
  extern __shared__ float sx[];
  for (int i = threadIdx.x; i < seg; i += blockDim.x) sx[i] = x[i];
  __syncthreads();
  float acc = 0.f;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m4;
       i += (int64_t)gridDim.x * blockDim.x) {
    uint4 v = __ldg(idx4 + i);
    acc += sx[v.x % seg] + sx[v.y % seg] + sx[v.z % seg] + sx[v.w % seg];
  }
  if (acc == -1.f) out[0] = acc;
}

// 16-bit index variant, smem segment of 65536 max: idx pairs packed in uint32
__global__ void __launch_bounds__(1024) gather_smem16(const uint4* __restrict__ idx4, int64_t m4,
                                                      const float* __restrict__ x, int seg, float* out) {
  extern __shared__ float sx[];
  for (int i = threadIdx.x; i < seg; i += blockDim.x) sx[i] = x[i];
  __syncthreads();
  float acc = 0.f;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m4;
       i += (int64_t)gridDim.x * blockDim.x) {
    uint4 v = __ldg(idx4 + i);
    uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int k = 0; k < 4; ++k) acc += sx[(w[k] & 0xFFFF) % seg] + sx[(w[k] >> 16) % seg];
  }
  if (acc == -1.f) out[0] = acc;
}

// DSMEM gather across a cluster of CS CTAs, each holding seg floats
template <int CS>
__global__ void __launch_bounds__(1024) gather_dsmem(const uint4* __restrict__ idx4, int64_t m4,
                                                     const float* __restrict__ x, int seg, float* out) {
  extern __shared__ float sx[];
  cg::cluster_group cl = cg::this_cluster();
  int rank = cl.block_rank();
  for (int i = threadIdx.x; i < seg; i += blockDim.x) sx[i] = x[rank * seg + i];
  cl.sync();
  float* rem[CS];
#pragma unroll
  for (int r = 0; r < CS; ++r) rem[r] = cl.map_shared_rank(sx, r);
  float acc = 0.f;
  uint32_t tot = (uint32_t)seg * CS;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m4;
       i += (int64_t)gridDim.x * blockDim.x) {
    uint4 v = __ldg(idx4 + i);
    uint32_t w[4] = {v.x % tot, v.y % tot, v.z % tot, v.w % tot};
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      uint32_t r = w[k] / seg, o = w[k] - r * seg;
      float* base = sx;
#pragma unroll
      for (int q = 0; q < CS; ++q) if (q == (int)r) base = rem[q];
      acc += base[o];
    }
  }
  cl.sync();
  if (acc == -1.f) out[0] = acc;
}

int main(int argc, char** argv) {
  int dev = 0;
  CK(cudaSetDevice(dev));
  cudaDeviceProp prop;
  CK(cudaGetDeviceProperties(&prop, dev));
  int sms = prop.multiProcessorCount;
  int clk_khz = 0;
  CK(cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, dev));
  printf("device %s SMs %d clock %d MHz L2 %d MB smem/block optin %zu\n", prop.name, sms,
         clk_khz / 1000, prop.l2CacheSize >> 20, prop.sharedMemPerBlockOptin);
  const int64_t m = 1ll << 28;  // 268M indices = 1 GiB
  uint32_t* idx;
  float *x, *out;
  const int64_t nx = 1ll << 26;  // 64M floats = 256 MB
  CK(cudaMalloc(&idx, m * 4));
  CK(cudaMalloc(&x, nx * 4));
  CK(cudaMalloc(&out, 4));
  init_x<<<sms * 8, 256>>>(x, nx);
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  auto timeit = [&](auto fn) {
    fn();
    CK(cudaDeviceSynchronize());
    float best = 1e30f;
    for (int r = 0; r < 5; ++r) {
      CK(cudaEventRecord(e0));
      fn();
      CK(cudaEventRecord(e1));
      CK(cudaEventSynchronize(e1));
      float ms;
      CK(cudaEventElapsedTime(&ms, e0, e1));
      if (ms < best) best = ms;
    }
    CK(cudaGetLastError());
    return best;
  };
  // nominal SM clock under load ~ 1.9 GHz; report per-SM-per-ns and per-clk at 1.9 GHz
  auto report = [&](const char* name, float ms, double items, double bytes) {
    double rate = items / (ms * 1e-3);
    printf("%-44s %8.3f ms  %8.2f Gitems/s  %6.2f items/clk/SM@1.9GHz  %8.1f GB/s\n", name, ms,
           rate / 1e9, rate / (sms * 1.9e9), bytes / (ms * 1e-3) / 1e9);
  };
  int grid = sms * 4;
  struct Dist { const char* name; int bits; int skew; uint32_t limit; };
  Dist dists[] = {
      {"uniform 4M (16MB, L2)", 22, 0, 1u << 22},
      {"rmat-skew 4M (16MB, L2)", 22, 1, 1u << 22},
      {"uniform 32M (128MB)", 25, 0, 1u << 25},
      {"rmat-skew 32M (128MB)", 25, 1, 1u << 25},
      {"uniform 64M (256MB, HBM)", 26, 0, 1u << 26},
      {"uniform 64K (256KB)", 16, 0, 1u << 16},
  };
  {
    gen_idx<<<sms * 8, 256>>>(idx, m, 22, 0, 1u << 22);
    float ms = timeit([&] { stream_only<<<grid, 512>>>((const uint4*)idx, m / 4, out); });
    report("stream idx only (1 GiB)", ms, (double)m, (double)m * 4);
  }
  for (auto& d : dists) {
    gen_idx<<<sms * 8, 256>>>(idx, m, d.bits, d.skew, d.limit);
    CK(cudaDeviceSynchronize());
    char nm[128];
    for (int mode = 0; mode < 3; ++mode) {
      float ms;
      if (mode == 0) ms = timeit([&] { gather_global<0><<<grid, 512>>>((const uint4*)idx, m / 4, x, out); });
      else if (mode == 1) ms = timeit([&] { gather_global<1><<<grid, 512>>>((const uint4*)idx, m / 4, x, out); });
      else ms = timeit([&] { gather_global<2><<<grid, 512>>>((const uint4*)idx, m / 4, x, out); });
      snprintf(nm, sizeof nm, "LDG%s %s", mode == 0 ? "" : mode == 1 ? ".nc" : ".cg", d.name);
      report(nm, ms, (double)m, (double)m * 4);
    }
  }
  // shared memory
  gen_idx<<<sms * 8, 256>>>(idx, m, 22, 0, 1u << 22);
  CK(cudaDeviceSynchronize());
  for (int seg : {16384, 49152, 56320}) {
    size_t sm = (size_t)seg * 4;
    CK(cudaFuncSetAttribute(gather_smem, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
    CK(cudaFuncSetAttribute(gather_smem16, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
    char nm[128];
    float ms = timeit([&] { gather_smem<<<sms, 1024, sm>>>((const uint4*)idx, m / 4, x, seg, out); });
    snprintf(nm, sizeof nm, "LDS seg=%d 32b idx", seg);
    report(nm, ms, (double)m, (double)m * 4);
    ms = timeit([&] { gather_smem16<<<sms, 1024, sm>>>((const uint4*)idx, m / 4, x, seg, out); });
    snprintf(nm, sizeof nm, "LDS seg=%d 16b idx", seg);
    report(nm, ms, (double)m * 2, (double)m * 4);
  }
  // DSMEM
  {
    int seg = 49152;
    size_t sm = (size_t)seg * 4;
    CK(cudaFuncSetAttribute(gather_dsmem<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((sms / 8) * 8);
    cfg.blockDim = dim3(1024);
    cfg.dynamicSmemBytes = sm;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = 8; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
    cfg.attrs = at; cfg.numAttrs = 1;
    float ms = timeit([&] {
      CK(cudaLaunchKernelEx(&cfg, gather_dsmem<8>, (const uint4*)idx, (int64_t)(m / 4), (const float*)x, seg, out));
    });
    report("DSMEM cluster8 seg=49152", ms, (double)m, (double)m * 4);
  }
  printf("done\n");
  return 0;
}
