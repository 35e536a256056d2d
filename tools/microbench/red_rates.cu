// Microbenchmark: scattered fp32 reductions (RED.ADD.F32) and scattered stores on B200.
//
// Question it answers: can the segmented pull PageRank fold its
// per-piece partial sums (one per (source segment, destination) pair, ~7.9 M
// per iteration on config 2) straight into an L2-resident accumulator s[n]
// with red.global.add.f32, instead of writing partials to HBM and merging them
// in a second pass? Pieces of one segment are emitted in destination order, so
// the addresses a warp reduces into are increasing with a mean gap g that
// depends on the segment's density (g ~ 2 for the hub segment, 10-1000 for the
// tail); g = "rand" is the uniform-random worst case.
//
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -o rr red_rates.cu
#include <cstdio>
#include <cstdint>
#include <cstdlib>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { \
  fprintf(stderr, "CUDA %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__); exit(1);} } while (0)

__host__ __device__ inline uint64_t mix64(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

// gap == 0: uniform random in [0, nx); else increasing ids with gaps uniform in [1, 2*gap-1], wrapped mod nx
__global__ void gen_idx(uint32_t* idx, int64_t m, uint32_t nx, int gap) {
  const int64_t per = 4096;  // each block of 4096 entries is an increasing run starting at a random id
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r * per < m; r += (int64_t)gridDim.x * blockDim.x) {
    uint64_t cur = mix64(r * 31 + 7) % nx;
    for (int64_t i = r * per; i < (r + 1) * per && i < m; ++i) {
      if (gap == 0) {
        idx[i] = (uint32_t)(mix64(i * 7919 + 17) % nx);
      } else {
        cur += 1 + mix64(i) % (2 * gap - 1);
        idx[i] = (uint32_t)(cur % nx);
      }
    }
  }
}

template <int OP>  // 0: red.add.f32, 1: st.f32, 2: ld (gather, for comparison)
__global__ void __launch_bounds__(512) scatter(const uint4* __restrict__ idx4, int64_t m4, float* __restrict__ s,
                                               float* out) {
  float acc = 0.f;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m4; i += (int64_t)gridDim.x * blockDim.x) {
    const uint4 v = __ldg(idx4 + i);
    const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      if (OP == 0) atomicAdd(s + w[k], 1.0f);
      else if (OP == 1) s[w[k]] = (float)w[k];
      else acc += __ldg(s + w[k]);
    }
  }
  if (OP == 2 && acc == -1.f) out[0] = acc;
}

int main() {
  cudaDeviceProp prop;
  CK(cudaGetDeviceProperties(&prop, 0));
  const int sms = prop.multiProcessorCount;
  printf("device %s SMs %d L2 %d MB\n", prop.name, sms, prop.l2CacheSize >> 20);
  const int64_t m = 1ll << 26;  // 64M ops
  uint32_t* idx;
  float *s, *out;
  CK(cudaMalloc(&idx, m * 4));
  CK(cudaMalloc(&s, (1ll << 25) * 4));
  CK(cudaMalloc(&out, 4));
  CK(cudaMemset(s, 0, (1ll << 25) * 4));
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
      best = ms < best ? ms : best;
    }
    CK(cudaGetLastError());
    return best;
  };
  const int grid = sms * 4;
  const uint32_t sizes[] = {1u << 22, 1u << 25};
  const int gaps[] = {0, 1, 2, 4, 16, 64, 1024};
  const char* ops[] = {"RED.ADD.F32", "STG scatter", "LDG gather"};
  for (uint32_t nx : sizes) {
    for (int gap : gaps) {
      gen_idx<<<sms * 4, 128>>>(idx, m, nx, gap);
      CK(cudaDeviceSynchronize());
      for (int op = 0; op < 3; ++op) {
        float ms;
        if (op == 0) ms = timeit([&] { scatter<0><<<grid, 512>>>((const uint4*)idx, m / 4, s, out); });
        else if (op == 1) ms = timeit([&] { scatter<1><<<grid, 512>>>((const uint4*)idx, m / 4, s, out); });
        else ms = timeit([&] { scatter<2><<<grid, 512>>>((const uint4*)idx, m / 4, s, out); });
        const double rate = m / (ms * 1e-3);
        char g[16];
        if (gap) snprintf(g, sizeof g, "%d", gap); else snprintf(g, sizeof g, "rand");
        printf("%-12s nx=%9u (%4u MB) gap=%-5s %8.3f ms %8.1f Gops/s %6.2f ops/clk/SM@1.9GHz\n", ops[op], nx,
               (unsigned)((uint64_t)nx * 4 >> 20), g, ms, rate / 1e9, rate / (sms * 1.9e9));
      }
    }
  }
  printf("done\n");
  return 0;
}
