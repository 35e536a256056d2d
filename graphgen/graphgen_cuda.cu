// graphgen_cuda.cu — the same counter-based RMAT generator as graphgen.c, on
// the GPU (input infrastructure for the billion-edge configs; no method
// arithmetic). Edge i of the stream is a pure function of (seed, i): for each
// bit level l (most significant first) u = U(seed, i*64 + l), quadrant
// a -> (0,0), b -> (0,1), c -> (1,0), d -> (1,1). Both implementations use the
// same 64-bit mixer and the same double comparisons, so they emit identical
// edges (tests/test_gpu_scale.py checks a window).
#include <cstdint>

namespace {

__host__ __device__ inline uint64_t mix64(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

__device__ inline double unif(uint64_t key, uint64_t ctr) {
  return (double)(mix64(key + ctr) >> 11) * (1.0 / 9007199254740992.0);
}

__global__ void k_rmat(int scale, double a, double ab, double abc, uint64_t key, int64_t first, int64_t count,
                       int32_t* __restrict__ src, int32_t* __restrict__ dst) {
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < count; j += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t i = (uint64_t)(first + j);
    uint32_t s = 0, d = 0;
    for (int l = 0; l < scale; ++l) {
      const double u = unif(key, i * 64u + (uint64_t)l);
      uint32_t sb, db;
      if (u < a) { sb = 0; db = 0; }
      else if (u < ab) { sb = 0; db = 1; }
      else if (u < abc) { sb = 1; db = 0; }
      else { sb = 1; db = 1; }
      s = (s << 1) | sb;
      d = (d << 1) | db;
    }
    src[j] = (int32_t)s;
    dst[j] = (int32_t)d;
  }
}

}  // namespace

extern "C" __attribute__((visibility("default"))) int gg_rmat_device(int scale, double a, double b, double c,
                                                                      uint64_t seed, int64_t first, int64_t count,
                                                                      int32_t* src, int32_t* dst, void* stream) {
  if (count <= 0) return 0;
  k_rmat<<<148 * 16, 256, 0, (cudaStream_t)stream>>>(scale, a, a + b, a + b + c, mix64(seed), first, count, src, dst);
  return (int)cudaStreamSynchronize((cudaStream_t)stream);
}
