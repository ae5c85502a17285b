// Do IMAD (fmaheavy pipe) and DFMA (fp64 pipe) issue concurrently on sm_100a? Times an IMAD-only,
// a DFMA-only and a 1:1 interleaved loop of independent chains (8 per type per thread).
#include <cstdio>
#include <cstdint>
template <int MODE>
__global__ void k(uint32_t* out, double* outd, int iters, uint32_t a, double b) {
  uint32_t x[8];
  double d[8];
  for (int i = 0; i < 8; ++i) x[i] = threadIdx.x + i, d[i] = threadIdx.x * 0.5 + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (MODE != 1) x[i] = x[i] * a + 0x9e3779b9u;
      if (MODE != 0) d[i] = fma(d[i], b, 0.25);
    }
  }
  uint32_t s = 0;
  double t = 0;
  for (int i = 0; i < 8; ++i) s ^= x[i], t += d[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  outd[blockIdx.x * blockDim.x + threadIdx.x] = t;
}
int main() {
  uint32_t* o;
  double* od;
  cudaMalloc(&o, 148 * 8 * 256 * 4);
  cudaMalloc(&od, 148 * 8 * 256 * 8);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int iters = 4096;
  const double ops = 148.0 * 8 * 256 * iters * 8;
  for (int mode = 0; mode < 3; ++mode) {
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(e0);
      if (mode == 0) k<0><<<148 * 8, 256>>>(o, od, iters, 3u, 1.0000001);
      if (mode == 1) k<1><<<148 * 8, 256>>>(o, od, iters, 3u, 1.0000001);
      if (mode == 2) k<2><<<148 * 8, 256>>>(o, od, iters, 3u, 1.0000001);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
    }
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    printf("%s %.3f ms  %.1f Gop/s per type  %.2f op/clk/SM per type @1.965GHz\n",
           mode == 0 ? "imad-only " : mode == 1 ? "dfma-only " : "interleaved", ms, ops / ms / 1e6,
           ops / (ms * 1e-3) / 148 / 1.965e9);
  }
  return 0;
}
