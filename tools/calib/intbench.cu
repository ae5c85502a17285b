// Integer-pipe calibration microbenchmarks for the sm_100a roofline model.
// Each kernel runs ITERS iterations of 4 independent chains per thread over a full grid and
// reports operations per second. Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 intbench.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define ITERS 4096
#define CHAINS 4

__device__ __forceinline__ uint64_t mulhi64(uint64_t a, uint64_t b) { return __umul64hi(a, b); }

__global__ void k_imad32(uint32_t* out, uint32_t s) {
  uint32_t x[CHAINS];
  for (int c = 0; c < CHAINS; ++c) x[c] = threadIdx.x + c * 7 + s;
  for (int i = 0; i < ITERS; ++i) {
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) x[c] = x[c] * 0x9E3779B1u + s;
  }
  uint32_t r = 0;
  for (int c = 0; c < CHAINS; ++c) r ^= x[c];
  out[blockIdx.x * blockDim.x + threadIdx.x] = r;
}

__global__ void k_imadwide(uint64_t* out, uint32_t s) {
  uint64_t x[CHAINS];
  for (int c = 0; c < CHAINS; ++c) x[c] = threadIdx.x + c * 7 + s;
  for (int i = 0; i < ITERS; ++i) {
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) x[c] = (uint64_t)(uint32_t)x[c] * 0x9E3779B1u + (x[c] >> 32);
  }
  uint64_t r = 0;
  for (int c = 0; c < CHAINS; ++c) r ^= x[c];
  out[blockIdx.x * blockDim.x + threadIdx.x] = r;
}

__global__ void k_mulhi64(uint64_t* out, uint64_t s) {
  uint64_t x[CHAINS];
  for (int c = 0; c < CHAINS; ++c) x[c] = threadIdx.x + c * 7 + s;
  for (int i = 0; i < ITERS; ++i) {
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) x[c] = mulhi64(x[c], 0x9E3779B97F4A7C15ull) + s;
  }
  uint64_t r = 0;
  for (int c = 0; c < CHAINS; ++c) r ^= x[c];
  out[blockIdx.x * blockDim.x + threadIdx.x] = r;
}

// Shoup modmul: x*w mod q with wp = floor(w*2^64/q); result in [0,2q).
__global__ void k_shoup64(uint64_t* out, uint64_t q, uint64_t w, uint64_t wp) {
  uint64_t x[CHAINS];
  for (int c = 0; c < CHAINS; ++c) x[c] = threadIdx.x + c * 7;
  for (int i = 0; i < ITERS; ++i) {
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) {
      uint64_t h = mulhi64(x[c], wp);
      x[c] = x[c] * w - h * q;
    }
  }
  uint64_t r = 0;
  for (int c = 0; c < CHAINS; ++c) r ^= x[c];
  out[blockIdx.x * blockDim.x + threadIdx.x] = r;
}

// Harvey lazy CT butterfly on [0,4q).
__global__ void k_bfly64(uint64_t* out, uint64_t q, uint64_t w, uint64_t wp) {
  uint64_t X[CHAINS], Y[CHAINS];
  const uint64_t q2 = 2 * q;
  for (int c = 0; c < CHAINS; ++c) { X[c] = threadIdx.x + c * 7; Y[c] = threadIdx.x * 3 + c; }
  for (int i = 0; i < ITERS; ++i) {
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) {
      uint64_t x = X[c];
      x = x >= q2 ? x - q2 : x;
      uint64_t h = mulhi64(Y[c], wp);
      uint64_t t = Y[c] * w - h * q;
      X[c] = x + t;
      Y[c] = x - t + q2;
    }
  }
  uint64_t r = 0;
  for (int c = 0; c < CHAINS; ++c) r ^= X[c] ^ Y[c];
  out[blockIdx.x * blockDim.x + threadIdx.x] = r;
}

// 64x64->128 multiply-accumulate.
__global__ void k_mac128(uint64_t* out, uint64_t s) {
  uint64_t a[CHAINS], lo[CHAINS], hi[CHAINS];
  for (int c = 0; c < CHAINS; ++c) { a[c] = threadIdx.x + c * 7 + s; lo[c] = 0; hi[c] = 0; }
  for (int i = 0; i < ITERS; ++i) {
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) {
      uint64_t b = a[c] ^ (uint64_t)i;
      uint64_t pl = a[c] * b, ph = mulhi64(a[c], b);
      uint64_t nl = lo[c] + pl;
      hi[c] += ph + (nl < pl);
      lo[c] = nl;
    }
  }
  uint64_t r = 0;
  for (int c = 0; c < CHAINS; ++c) r ^= lo[c] ^ hi[c];
  out[blockIdx.x * blockDim.x + threadIdx.x] = r;
}

// 32-bit Shoup modmul.
__global__ void k_shoup32(uint32_t* out, uint32_t q, uint32_t w, uint32_t wp) {
  uint32_t x[CHAINS];
  for (int c = 0; c < CHAINS; ++c) x[c] = threadIdx.x + c * 7;
  for (int i = 0; i < ITERS; ++i) {
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) {
      uint32_t h = __umulhi(x[c], wp);
      x[c] = x[c] * w - h * q;
    }
  }
  uint32_t r = 0;
  for (int c = 0; c < CHAINS; ++c) r ^= x[c];
  out[blockIdx.x * blockDim.x + threadIdx.x] = r;
}

__global__ void k_dfma(double* out, double s) {
  double x[CHAINS];
  for (int c = 0; c < CHAINS; ++c) x[c] = threadIdx.x + c * 7 + s;
  for (int i = 0; i < ITERS; ++i) {
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) x[c] = fma(x[c], 0.999999, s);
  }
  double r = 0;
  for (int c = 0; c < CHAINS; ++c) r += x[c];
  out[blockIdx.x * blockDim.x + threadIdx.x] = r;
}

// Mixed: one Shoup64 chain and one DFMA chain per iteration (do the pipes overlap?).
__global__ void k_mixed(uint64_t* out, uint64_t q, uint64_t w, uint64_t wp, double s) {
  uint64_t x[CHAINS];
  double d[CHAINS];
  for (int c = 0; c < CHAINS; ++c) { x[c] = threadIdx.x + c * 7; d[c] = threadIdx.x + c + s; }
  for (int i = 0; i < ITERS; ++i) {
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) {
      uint64_t h = mulhi64(x[c], wp);
      x[c] = x[c] * w - h * q;
      d[c] = fma(d[c], 0.999999, s);
      d[c] = fma(d[c], 0.999998, s);
      d[c] = fma(d[c], 0.999997, s);
      d[c] = fma(d[c], 0.999996, s);
    }
  }
  uint64_t r = 0;
  for (int c = 0; c < CHAINS; ++c) r ^= x[c] ^ (uint64_t)d[c];
  out[blockIdx.x * blockDim.x + threadIdx.x] = r;
}

__global__ void k_copy(const uint4* __restrict__ a, uint4* __restrict__ b, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) b[i] = a[i];
}

int main() {
  const int blocks = 148 * 8, threads = 256;
  const double nthreads = (double)blocks * threads;
  void* buf;
  cudaMalloc(&buf, blocks * threads * 8);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const uint64_t q = 0x0FFFFFFFFFFFC001ull, w = 116777451583545ull;
  const uint64_t wp = (uint64_t)(((unsigned __int128)w << 64) / q);
  const uint32_t q32 = 0x7FFE001u /* placeholder */, w32 = 12345u;
  const uint32_t wp32 = (uint32_t)(((uint64_t)w32 << 32) / q32);
  auto run = [&](const char* name, double ops_per_iter, auto launch) {
    launch();
    cudaDeviceSynchronize();
    cudaEventRecord(e0);
    for (int r = 0; r < 5; ++r) launch();
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    double ops = 5.0 * nthreads * ITERS * CHAINS * ops_per_iter;
    printf("%-12s %8.3f ms  %10.3f Gop/s  %8.2f op/clk/SM@1.965GHz\n", name, ms / 5, ops / (ms * 1e-3) / 1e9,
           ops / (ms * 1e-3) / 148 / 1.965e9);
  };
  run("imad32", 1, [&] { k_imad32<<<blocks, threads>>>((uint32_t*)buf, 3); });
  run("imadwide", 1, [&] { k_imadwide<<<blocks, threads>>>((uint64_t*)buf, 3); });
  run("mulhi64", 1, [&] { k_mulhi64<<<blocks, threads>>>((uint64_t*)buf, 3); });
  run("shoup64", 1, [&] { k_shoup64<<<blocks, threads>>>((uint64_t*)buf, q, w, wp); });
  run("bfly64", 1, [&] { k_bfly64<<<blocks, threads>>>((uint64_t*)buf, q, w, wp); });
  run("mac128", 1, [&] { k_mac128<<<blocks, threads>>>((uint64_t*)buf, 3); });
  run("shoup32", 1, [&] { k_shoup32<<<blocks, threads>>>((uint32_t*)buf, q32, w32, wp32); });
  run("dfma", 1, [&] { k_dfma<<<blocks, threads>>>((double*)buf, 0.5); });
  run("mixed(shoup)", 1, [&] { k_mixed<<<blocks, threads>>>((uint64_t*)buf, q, w, wp, 0.5); });
  // HBM copy
  size_t n = (size_t)1 << 30;  // 1 GiB each
  void *a, *b;
  cudaMalloc(&a, n);
  cudaMalloc(&b, n);
  cudaMemset(a, 1, n);
  k_copy<<<148 * 16, 256>>>((uint4*)a, (uint4*)b, n / 16);
  cudaDeviceSynchronize();
  cudaEventRecord(e0);
  for (int r = 0; r < 10; ++r) k_copy<<<148 * 16, 256>>>((uint4*)a, (uint4*)b, n / 16);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  printf("copy 1GiB    %8.3f ms  %10.1f GB/s (r+w)\n", ms / 10, 2.0 * n * 10 / (ms * 1e-3) / 1e9);
  cudaError_t err = cudaGetLastError();
  printf("status: %s\n", cudaGetErrorString(err));
  return 0;
}
