// Where does a single-CTA 4096-point NTT spend its time? Replicates k_ntt_fwd's structure
// (32-bit words, one poly per CTA, 256 threads, 3 radix-16 rounds) with clock64() marks after
// each phase, for 8 CTAs (a latency-bound batch) and 2048 CTAs (a throughput-bound batch).
#include <cstdio>
#include <cstdint>
#include "../../paper_2506_11586_b200/csrc/ntt_core.cuh"
using namespace secn;
constexpr int LOGN = 12, N = 4096;
__global__ void __launch_bounds__(256) k(const uint32_t* in, uint32_t* out, const uint2* tw, uint32_t q,
                                         long long* marks) {
  using A = Arith32;
  using R0 = CtRound<LOGN, 0>;
  __shared__ uint32_t sm[smem_words<LOGN>()];
  long long t[8];
  t[0] = clock64();
  uint2 tws[15];
  ct_twiddles<A, LOGN, 0>(tws, tw);
  uint32_t x[1][16];
  const uint32_t* src = in + (size_t)blockIdx.x * N;
#pragma unroll
  for (int i = 0; i < 16; ++i) x[0][i] = src[R0::addr(0, i)];
  const uint32_t qb = 2 * q;
  // force the loads to complete before the mark
  uint32_t s = 0;
#pragma unroll
  for (int i = 0; i < 16; ++i) s |= x[0][i];
  if (s == 0xffffffffu) out[0] = s;
  t[1] = clock64();
  ct_compute<A, LOGN, 0, 1>(x, tws, q, qb);
  round_store<R0, uint32_t, 1, LOGN>(x, sm);
  t[2] = clock64();
  using R1 = CtRound<LOGN, 4>;
  ct_twiddles<A, LOGN, 4>(tws, tw);
  __syncthreads();
  t[3] = clock64();
  round_load<R1, uint32_t, 1, LOGN>(x, sm);
  ct_compute<A, LOGN, 4, 1>(x, tws, q, qb);
  round_store<R1, uint32_t, 1, LOGN>(x, sm);
  t[4] = clock64();
  using R2 = CtRound<LOGN, 8>;
  ct_twiddles<A, LOGN, 8>(tws, tw);
  __syncthreads();
  t[5] = clock64();
  round_load<R2, uint32_t, 1, LOGN>(x, sm);
  ct_compute<A, LOGN, 8, 1>(x, tws, q, qb);
  t[6] = clock64();
  uint32_t* dst[1] = {out + (size_t)blockIdx.x * N};
  round_gstore<R2, uint32_t, 1>(x, dst);
  t[7] = clock64();
  if (threadIdx.x == 0 && blockIdx.x < 8)
    for (int i = 0; i < 8; ++i) marks[blockIdx.x * 8 + i] = t[i];
}
int main() {
  uint32_t *in, *out;
  uint2* tw;
  long long* marks;
  cudaMalloc(&in, 2048ull * N * 4);
  cudaMalloc(&out, 2048ull * N * 4);
  cudaMalloc(&tw, N * 8);
  cudaMalloc(&marks, 64 * 8);
  cudaMemset(in, 1, 2048ull * N * 4);
  cudaMemset(tw, 3, N * 8);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int grid : {8, 148, 2048}) {
    for (int rep = 0; rep < 3; ++rep) {
      cudaEventRecord(e0);
      k<<<grid, 256>>>(in, out, tw, 0x7e90001u, marks);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
    }
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    long long h[64];
    cudaMemcpy(h, marks, sizeof(h), cudaMemcpyDeviceToHost);
    printf("grid %5d: %.2f us; CTA0 phases (cycles): load %lld r0 %lld tw1+sync %lld r1 %lld tw2+sync %lld r2 %lld store %lld total %lld\n",
           grid, ms * 1e3, h[1] - h[0], h[2] - h[1], h[3] - h[2], h[4] - h[3], h[5] - h[4], h[6] - h[5], h[7] - h[6],
           h[7] - h[0]);
  }
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
}
