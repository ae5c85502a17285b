// Launch-chain latency on sm_100a: time per kernel in a chain of dependent launches (stream order,
// with and without programmatic dependent launch), for an empty kernel and for a kernel that reads
// and writes one 16 KiB poly per CTA.
#include <cstdio>
#include <cstdint>
__global__ void k_empty(int* p) {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  if (p && threadIdx.x == 1000000) p[0] = 1;
}
__global__ void k_copy(const uint32_t* __restrict__ in, uint32_t* __restrict__ out) {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  uint32_t v[16];
  const size_t base = (size_t)blockIdx.x * 4096;
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = in[base + threadIdx.x + 256 * i];
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 16; ++i) out[base + threadIdx.x + 256 * i] = v[i] + 1;
}
template <class K, class... A>
static void launch(K k, int grid, bool pdl, cudaStream_t s, A... a) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = 256;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl ? 1 : 0;
  cudaLaunchKernelEx(&cfg, k, a...);
}
int main() {
  uint32_t *a, *b;
  cudaMalloc(&a, 1 << 26);
  cudaMalloc(&b, 1 << 26);
  cudaStream_t s;
  cudaStreamCreate(&s);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int graph = 0; graph < 2; ++graph)
    for (int kind = 0; kind < 2; ++kind)
      for (int pdl = 0; pdl < 2; ++pdl)
        for (int grid : {8, 148, 1024}) {
          const int K = 50;
          auto body = [&]() {
            for (int i = 0; i < K; ++i) {
              if (kind == 0) launch(k_empty, grid, pdl, s, (int*)nullptr);
              else launch(k_copy, grid, pdl, s, (const uint32_t*)(i & 1 ? b : a), i & 1 ? a : b);
            }
          };
          cudaGraphExec_t ge = nullptr;
          if (graph) {
            cudaGraph_t g;
            cudaStreamBeginCapture(s, cudaStreamCaptureModeGlobal);
            body();
            cudaStreamEndCapture(s, &g);
            cudaGraphInstantiate(&ge, g, 0);
          }
          float best = 1e9;
          for (int rep = 0; rep < 5; ++rep) {
            cudaEventRecord(e0, s);
            if (graph) cudaGraphLaunch(ge, s); else body();
            cudaEventRecord(e1, s);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            best = ms < best ? ms : best;
          }
          printf("%s %-5s pdl=%d grid=%5d: %.2f us per kernel\n", graph ? "graph " : "stream", kind ? "copy" : "empty",
                 pdl, grid, best * 1e3 / K);
        }
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
