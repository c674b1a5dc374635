// sync_floor.cu — the latency floor of a dependent layer chain on B200, two ways:
//  (A) L kernels in one CUDA graph, programmatic dependent launch between them
//      (griddepcontrol), 148 CTAs each, optionally with the GEMM kernel's
//      prologue (large dynamic smem + TMEM alloc/free);
//  (B) ONE persistent kernel, 148 CTAs, L "layers" handed over through a
//      per-layer completion counter (writer: bar.sync + threadfence + atomicAdd;
//      reader: ld.acquire.gpu poll).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o sync_floor scripts/sync_floor.cu && ./sync_floor
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <vector>

#define CK(x)                                                                       \
  do {                                                                              \
    cudaError_t e = (x);                                                            \
    if (e != cudaSuccess) {                                                         \
      std::printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e));         \
      return 1;                                                                     \
    }                                                                               \
  } while (0)

__global__ void chain_kernel(int* buf, int layer, int prologue) {
  extern __shared__ uint8_t smem[];
  __shared__ uint32_t tbase;
  if (prologue && threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 128;" ::"r"(
                     uint32_t(__cvta_generic_to_shared(&tbase)))
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  __syncthreads();
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  asm volatile("griddepcontrol.wait;" ::: "memory");
  if (threadIdx.x == 0) buf[blockIdx.x] = buf[blockIdx.x] + layer + smem[0] * 0;
  __syncthreads();
  if (prologue && threadIdx.x < 32)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 128;" ::"r"(tbase) : "memory");
}

__device__ __forceinline__ uint32_t ld_acquire(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// Every CTA does one item per layer; layer l waits for all CTAs' layer l-1.
__global__ void persistent_kernel(uint32_t* done, int* buf, int layers, int deps_all) {
  for (int l = 0; l < layers; ++l) {
    if (l > 0) {
      if (threadIdx.x == 0) {
        const uint32_t want = deps_all ? gridDim.x : 1;
        while (ld_acquire(done + l - 1) < want) {
        }
      }
      __syncthreads();
    }
    if (threadIdx.x < 32) buf[blockIdx.x * 32 + threadIdx.x] += l;
    __syncthreads();
    if (threadIdx.x == 0) {
      __threadfence();
      atomicAdd(done + l, 1u);
    }
  }
}

int main() {
  const int L = 57, G = 148, reps = 20;
  int* buf;
  uint32_t* done;
  CK(cudaMalloc(&buf, 1 << 20));
  CK(cudaMalloc(&done, 4096 * 4));
  cudaStream_t s;
  CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  CK(cudaFuncSetAttribute(chain_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
  for (int prologue = 0; prologue < 2; ++prologue) {
    for (int pdl = 0; pdl < 2; ++pdl) {
      cudaGraph_t g;
      cudaGraphExec_t ge;
      CK(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
      for (int l = 0; l < L; ++l) {
        cudaLaunchConfig_t cfg{};
        cfg.gridDim = dim3(G);
        cfg.blockDim = dim3(256);
        cfg.dynamicSmemBytes = prologue ? 165 * 1024 : 0;
        cfg.stream = s;
        cudaLaunchAttribute a[1];
        a[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        a[0].val.programmaticStreamSerializationAllowed = 1;
        cfg.attrs = a;
        cfg.numAttrs = pdl;
        CK(cudaLaunchKernelEx(&cfg, chain_kernel, buf, l, prologue));
      }
      CK(cudaStreamEndCapture(s, &g));
      CK(cudaGraphInstantiate(&ge, g, 0));
      for (int i = 0; i < 3; ++i) CK(cudaGraphLaunch(ge, s));
      CK(cudaEventRecord(e0, s));
      for (int i = 0; i < reps; ++i) CK(cudaGraphLaunch(ge, s));
      CK(cudaEventRecord(e1, s));
      CK(cudaStreamSynchronize(s));
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      std::printf("{\"mode\": \"graph_chain\", \"prologue\": %d, \"pdl\": %d, \"us_per_kernel\": %.3f}\n", prologue,
                  pdl, ms * 1e3 / reps / L);
      cudaGraphExecDestroy(ge);
      cudaGraphDestroy(g);
    }
  }
  for (int deps_all = 0; deps_all < 2; ++deps_all) {
    float best = 1e9;
    for (int i = 0; i < reps; ++i) {
      CK(cudaMemsetAsync(done, 0, 4096 * 4, s));
      CK(cudaEventRecord(e0, s));
      persistent_kernel<<<G, 256, 0, s>>>(done, buf, L, deps_all);
      CK(cudaEventRecord(e1, s));
      CK(cudaStreamSynchronize(s));
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      if (ms < best) best = ms;
    }
    std::printf("{\"mode\": \"persistent\", \"deps\": \"%s\", \"us_per_layer\": %.3f}\n",
                deps_all ? "all 148 CTAs" : "one CTA", best * 1e3 / L);
  }
  return 0;
}
