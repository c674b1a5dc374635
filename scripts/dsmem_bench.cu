// dsmem_bench.cu — latency of the split-K reduction building blocks on B200,
// inside one (1,1,8) cluster of 384-thread CTAs (the GEMM's shape):
//   barrier_relaxed  barrier.cluster.arrive.relaxed + wait
//   barrier_relacq   barrier.cluster.arrive.release + wait.acquire after a global store
//   st_async         every epilogue thread (256) pushes 2 x 16 B to each of 7 peers
//                    (st.async, complete_tx on the peer's mbarrier); issue time and
//                    time until this CTA's own receive barrier completes
//   ld_remote        every epilogue thread loads 2 x 16 B from each of 7 peers
//                    (ld.shared::cluster.v4), all in flight
//   bulk             one thread bulk-copies 7 x 6 KiB blocks to the peers; time
//                    until this CTA's receive barrier completes
//   ldtm             tcgen05.ld 32x32b.x16 x 2 + wait (one warp per lane quarter)
// Cycles (clock64) per CTA, median over CTAs and launches; cold = first launch.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o dsmem_bench scripts/dsmem_bench.cu && ./dsmem_bench
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <vector>

#define CK(x)                                                               \
  do {                                                                      \
    cudaError_t e = (x);                                                    \
    if (e != cudaSuccess) {                                                 \
      std::printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); \
      return 1;                                                             \
    }                                                                       \
  } while (0)

constexpr int S = 8, kT = 384, kRecvRow = 12;  // floats per received row (8 + 4 pad)
constexpr int kSlots = 8;

__device__ __forceinline__ uint32_t su32(const void* p) { return uint32_t(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ uint32_t mapa(uint32_t a, uint32_t r) {
  uint32_t o;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(o) : "r"(a), "r"(r));
  return o;
}
__device__ __forceinline__ uint32_t cta_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  asm volatile(
      "{\n .reg .pred p;\nW_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra W_%=;\n}" ::"r"(bar),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void csync_relaxed() {
  asm volatile("barrier.cluster.arrive.relaxed.aligned;\n\tbarrier.cluster.wait.aligned;" ::: "memory");
}
__device__ __forceinline__ void csync_relacq() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

__global__ void __cluster_dims__(1, 1, S) __launch_bounds__(kT, 1)
    bench_kernel(long long* out, int* gbuf) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ __align__(8) uint64_t bar_st, bar_bulk;
  __shared__ uint32_t tbase;
  float* recv = reinterpret_cast<float*>(smem);                   // [S][128][12]
  float* outgoing = reinterpret_cast<float*>(smem + 64 * 1024);   // [S][128][12]
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t me = cta_rank();
  const int ep = threadIdx.x - 128;  // epilogue thread 0..255 (warps 4..11)
  const int rl = (warp & 3) * 32 + lane, half = (warp - 4) >> 2;
  long long t[kSlots] = {0};
  const uint32_t block = 128 * kRecvRow * 4;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar_st)));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar_bulk)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    // st_async: 7 peers x 256 threads x 16 B; bulk: 7 blocks
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&bar_st)),
                 "r"(uint32_t((S - 1) * 256 * 16)));
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&bar_bulk)),
                 "r"(uint32_t((S - 1) * block)));
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 64;" ::"r"(su32(&tbase)) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  for (int i = threadIdx.x; i < 2 * S * 128 * kRecvRow; i += kT) recv[i] = float(i);
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  csync_relacq();

  // 0: relaxed cluster barrier
  long long c0 = clock64();
  csync_relaxed();
  t[0] = clock64() - c0;
  // 1: release/acquire cluster barrier after a global store
  gbuf[blockIdx.z * kT + threadIdx.x] += 1;
  c0 = clock64();
  csync_relacq();
  t[1] = clock64() - c0;
  // 2: st.async push (epilogue warps), issue time
  if (ep >= 0) {
    c0 = clock64();
#pragma unroll
    for (int j = 1; j < S; ++j) {
      const uint32_t peer = (me + j) % S;
      // my partial of peer's slice: row rl, columns [half*4, half*4+4) -> recv[me][rl]
      const uint32_t dst = mapa(su32(recv + (me * 128 + rl) * kRecvRow + half * 4), peer);
      const uint32_t rbar = mapa(su32(&bar_st), peer);
      asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v4.b32 [%0], {%1, %2, %3, %4}, [%5];" ::"r"(
                       dst),
                   "r"(j), "r"(rl), "r"(half), "r"(me), "r"(rbar)
                   : "memory");
    }
    t[2] = clock64() - c0;
    mbar_wait(su32(&bar_st), 0);
    t[3] = clock64() - c0;
  }
  csync_relaxed();
  // 4: remote loads (all in flight), then use them
  if (ep >= 0) {
    c0 = clock64();
    float4 v[S - 1];
#pragma unroll
    for (int j = 1; j < S; ++j) {
      const uint32_t src = mapa(su32(outgoing + (j * 128 + rl) * kRecvRow + half * 4), (me + j) % S);
      asm volatile("ld.shared::cluster.v4.f32 {%0, %1, %2, %3}, [%4];"
                   : "=f"(v[j - 1].x), "=f"(v[j - 1].y), "=f"(v[j - 1].z), "=f"(v[j - 1].w)
                   : "r"(src)
                   : "memory");
    }
    float s = 0.f;
#pragma unroll
    for (int j = 0; j < S - 1; ++j) s += v[j].x + v[j].y + v[j].z + v[j].w;
    t[4] = clock64() - c0;
    if (s == 12345.f) gbuf[0] = 1;
  }
  csync_relaxed();
  // 5: bulk copies by one thread, until my own receive barrier completes
  if (threadIdx.x == 128) {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    c0 = clock64();
    for (int j = 1; j < S; ++j) {
      const uint32_t peer = (me + j) % S;
      asm volatile(
          "cp.async.bulk.shared::cluster.shared::cta.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
              mapa(su32(recv) + me * block, peer)),
          "r"(su32(outgoing) + peer * block), "r"(block), "r"(mapa(su32(&bar_bulk), peer))
          : "memory");
    }
    t[5] = clock64() - c0;
    mbar_wait(su32(&bar_bulk), 0);
    t[6] = clock64() - c0;
  }
  csync_relaxed();
  // 7: TMEM load round trip (x16 x 2 + wait), warps 4..7
  if (warp >= 4 && warp < 8) {
    uint32_t r[32];
    const uint32_t ta = tbase + (uint32_t((warp & 3) * 32) << 16);
    c0 = clock64();
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
          "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
        : "r"(ta));
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
          "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
        : "r"(ta + 16));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    t[7] = clock64() - c0;
    uint32_t x = 0;
    for (int i = 0; i < 32; ++i) x ^= r[i];
    if (x == 0xdeadbeef) gbuf[1] = 1;
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  csync_relaxed();
  if (warp == 1) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 64;" ::"r"(tbase) : "memory");
  }
  // one row per CTA: thread 0 for the barriers, thread 128 for the rest
  if (threadIdx.x == 0) {
    out[blockIdx.z * kSlots + 0] = t[0];
    out[blockIdx.z * kSlots + 1] = t[1];
  }
  if (threadIdx.x == 128)
    for (int i = 2; i < kSlots; ++i) out[blockIdx.z * kSlots + i] = t[i];
}

int main() {
  long long* out;
  int* gbuf;
  CK(cudaMalloc(&out, S * kSlots * sizeof(long long)));
  CK(cudaMalloc(&gbuf, S * kT * 4 + 64));
  CK(cudaMemset(gbuf, 0, S * kT * 4 + 64));
  const int smem = 2 * 64 * 1024;
  CK(cudaFuncSetAttribute(bench_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  const char* names[kSlots] = {"barrier_relaxed", "barrier_relacq", "st_async_issue", "st_async_landed",
                               "ld_remote_x7",    "bulk_issue_x7",  "bulk_landed",     "ldtm_x16x2"};
  std::vector<std::vector<long long>> acc(kSlots);
  std::vector<long long> h(S * kSlots);
  for (int rep = 0; rep < 21; ++rep) {
    bench_kernel<<<dim3(1, 1, S), kT, smem>>>(out, gbuf);
    CK(cudaGetLastError());
    CK(cudaDeviceSynchronize());
    CK(cudaMemcpy(h.data(), out, h.size() * sizeof(long long), cudaMemcpyDeviceToHost));
    if (rep == 0) {
      std::printf("{\"launch\": \"cold\"");
      for (int i = 0; i < kSlots; ++i) {
        std::vector<long long> v;
        for (int c = 0; c < S; ++c) v.push_back(h[c * kSlots + i]);
        std::sort(v.begin(), v.end());
        std::printf(", \"%s\": %lld", names[i], v[S / 2]);
      }
      std::printf("}\n");
      continue;
    }
    for (int i = 0; i < kSlots; ++i)
      for (int c = 0; c < S; ++c) acc[i].push_back(h[c * kSlots + i]);
  }
  std::printf("{\"launch\": \"warm\", \"unit\": \"cycles\"");
  for (int i = 0; i < kSlots; ++i) {
    std::sort(acc[i].begin(), acc[i].end());
    std::printf(", \"%s\": %lld", names[i], acc[i][acc[i].size() / 2]);
  }
  std::printf("}\n");
  return 0;
}
