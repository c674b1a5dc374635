// Probe: hardware cvt.rn.bf16x2.f32 vs the integer RNE definition, over
// special values and a dense random sweep. Prints mismatch classes.
#include <cstdio>
#include <cstdint>
#include <cstring>
#include <cuda_bf16.h>
#include <random>
#include <vector>

__global__ void k(const uint32_t* in, uint32_t* out, int n) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (2 * i + 1 >= n) return;
  float a = __uint_as_float(in[2 * i]), b = __uint_as_float(in[2 * i + 1]);
  uint32_t r;
  asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(b), "f"(a));
  out[i] = r;
}

static uint16_t ref(uint32_t u) {
  if ((u & 0x7fffffffu) > 0x7f800000u) return uint16_t(((u >> 16) & 0x8000u) | 0x7fc0u);
  return uint16_t((u + 0x7fffu + ((u >> 16) & 1u)) >> 16);
}

int main() {
  std::vector<uint32_t> v = {0x7fc00000u, 0xffc00000u, 0x7f800001u, 0xff800001u, 0x7fbfffffu, 0x7fffffffu,
                             0xffffffffu, 0x7f800000u, 0xff800000u, 0, 0x80000000u, 1, 0x80000001u, 0x007fffffu,
                             0x3f808000u, 0x3f818000u, 0x7f7fffffu, 0xff7fffffu, 0x7f7f8000u, 0x00008000u};
  std::mt19937 rng(1);
  for (int i = 0; i < (1 << 22); ++i) v.push_back(rng());
  if (v.size() & 1) v.push_back(0);
  int n = int(v.size());
  uint32_t *din, *dout;
  cudaMalloc(&din, n * 4);
  cudaMalloc(&dout, n * 2);
  cudaMemcpy(din, v.data(), n * 4, cudaMemcpyHostToDevice);
  k<<<(n / 2 + 255) / 256, 256>>>(din, dout, n);
  std::vector<uint16_t> o(n);
  cudaMemcpy(o.data(), dout, n * 2, cudaMemcpyDeviceToHost);
  long nan_mis = 0, other_mis = 0;
  for (int i = 0; i < n; ++i) {
    uint16_t want = ref(v[i]);
    if (o[i] != want) {
      bool isnan = (v[i] & 0x7fffffffu) > 0x7f800000u;
      if (isnan) { if (nan_mis < 6) printf("nan %08x -> hw %04x ref %04x\n", v[i], o[i], want); ++nan_mis; }
      else { if (other_mis < 10) printf("MISMATCH %08x -> hw %04x ref %04x\n", v[i], o[i], want); ++other_mis; }
    }
  }
  printf("n=%d nan_mismatch=%ld other_mismatch=%ld\n", n, nan_mis, other_mis);
  return 0;
}
