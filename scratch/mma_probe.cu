// Probe: (1) fp16 subnormal A operands in mma.sync m16n8k16 on sm_100a; (2) HMMA throughput.
#include <cstdio>
#include <cstdint>
#include <cuda_fp16.h>
__device__ __forceinline__ void mma16816(float* d, const uint32_t* a, const uint32_t* b) {
  asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
    : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3]) : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
}
__global__ void subnormal_test(float* out, uint32_t abits, uint32_t bbits) {
  uint32_t a[4] = {abits, abits, abits, abits};
  uint32_t b[2] = {bbits, bbits};
  float d[4] = {0, 0, 0, 0};
  mma16816(d, a, b);
  int lane = threadIdx.x;
  for (int i = 0; i < 4; i++) out[lane * 4 + i] = d[i];
}
__global__ void tput(float* out, int iters) {
  uint32_t a[4] = {0x00010001u ^ threadIdx.x, 0x00020002u, 0x00030003u, 0x00010002u};
  uint32_t b[2] = {0x3c003c00u, 0x3c003c00u};
  float d0[4] = {0}, d1[4] = {0}, d2[4] = {0}, d3[4] = {0};
  for (int i = 0; i < iters; i++) {
    mma16816(d0, a, b); mma16816(d1, a, b); mma16816(d2, a, b); mma16816(d3, a, b);
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = d0[0] + d1[1] + d2[2] + d3[3];
}
int main() {
  float* d; cudaMalloc(&d, 1 << 24);
  float h[128];
  // A = code 1 in subnormal (0x0001 = 2^-24) both halves; B = 1.0 (0x3c00)
  struct { uint32_t a, b; const char* what; double expect; } cases[] = {
    {0x00010001u, 0x3c003c00u, "A=2^-24 (subnormal), B=1 -> 16 * 2^-24", 16.0 / 16777216.0},
    {0x00030003u, 0x3c003c00u, "A=3*2^-24, B=1 -> 48*2^-24", 48.0 / 16777216.0},
    {0x02000200u, 0x3c003c00u, "A=512*2^-24 (max subnormal bit 9), B=1", 16 * 512.0 / 16777216.0},
    {0x00010001u, 0x00010001u, "A=2^-24, B=2^-24 -> 16*2^-48", 16.0 / 281474976710656.0},
    {0x00030003u, 0x5bd05bd0u, "A=3*2^-24, B=250 -> 16*750*2^-24", 16 * 750.0 / 16777216.0},
  };
  for (auto& c : cases) {
    subnormal_test<<<1, 32>>>(d, c.a, c.b);
    cudaMemcpy(h, d, 128 * 4, cudaMemcpyDeviceToHost);
    printf("%-45s got %.10g expect %.10g %s\n", c.what, h[0], c.expect, h[0] == (float)c.expect ? "EXACT" : "MISMATCH");
  }
  int dev; cudaGetDevice(&dev); int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int warps : {4, 8, 16}) {
    int iters = 4096;
    tput<<<sms, warps * 32>>>(d, 16);
    cudaEventRecord(e0);
    tput<<<sms, warps * 32>>>(d, iters);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double mmas = (double)sms * warps * iters * 4;
    double flops = mmas * 16 * 8 * 16 * 2;
    printf("warps/SM=%d: %.3f ms, %.1f TFLOP/s, %.2f cycles/MMA/SM @1.9GHz\n", warps, ms, flops / ms / 1e9,
           (ms * 1e-3 * 1.9e9) / (mmas / sms));
  }
  return 0;
}
