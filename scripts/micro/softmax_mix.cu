// The prefill softmax's per-pair instruction mix with one (or two) warps per SMSP:
// FFMA2 (argument), 2 x MUFU.EX2, FADD2 (row sum), F2FP (bf16 pack) -- cycles per pair.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__device__ __forceinline__ unsigned long long f2u(float a, float b) { unsigned long long r; asm("mov.b64 %0, {%1,%2};" : "=l"(r) : "f"(a), "f"(b)); return r; }
template <int MODE>
__global__ void k(float* out, long long* cyc, int iters) {
  float x[64];
  for (int i = 0; i < 64; ++i) x[i] = -(threadIdx.x * 1e-3f + i * 0.01f);
  float2 rs = make_float2(0.f, 0.f);
  uint32_t acc = 0;
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int c = 0; c < 64; c += 2) {
      unsigned long long arg, a2 = f2u(x[c], x[c + 1]);
      asm volatile("fma.rn.ftz.f32x2 %0, %1, %2, %3;" : "=l"(arg) : "l"(a2), "l"(f2u(1.0001f, 1.0001f)), "l"(f2u(-0.5f, -0.5f)));
      float lo, hi;
      asm("mov.b64 {%0,%1}, %2;" : "=f"(lo), "=f"(hi) : "l"(arg));
      float e0, e1;
      asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(e0) : "f"(lo));
      asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(e1) : "f"(hi));
      if (MODE >= 1) {
        unsigned long long s2, r2 = f2u(rs.x, rs.y);
        asm volatile("add.rn.ftz.f32x2 %0, %1, %2;" : "=l"(s2) : "l"(r2), "l"(f2u(e0, e1)));
        asm("mov.b64 {%0,%1}, %2;" : "=f"(rs.x), "=f"(rs.y) : "l"(s2));
      }
      if (MODE >= 2) {
        uint32_t p;
        asm volatile("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(p) : "f"(e1), "f"(e0));
        acc ^= p;
      }
      x[c] = e0 * 0.5f - 1.f;
      x[c + 1] = e1 * 0.5f - 1.f;
    }
  }
  long long t1 = clock64();
  out[blockIdx.x * blockDim.x + threadIdx.x] = rs.x + rs.y + acc + x[3];
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}
int main() {
  float* out; long long* cyc; cudaMalloc(&out, 148 * 1024 * 4); cudaMalloc(&cyc, 148 * 8);
  const char* names[] = {"ex2 pairs only", "+ fadd2 sum", "+ fadd2 + cvt bf16x2 pack"};
  for (int mode = 0; mode < 3; ++mode) for (int warps : {4, 8}) {
    int iters = 200;
    void (*f)(float*, long long*, int) = mode == 0 ? k<0> : mode == 1 ? k<1> : k<2>;
    f<<<148, warps * 32>>>(out, cyc, iters); cudaDeviceSynchronize();
    f<<<148, warps * 32>>>(out, cyc, iters); cudaDeviceSynchronize();
    long long c; cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
    double pairs_per_smsp = double(iters) * 32 * (warps / 4);
    printf("%-28s warps/SMSP=%d: %.2f cycles per pair per SMSP (ideal 16 for 2 x MUFU)\n", names[mode], warps / 4,
           c / pairs_per_smsp);
    fflush(stdout);
  }
  return 0;
}
