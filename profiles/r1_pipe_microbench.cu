// Pipe throughput microbenchmark: independent chains per thread, cycles per warp-instruction per SM.
#include <cstdio>
#include <cuda_runtime.h>
template <int OP>
__global__ void k(float* out, long long* cyc, int iters) {
  float a[8];
  for (int i = 0; i < 8; ++i) a[i] = threadIdx.x * 1e-3f + i;
  unsigned long long x2[4];
  for (int i = 0; i < 4; ++i) asm("mov.b64 %0, {%1, %2};" : "=l"(x2[i]) : "f"(a[2*i]), "f"(a[2*i+1]));
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (OP == 0) asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a[i]));
      if (OP == 1) asm volatile("fma.rn.ftz.f32 %0, %0, %0, %0;" : "+f"(a[i]));
      if (OP == 2 && i < 4) asm volatile("fma.rn.ftz.f32x2 %0, %0, %0, %0;" : "+l"(x2[i]));
      if (OP == 3 && i < 4) asm volatile("ex2.approx.f16x2 %0, %0;" : "+r"(*reinterpret_cast<unsigned*>(&x2[i])));
      if (OP == 4) asm volatile("add.rn.ftz.f32 %0, %0, %0;" : "+f"(a[i]));
    }
  }
  long long t1 = clock64();
  float s = 0; for (int i = 0; i < 8; ++i) s += a[i];
  for (int i = 0; i < 4; ++i) { float lo, hi; asm("mov.b64 {%0,%1}, %2;" : "=f"(lo), "=f"(hi) : "l"(x2[i])); s += lo + hi; }
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}
int main() {
  float* out; long long* cyc; cudaMalloc(&out, 148 * 1024 * 4); cudaMalloc(&cyc, 148 * 8);
  const char* names[] = {"MUFU.EX2 f32", "FFMA", "FFMA2 (f32x2)", "MUFU.EX2 f16x2", "FADD"};
  int ninst[] = {8, 8, 4, 4, 8};
  for (int op = 0; op < 5; ++op) for (int warps : {8, 16, 32}) {
    int iters = 2000;
    void (*f)(float*, long long*, int) = op == 0 ? k<0> : op == 1 ? k<1> : op == 2 ? k<2> : op == 3 ? k<3> : k<4>;
    f<<<148, warps * 32>>>(out, cyc, iters); cudaDeviceSynchronize();
    f<<<148, warps * 32>>>(out, cyc, iters); cudaDeviceSynchronize();
    long long c; cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
    double winst = double(iters) * ninst[op] * warps;  // warp instructions per SM
    printf("%-16s warps=%2d: %.3f cycles per warp-instr per SM  (%.1f lane-ops/clk/SM)\n", names[op], warps, c / winst,
           32.0 * (op == 2 || op == 3 ? 2 : 1) * winst / c);
  }
  return 0;
}
