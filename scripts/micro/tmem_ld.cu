// TMEM read throughput: W warps (W/4 per TMEM lane quarter) each issue R rounds of
// tcgen05.ld.32x32b.x32 (32 lanes x 32 columns x 4 B = 4 KB per warp-instruction) over the
// 128 columns of their slot, waiting after every load (as the softmax does) or after 4.
// Prints cycles per 4-KB load per warp and the SM's aggregate TMEM read rate in B/cycle.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tmem_ld tmem_ld.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

template <int WAITEVERY>
__global__ void __launch_bounds__(256, 1) tmem_ld(int rounds, long long* out, float* sink) {
  __shared__ uint32_t tslot;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
        uint32_t(__cvta_generic_to_shared(&tslot))));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = tslot;
  const int quarter = warp & 3, slot = warp >> 2;  // warps 4..7 read the other 256 columns
  const uint32_t base = tmem + (uint32_t(quarter * 32) << 16) + slot * 256;
  float acc = 0.f;
  long long t0 = clock64();
  for (int r = 0; r < rounds; ++r) {
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      uint32_t v[32];
      asm volatile(
          "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
          "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
          : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
            "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]),
            "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]),
            "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
          : "r"(base + c * 32));
      if (WAITEVERY == 1 || c == 3) asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
      if (c == 3 && r == rounds - 1) {  // consume once (the asm is volatile: no load is dropped)
#pragma unroll
        for (int k = 0; k < 32; ++k) acc += __uint_as_float(v[k]);
      }
    }
  }
  long long t1 = clock64();
  if ((threadIdx.x & 31) == 0) out[blockIdx.x * 8 + warp] = t1 - t0;
  if (acc == 12345.f) sink[threadIdx.x] = acc;
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

int main() {
  long long* d_out;
  float* sink;
  cudaMalloc(&d_out, 148 * 8 * sizeof(long long));
  cudaMalloc(&sink, 1024 * 4);
  const int rounds = 2000;
  for (int warps : {4, 8}) {
    for (int we : {1, 4}) {
      if (we == 1) tmem_ld<1><<<148, warps * 32>>>(rounds, d_out, sink);
      else tmem_ld<4><<<148, warps * 32>>>(rounds, d_out, sink);
      cudaDeviceSynchronize();
      long long h[148 * 8];
      cudaMemcpy(h, d_out, sizeof(h), cudaMemcpyDeviceToHost);
      double cyc = 0;
      for (int w = 0; w < warps; ++w) cyc += double(h[w]);
      cyc /= warps;
      const double per_ld = cyc / (rounds * 4.0);
      printf("%d warps, wait every %d load(s): %.1f cycles per 4-KB tcgen05.ld per warp; SM aggregate %.1f B/cycle\n",
             warps, we, per_ld, warps * 4096.0 / per_ld);
    }
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
