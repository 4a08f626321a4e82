// tcgen05.mma (kind::f16, bf16, cta_group::1) issue-rate microbenchmark on B200.
// One CTA per SM; one thread issues `iters` MMAs of one shape back to back, commits, waits;
// cycles per MMA vs the nominal rate (M*N*K*2 flop / 8192 flop/clk/SM).
// Variants: SS (A and B from smem) and TS (A from TMEM), N in {64, 128, 256}, with and
// without a concurrent bulk-copy stream writing smem (the prefill's K/V TMA traffic).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o umma umma.cu && ./umma
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ uint64_t sdesc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= uint64_t((saddr >> 4) & 0x3fff);
  d |= uint64_t((lbo >> 4) & 0x3fff) << 16;
  d |= uint64_t((sbo >> 4) & 0x3fff) << 32;
  d |= uint64_t(1) << 46;
  d |= uint64_t(2) << 61;
  return d;
}
__host__ __device__ constexpr uint32_t idesc_bf16(int M, int N) {
  return (1u << 4) | (1u << 7) | (1u << 10) | (uint32_t(N >> 3) << 17) | (uint32_t(M >> 4) << 24);
}

template <int N, bool TS, bool COPY, bool TMEMLD = false>
__global__ void __launch_bounds__(128, 1) umma_bench(int iters, long long* out, const uint4* src) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint32_t tmem_slot;
  __shared__ __align__(8) uint64_t bar, cbar;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_slot)),
                 "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&cbar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = tmem_slot;
  const uint32_t a_s = smem_u32(smem), b_s = a_s + 32768;  // A 128x128 bf16, B up to 256x128
  if (threadIdx.x == 0) {
    constexpr uint32_t id = idesc_bf16(128, N);
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
      const int k = it & 7;
      const uint64_t bd = sdesc(b_s + (k >> 2) * (N * 128) + (k & 3) * 32, 16, 1024);
      if (TS) {
        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                     "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tmem),
                     "r"(tmem + 256 + k * 8), "l"(bd), "r"(id), "r"(1u)
                     : "memory");
      } else {
        const uint64_t ad = sdesc(a_s + (k >> 2) * (128 * 128) + (k & 3) * 32, 16, 1024);
        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                     "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem),
                     "l"(ad), "l"(bd), "r"(id), "r"(1u)
                     : "memory");
      }
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar))
                 : "memory");
    asm volatile("{\n\t.reg .pred p;\n\tW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n\t@!p bra W;\n\t}" ::"r"(
                     smem_u32(&bar)));
    long long t1 = clock64();
    out[blockIdx.x] = t1 - t0;
  } else if (COPY && threadIdx.x == 32) {
    // concurrent smem writes: 64 KB bulk copies from global (L2-resident source), one
    // outstanding at a time into a separate region -- about the prefill's K/V TMA write rate
    const uint32_t dst = a_s + 98304;
    for (int r = 0; r < iters / 16; ++r) {
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&cbar)), "r"(65536));
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
                   "l"(src + (blockIdx.x % 4) * 4096), "r"(65536), "r"(smem_u32(&cbar))
                   : "memory");
      asm volatile("{\n\t.reg .pred p;\n\tW2: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W2;\n\t}" ::"r"(
                       smem_u32(&cbar)), "r"(r & 1));
    }
  } else if (TMEMLD && warp >= 2) {
    // concurrent TMEM traffic: warps 2..3 stream tcgen05.ld of columns [256, 384) (their lane quarter)
    const uint32_t base = tmem + (uint32_t((warp & 3) * 32) << 16) + 384;
    float acc = 0.f;
    for (int r = 0; r < iters / 4; ++r) {
      uint32_t v[32];
      asm volatile("tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
                   "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
                   : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
                     "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]),
                     "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]),
                     "=r"(v[22]), "=r"(v[23]), "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]),
                     "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
                   : "r"(base));
      asm volatile("tcgen05.wait::ld.sync.aligned;");
      acc += __uint_as_float(v[r & 31]);
    }
    if (acc == 12345.f) out[0] = 0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
}

template <int N, bool TS, bool COPY, bool TMEMLD = false>
void run(const char* name, long long* d_out, const uint4* src, int sms) {
  const int iters = 4096;
  auto k = umma_bench<N, TS, COPY, TMEMLD>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  k<<<sms, 128, 200 * 1024>>>(iters, d_out, src);
  k<<<sms, 128, 200 * 1024>>>(iters, d_out, src);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) { printf("%s: %s\n", name, cudaGetErrorString(e)); return; }
  long long h[256];
  cudaMemcpy(h, d_out, sms * sizeof(long long), cudaMemcpyDeviceToHost);
  double avg = 0;
  for (int i = 0; i < sms; ++i) avg += h[i];
  avg /= sms;
  const double nominal = 128.0 * N * 16 * 2 / 8192.0;
  printf("%-34s %7.1f cycles/MMA  nominal %5.1f  -> %5.1f %% of peak\n", name, avg / iters, nominal,
         100.0 * nominal / (avg / iters));
  fflush(stdout);
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  long long* d_out;
  uint4* src;
  cudaMalloc(&d_out, 256 * sizeof(long long));
  cudaMalloc(&src, size_t(sms) * 64 * 1024 * 16);
  cudaMemset(src, 0, size_t(sms) * 64 * 1024 * 16);
  run<64, false, false>("SS M128 N64 K16", d_out, src, sms);
  run<128, false, false>("SS M128 N128 K16", d_out, src, sms);
  run<256, false, false>("SS M128 N256 K16", d_out, src, sms);
  run<64, true, false>("TS M128 N64 K16", d_out, src, sms);
  run<128, true, false>("TS M128 N128 K16", d_out, src, sms);
  run<256, true, false>("TS M128 N256 K16", d_out, src, sms);
  run<128, false, true>("SS M128 N128 K16 + smem copy", d_out, src, sms);
  run<128, true, true>("TS M128 N128 K16 + smem copy", d_out, src, sms);
  run<64, true, true>("TS M128 N64 K16 + smem copy", d_out, src, sms);
  run<128, false, false, true>("SS M128 N128 K16 + TMEM ld", d_out, src, sms);
  run<128, true, false, true>("TS M128 N128 K16 + TMEM ld", d_out, src, sms);
  run<128, false, true, true>("SS M128 N128 K16 + copy + TMEM ld", d_out, src, sms);
  return 0;
}
