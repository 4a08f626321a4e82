// Random-granule HBM read ceiling through cp.async.bulk (the decode producer's access path):
// one producer thread per CTA streams granules of G bytes at random (permuted) offsets into an
// NST-deep shared-memory ring; a consumer warp only waits on each stage and releases it. Also
// "pairs": two granules per stage (K and V of one chunk from two pools).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o bulk_read bulk_read.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t su32(const void* p) { return uint32_t(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ void mb_init(uint64_t* b, int n) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(n));
}
__device__ __forceinline__ void mb_expect(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mb_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(b)) : "memory");
}
__device__ __forceinline__ void mb_wait(uint64_t* b, uint32_t par) {
  asm volatile(
      "{\n .reg .pred p;\n W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra W;\n}" ::"r"(su32(b)),
      "r"(par)
      : "memory");
}
__device__ __forceinline__ void bulk(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   su32(dst)),
               "l"(src), "r"(bytes), "r"(su32(bar))
               : "memory");
}

// n_items stages; stage k reads granule g(k) (and g(k) from pool 2 when pairs); g(k) = perm[k]
// (mode bit 0 clear: a dependent global load per stage) or a multiplicative hash of k (bit 0 set:
// no load on the producer's path; n_items a power of two). Mode bit 1: the two copies of a pair
// stage are issued by lanes 0 and 1 of the producer warp (one instruction) instead of one thread.
__global__ void __launch_bounds__(64) ring_read(const uint8_t* pool, const uint8_t* pool2, const uint32_t* perm,
                                                int n_items, int gbytes, int stride, int nst, int pairs, int mode) {
  extern __shared__ __align__(1024) uint8_t sm[];
  const int sbytes = ((pairs ? 2 : 1) * gbytes + 127) & ~127;
  uint64_t* full = reinterpret_cast<uint64_t*>(sm + nst * sbytes);
  uint64_t* empty = full + nst;
  if (threadIdx.x == 0) {
    for (int i = 0; i < nst; ++i) {
      mb_init(&full[i], 1);
      mb_init(&empty[i], 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int per = (n_items + gridDim.x - 1) / gridDim.x;
  const int k0 = blockIdx.x * per, k1 = min(n_items, k0 + per);
  const int lane = threadIdx.x;
  if ((mode & 2) && pairs && lane < 2) {
    for (int k = k0, i = 0; k < k1; ++k, ++i) {
      const int s = i % nst;
      if (i >= nst) mb_wait(&empty[s], ((i / nst) - 1) & 1);
      if (lane == 0) mb_expect(&full[s], 2 * gbytes);
      __syncwarp(3u);
      const uint32_t g = (mode & 1) ? (uint32_t(k) * 2654435761u) & uint32_t(n_items - 1) : perm[k];
      bulk(sm + s * sbytes + lane * gbytes, (lane ? pool2 : pool) + size_t(g) * stride, gbytes, &full[s]);
    }
  } else if (threadIdx.x == 0) {
    for (int k = k0, i = 0; k < k1; ++k, ++i) {
      const int s = i % nst;
      if (i >= nst) mb_wait(&empty[s], ((i / nst) - 1) & 1);
      const uint32_t g = (mode & 1) ? (uint32_t(k) * 2654435761u) & uint32_t(n_items - 1) : perm[k];
      mb_expect(&full[s], (pairs ? 2 : 1) * gbytes);
      bulk(sm + s * sbytes, pool + size_t(g) * stride, gbytes, &full[s]);
      if (pairs) bulk(sm + s * sbytes + gbytes, pool2 + size_t(g) * stride, gbytes, &full[s]);
    }
  } else if (threadIdx.x == 32) {
    for (int k = k0, i = 0; k < k1; ++k, ++i) {
      const int s = i % nst;
      mb_wait(&full[s], (i / nst) & 1);
      mb_arrive(&empty[s]);
    }
  }
}

int main() {
  const size_t bytes = size_t(6) << 30;  // per pool
  uint8_t *p1, *p2;
  cudaMalloc(&p1, bytes);
  cudaMalloc(&p2, bytes);
  cudaMemset(p1, 1, bytes);
  cudaMemset(p2, 2, bytes);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  struct Cfg { int g, stride, pairs; };
  const Cfg cfgs[] = {{4096, 4096, 1}, {2112, 2112, 1}, {2112, 2112, 0}, {4224, 4224, 0}, {1056, 1056, 1}};
  for (const Cfg& c : cfgs) {
    const int nit = int(bytes / c.stride) - 1;
    uint32_t* ph = new uint32_t[nit];
    for (int i = 0; i < nit; ++i) ph[i] = i;
    unsigned long long s = 88172645463325252ull;
    for (int i = nit - 1; i > 0; --i) {
      s ^= s << 13; s ^= s >> 7; s ^= s << 17;
      int j = int(s % (i + 1));
      uint32_t t = ph[i]; ph[i] = ph[j]; ph[j] = t;
    }
    uint32_t* perm;
    cudaMalloc(&perm, size_t(nit) * 4);
    cudaMemcpy(perm, ph, size_t(nit) * 4, cudaMemcpyHostToDevice);
    delete[] ph;
    const int sbytes = ((c.pairs ? 2 : 1) * c.g + 127) & ~127;
    for (int mode = 0; mode < 4; ++mode) for (int ctas : {2, 3}) for (int nst : {8, 16}) {
      if ((mode & 2) && !c.pairs) continue;
      int nitm = nit;
      if (mode & 1) { nitm = 1; while (2 * nitm <= nit) nitm *= 2; }
      const int smem = nst * sbytes + 2 * nst * 8;
      if (smem * ctas > 220 * 1024) continue;
      cudaFuncSetAttribute(ring_read, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
      const int grid = 148 * ctas;
      ring_read<<<grid, 64, smem>>>(p1, p2, perm, nitm, c.g, c.stride, nst, c.pairs, mode);
      cudaDeviceSynchronize();
      cudaEventRecord(a);
      for (int r = 0; r < 3; ++r) ring_read<<<grid, 64, smem>>>(p1, p2, perm, nitm, c.g, c.stride, nst, c.pairs, mode);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      const double moved = 3.0 * nitm * c.g * (c.pairs ? 2 : 1);
      printf("granule %5d B x %d pool(s), %s, %s, %d CTAs/SM, ring %2d: %7.1f GB/s\n", c.g, c.pairs ? 2 : 1,
             (mode & 1) ? "hashed index" : "index load  ", (mode & 2) ? "2 lanes issue" : "1 thread     ", ctas, nst,
             moved / (ms / 1e3) / 1e9);
    }
    cudaFree(perm);
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
