// TMA feed micro-benchmark (debug aid, not product code): one CTA per SM, a
// producer thread streams 2-D tiled boxes (A rows x 128 B and B rows x 128 B
// per stage) from an L2-resident buffer into a ring of `stages` smem stages;
// a consumer thread waits on each stage and frees it (optionally after a
// spin of `work` cycles standing in for the MMA).  Reports bytes/s per SM.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tma_micro tma_micro.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

__device__ __forceinline__ uint32_t sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void wait(uint64_t* b, uint32_t par) {
  uint32_t done = 0;
  do {
    asm volatile("{.reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p;}"
                 : "=r"(done) : "r"(sa(b)), "r"(par) : "memory");
  } while (!done);
}

__device__ __forceinline__ uint64_t sw128(uint32_t addr) {
  return (uint64_t)((addr >> 4) & 0x3FFF) | (1ull << 16) | ((uint64_t)(1024 >> 4) << 32) | (1ull << 46) | (2ull << 61);
}

__global__ void __launch_bounds__(128, 1) feed(const __grid_constant__ CUtensorMap ma, const __grid_constant__ CUtensorMap mb,
                                               int iters, int stages, int a_rows, int b_rows, int work, int rows_total,
                                               unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* ring = (uint8_t*)(((uintptr_t)sm + 1023) & ~(uintptr_t)1023);
  const int stage_bytes = (a_rows + b_rows) * 128;
  uint64_t* full = (uint64_t*)(ring + stages * stage_bytes);
  uint64_t* empty = full + 16;
  if (threadIdx.x == 0) {
    for (int i = 0; i < 16; ++i) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&full[i])));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(sa(&empty[i])), "r"(work == 5 ? 2 : 1));
    }
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __shared__ uint32_t tslot;
  if (threadIdx.x / 32 == 2) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(sa(&tslot)) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem_base = tslot;
  unsigned long long t0 = clock64();
  unsigned long long tw = 0, ti = 0;
  if (threadIdx.x == 0) {
    for (int i = 0; i < iters; ++i) {
      const int s = i % stages;
      const unsigned long long c0 = clock64();
      wait(&empty[s], ((i / stages) & 1) ^ 1);
      const unsigned long long c1 = clock64();
      tw += c1 - c0;
      uint8_t* dst = ring + s * stage_bytes;
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(&full[s])), "r"(stage_bytes));
      const int row = ((blockIdx.x * 7 + i) * a_rows) % rows_total;
      asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];"
                   ::"r"(sa(dst)), "l"((uint64_t)&ma), "r"(sa(&full[s])), "r"(0), "r"(row) : "memory");
      const int brow = ((blockIdx.x * 3 + i) * b_rows) % rows_total;
      if (b_rows) asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];"
                   ::"r"(sa(dst + a_rows * 128)), "l"((uint64_t)&mb), "r"(sa(&full[s])), "r"(0), "r"(brow) : "memory");
      ti += clock64() - c1;
    }
  } else if (work == 5 && (threadIdx.x == 32 || threadIdx.x == 64)) {
    // two issuing threads (warps 1 and 2), 4 MMAs each per stage into their
    // own accumulator columns; each commit is one of the stage's two arrivals
    const uint32_t dcol = threadIdx.x == 64 ? 256u : 0u;
    for (int i = 0; i < iters; ++i) {
      const int s = i % stages;
      wait(&full[s], (i / stages) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const uint32_t a = sa(ring + s * stage_bytes), b = a + a_rows * 128;
      const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(b_rows >> 3) << 17) | ((128u >> 4) << 24);
      for (int k = 0; k < 4; ++k) {
        const uint64_t da = sw128(a + k * 32), db = sw128(b + k * 32);
        asm volatile("{.reg .pred p; setp.ne.b32 p, %4, 0; tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;}"
                     ::"r"(tmem_base + dcol), "l"(da), "l"(db), "r"(idesc), "r"(1));
      }
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(sa(&empty[s])) : "memory");
    }
  } else if (threadIdx.x == 32) {
    for (int i = 0; i < iters; ++i) {
      const int s = i % stages;
      wait(&full[s], (i / stages) & 1);
      if (work >= 1 && work <= 4) {
        // real tcgen05.mma: 4 x (M=128, N=b_rows, K=16) from the stage, commit frees it
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint32_t a = sa(ring + s * stage_bytes), b = a + a_rows * 128;
        const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(b_rows >> 3) << 17) | ((128u >> 4) << 24);
        // work 1: 4 MMAs (one K=64 k-block), 2: 8 (the k-block twice), 3: 2, 4: 1
        const int nmma = work == 1 ? 4 : work == 2 ? 8 : work == 3 ? 2 : 1;
        for (int k = 0; k < nmma; ++k) {
          const uint64_t da = sw128(a + (k & 3) * 32), db = sw128(b + (k & 3) * 32);
          asm volatile("{.reg .pred p; setp.ne.b32 p, %4, 0; tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;}"
                       ::"r"(tmem_base), "l"(da), "l"(db), "r"(idesc), "r"(1));
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(sa(&empty[s])) : "memory");
        continue;
      }
      if (work) {
        __nanosleep(work);
      }
      asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(sa(&empty[s])) : "memory");
    }
  }
  if ((threadIdx.x == 32 && ((work >= 1 && work <= 4) || work == 5))) wait(&empty[(iters - 1) % stages], ((iters - 1) / stages) & 1);
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (threadIdx.x == 0) {
    out[blockIdx.x] = clock64() - t0;
    if (blockIdx.x == 0) printf("    producer: wait %.1f issue %.1f cyc/iter\n", (double)tw / iters, (double)ti / iters);
  }
  if (threadIdx.x / 32 == 2) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem_base) : "memory");
  }
}

typedef CUresult (*EncFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                          const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                          CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main(int argc, char** argv) {
  const int rows_total = 1 << 16;  // 65536 rows x 128 B = 8 MB (L2 resident)
  void* buf;
  cudaMalloc(&buf, (size_t)rows_total * 128);
  cudaMemset(buf, 1, (size_t)rows_total * 128);
  EncFn enc;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaFuncSetAttribute(feed, cudaFuncAttributeMaxDynamicSharedMemorySize, 226 * 1024);
  unsigned long long* d_out;
  cudaMalloc(&d_out, sms * sizeof(unsigned long long));
  unsigned long long h[256];
  int clk;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  struct Cfg { int a, b, stages, ctas, work; } cfgs[] = {
      {128, 256, 4, 8, 0},   {128, 256, 4, 8, 1},   {128, 256, 3, 8, 1},   {128, 256, 4, 148, 1}, {128, 256, 4, 8, 250},
      {128, 128, 6, 8, 1},   {128, 128, 4, 8, 1},   {128, 128, 6, 148, 1}, {128, 64, 8, 8, 1},    {128, 64, 4, 8, 1},
      {128, 64, 8, 148, 1},  {64, 64, 8, 8, 250},   {64, 64, 8, 8, 0},     {8, 8, 8, 8, 500},     {8, 8, 2, 8, 500},
      // one TMA per stage (no B box): is the floor per instruction or per stage?
      {128, 0, 4, 8, 0},     {256, 0, 4, 8, 0},     {8, 0, 4, 8, 0},       {128, 0, 8, 148, 0},
      // two issuing warps x 4 MMAs per stage (work 5) vs one warp x 8 (work 2)
      {128, 64, 8, 8, 5},    {128, 128, 6, 8, 5},   {128, 256, 4, 8, 5},
      // MMAs per stage: 8 / 2 / 1 (work 2 / 3 / 4)
      {128, 256, 4, 8, 2},   {128, 256, 4, 8, 3},   {128, 256, 4, 8, 4},   {128, 128, 6, 8, 2},   {128, 128, 6, 8, 3},
      {128, 128, 6, 8, 4},   {128, 64, 8, 8, 2},    {128, 64, 8, 8, 4},
  };
  for (auto& c : cfgs) {
    CUtensorMap ma, mb;
    cuuint64_t dims[2] = {64, (cuuint64_t)rows_total};
    cuuint64_t str[1] = {128};
    cuuint32_t boxa[2] = {64, (cuuint32_t)c.a}, boxb[2] = {64, (cuuint32_t)(c.b ? c.b : 8)}, es[2] = {1, 1};
    enc(&ma, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, buf, dims, str, boxa, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
        CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    enc(&mb, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, buf, dims, str, boxb, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
        CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    const int iters = 2000;
    for (int rep = 0; rep < 2; ++rep)
      feed<<<c.ctas, 128, 226 * 1024>>>(ma, mb, iters, c.stages, c.a, c.b, c.work, rows_total, d_out);
    cudaError_t e = cudaGetLastError();
    if (e == cudaSuccess) e = cudaDeviceSynchronize();
    if (e != cudaSuccess) {
      printf("error %s\n", cudaGetErrorString(e));
      return 1;
    }
    cudaMemcpy(h, d_out, c.ctas * sizeof(unsigned long long), cudaMemcpyDeviceToHost);
    double mx = 0;
    for (int i = 0; i < c.ctas; ++i) mx = h[i] > mx ? h[i] : mx;
    const double cyc_per = mx / iters;
    const double bytes = (c.a + c.b) * 128.0;
    printf("A%3d B%3d stages %d ctas %3d work %4d: %7.1f cyc/stage  %6.1f B/cyc/SM  %7.1f GB/s/SM  chip %6.2f TB/s\n",
           c.a, c.b, c.stages, c.ctas, c.work, cyc_per, bytes / cyc_per, bytes / cyc_per * clk * 1e3 / 1e9,
           bytes / cyc_per * clk * 1e3 * c.ctas / 1e12);
  }
  return 0;
}
