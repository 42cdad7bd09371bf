// The space-time super-kernel for sm_100a.
//
// One persistent launch executes every tile of a space-time plan: the
// members are independent tenants' conv / GEMM operators, each with its own
// shape, weights and batch (the reference's SuperKernel, scheduler.hpp:37-42;
// the paper's batched-SGEMM super-kernel).  The CTA walks a
// tile-dispatch table (member, m-tile, n-tile) built by the host planner.
//
// Per CTA (256 threads, 1 CTA per SM):
//   warp 0   TMA producer: A tile (2-D tiled map, or 4-D im2col map for
//            implicit-GEMM conv) + B tile (weights, K-major) into a
//            kStages-deep ring of 128B-swizzled smem stages
//   warp 1   MMA issuer: one elected thread issues tcgen05.mma
//            (kind::f16, bf16 x bf16 -> fp32, M=128, N = member width)
//            into a double-buffered TMEM accumulator
//   warp 2   TMEM allocator (256 columns)
//   warps 4-7 epilogue: tcgen05.ld 32x32b -> bf16 -> global (row per thread)
// Pipelines: smem full/empty mbarriers (TMA <-> MMA, tcgen05.commit frees a
// stage), TMEM full/empty mbarriers (MMA <-> epilogue), so the epilogue of
// tile i overlaps the mainloop of tile i+1.
#pragma once

#include <cuda.h>
#include <cuda_bf16.h>
#include <stdint.h>

namespace gmb {
namespace dev {

constexpr int kBM = 128;  // UMMA M; == b200 DeviceSpec.tile_m
constexpr int kBN = 128;  // max UMMA N per tile; == b200 DeviceSpec.tile_n
constexpr int kBK = 64;   // 64 bf16 = 128 B = one SWIZZLE_128B row
constexpr int kStages = 6;
constexpr int kThreads = 256;
constexpr int kABytes = kBM * kBK * 2;
constexpr int kBBytes = kBN * kBK * 2;
constexpr int kAccCols = kBN;
constexpr int kTmemCols = 2 * kAccCols;
constexpr int kSmemBytes = kStages * (kABytes + kBBytes) + 1024 /*align slack*/ + 256 /*barriers*/;

enum : int32_t { kATiled = 0, kAIm2col = 1 };

// Device-resident descriptor of one registered (tenant, layer) operator.
struct alignas(128) MemberDesc {
  CUtensorMap a;        // A operand: [M, K] tiled, or NHWC im2col
  CUtensorMap b;        // B operand: weights [N, K], K-major
  __nv_bfloat16* y;     // output [M, N] row-major
  int64_t ldy;
  int32_t m, n;
  int32_t k_blocks;     // ceil(K / kBK)
  uint32_t idesc;       // tcgen05 instruction descriptor (N of this member)
  int32_t a_mode;
  int32_t pq, q;        // im2col: output pixels per image, output width
  int32_t stride, pad;
  int32_t s_taps;       // filter width S
  int32_t c_blocks;     // Cin / kBK
  int32_t relu;
};

// Device tile-table entry; `member` is the registered slot index.
struct TileEntry {
  uint16_t member, flags, m_tile, n_tile;
};

// ---------------------------------------------------------------- PTX helpers

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  const uint32_t addr = smem_u32(bar);
  uint32_t done = 0;
  do {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(done)
        : "r"(addr), "r"(parity)
        : "memory");
  } while (!done);
}

__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, uint64_t* bar, int32_t c0, int32_t c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(
          smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1)
      : "memory");
}

// im2col: {c, w, h, n} start coordinate of the first output pixel's filter
// window, plus the (s, r) filter-tap offsets.
__device__ __forceinline__ void tma_load_im2col(void* dst, const CUtensorMap* map, uint64_t* bar, int32_t c, int32_t w,
                                                int32_t h, int32_t n, uint16_t off_w, uint16_t off_h) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.im2col.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5, %6}], "
      "[%2], {%7, %8};" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c), "r"(w), "r"(h), "r"(n), "h"(off_w), "h"(off_h)
      : "memory");
}

__device__ __forceinline__ void prefetch_tmap(const CUtensorMap* map) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(map)) : "memory");
}

__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

// SWIZZLE_128B K-major smem matrix descriptor (SM100 format): start >> 4,
// LBO unused (1), SBO = 1024 B between 8-row core-matrix groups, version 1.
__device__ __forceinline__ uint64_t sw128_desc(uint32_t smem_addr) {
  uint64_t d = 0;
  d |= static_cast<uint64_t>((smem_addr >> 4) & 0x3FFFu);
  d |= static_cast<uint64_t>(1u) << 16;
  d |= static_cast<uint64_t>(1024u >> 4) << 32;
  d |= static_cast<uint64_t>(1u) << 46;
  d |= static_cast<uint64_t>(2u) << 61;
  return d;
}

__device__ __forceinline__ void umma_bf16(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc,
                                          uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate)
      : "memory");
}

__device__ __forceinline__ void umma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}

__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&v)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
      "{%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, "
      "%16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]), "=r"(v[8]),
        "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]), "=r"(v[16]),
        "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]),
        "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

__device__ __forceinline__ uint32_t pack_bf16(float lo, float hi, int relu) {
  if (relu) {
    lo = fmaxf(lo, 0.f);
    hi = fmaxf(hi, 0.f);
  }
  __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&v);
}

// ---------------------------------------------------------------- kernel

__global__ void __launch_bounds__(kThreads, 1)
    superkernel(const MemberDesc* __restrict__ slots, const TileEntry* __restrict__ tiles, int n_tiles) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + kStages * kABytes;
  uint64_t* full = reinterpret_cast<uint64_t*>(sB + kStages * kBBytes);
  uint64_t* empty = full + kStages;
  uint64_t* acc_full = empty + kStages;
  uint64_t* acc_empty = acc_full + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_empty + 2);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;

  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&acc_full[a], 1);
      mbar_init(&acc_empty[a], 128);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(kTmemCols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      // ------------------------------------------------ TMA producer
      uint32_t stage = 0, phase = 0;
      for (int t = blockIdx.x; t < n_tiles; t += gridDim.x) {
        const TileEntry te = tiles[t];
        const MemberDesc* md = slots + te.member;
        const int k_blocks = md->k_blocks;
        const int m0 = te.m_tile * kBM;
        const int n0 = te.n_tile * kBN;
        const bool im2col = md->a_mode == kAIm2col;
        int img = 0, h0 = 0, w0 = 0, c_blocks = 1, s_taps = 1;
        if (im2col) {
          img = m0 / md->pq;
          const int rem = m0 - img * md->pq;
          const int p0 = rem / md->q;
          const int q0 = rem - p0 * md->q;
          h0 = p0 * md->stride - md->pad;
          w0 = q0 * md->stride - md->pad;
          c_blocks = md->c_blocks;
          s_taps = md->s_taps;
        }
        for (int kb = 0; kb < k_blocks; ++kb) {
          mbar_wait(&empty[stage], phase ^ 1);
          mbar_expect_tx(&full[stage], kABytes + kBBytes);
          uint8_t* a_dst = sA + stage * kABytes;
          if (im2col) {
            const int tap = kb / c_blocks;
            const int c0 = (kb - tap * c_blocks) * kBK;
            const int r = tap / s_taps;
            const int s = tap - r * s_taps;
            tma_load_im2col(a_dst, &md->a, &full[stage], c0, w0, h0, img, static_cast<uint16_t>(s),
                            static_cast<uint16_t>(r));
          } else {
            tma_load_2d(a_dst, &md->a, &full[stage], kb * kBK, m0);
          }
          tma_load_2d(sB + stage * kBBytes, &md->b, &full[stage], kb * kBK, n0);
          if (++stage == kStages) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      // ------------------------------------------------ MMA issuer
      uint32_t stage = 0, phase = 0, acc = 0, acc_phase = 0;
      for (int t = blockIdx.x; t < n_tiles; t += gridDim.x) {
        const TileEntry te = tiles[t];
        const MemberDesc* md = slots + te.member;
        const int k_blocks = md->k_blocks;
        const uint32_t idesc = md->idesc;
        mbar_wait(&acc_empty[acc], acc_phase ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * kAccCols;
        for (int kb = 0; kb < k_blocks; ++kb) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          const uint32_t a_addr = smem_u32(sA + stage * kABytes);
          const uint32_t b_addr = smem_u32(sB + stage * kBBytes);
#pragma unroll
          for (int k = 0; k < kBK / 16; ++k) {
            // advance 16 bf16 (32 B) along K inside the 128 B swizzle atom
            umma_bf16(d_tmem, sw128_desc(a_addr + k * 32), sw128_desc(b_addr + k * 32), idesc,
                      (kb | k) != 0 ? 1u : 0u);
          }
          umma_commit(&empty[stage]);  // frees the smem stage once these MMAs retire
          if (++stage == kStages) {
            stage = 0;
            phase ^= 1;
          }
        }
        umma_commit(&acc_full[acc]);  // accumulator ready for the epilogue
        acc ^= 1;
        if (acc == 0) acc_phase ^= 1;
      }
    }
  } else if (warp >= 4) {
    // -------------------------------------------------- epilogue (128 threads)
    const int quarter = warp - 4;  // == warp % 4: the TMEM lane quarter this warp may access
    uint32_t acc = 0, acc_phase = 0;
    for (int t = blockIdx.x; t < n_tiles; t += gridDim.x) {
      const TileEntry te = tiles[t];
      const MemberDesc* md = slots + te.member;
      const int m0 = te.m_tile * kBM;
      const int n0 = te.n_tile * kBN;
      const int cols = min(kBN, md->n - n0);  // multiple of 8
      const int row = m0 + quarter * 32 + lane;
      const bool row_ok = row < md->m;
      const int relu = md->relu;
      __nv_bfloat16* yrow = md->y + static_cast<int64_t>(row) * md->ldy + n0;
      mbar_wait(&acc_full[acc], acc_phase);
      tc_fence_after();
      const uint32_t taddr = tmem_base + (static_cast<uint32_t>(quarter * 32) << 16) + acc * kAccCols;
      for (int c = 0; c < cols; c += 32) {
        uint32_t v[32];
        tmem_ld32(taddr + c, v);
        if (row_ok) {
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            if (c + 8 * j < cols) {
              uint4 pk;
              pk.x = pack_bf16(__uint_as_float(v[8 * j + 0]), __uint_as_float(v[8 * j + 1]), relu);
              pk.y = pack_bf16(__uint_as_float(v[8 * j + 2]), __uint_as_float(v[8 * j + 3]), relu);
              pk.z = pack_bf16(__uint_as_float(v[8 * j + 4]), __uint_as_float(v[8 * j + 5]), relu);
              pk.w = pack_bf16(__uint_as_float(v[8 * j + 6]), __uint_as_float(v[8 * j + 7]), relu);
              *reinterpret_cast<uint4*>(yrow + c + 8 * j) = pk;
            }
          }
        }
      }
      tc_fence_before();
      mbar_arrive(&acc_empty[acc]);
      acc ^= 1;
      if (acc == 0) acc_phase ^= 1;
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(kTmemCols) : "memory");
  }
}

// Explicit im2col pre-pass for convs whose Cin does not fill a 128 B TMA
// channel box (e.g. the 3-channel stem): writes [M, ldk] bf16 rows with
// k = (r*S + s)*Cin + c and zero padding, consumed as a plain GEMM A operand.
__global__ void im2col_prepass(const __nv_bfloat16* __restrict__ x, __nv_bfloat16* __restrict__ out, int batch, int H,
                               int W, int Cin, int R, int S, int stride, int pad, int P, int Q, int ldk) {
  const int64_t total = static_cast<int64_t>(batch) * P * Q * ldk;
  const int K = R * S * Cin;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t m = i / ldk;
    const int k = static_cast<int>(i - m * ldk);
    __nv_bfloat16 v = __float2bfloat16(0.f);
    if (k < K) {
      const int c = k % Cin;
      const int tap = k / Cin;
      const int s = tap % S, r = tap / S;
      const int q = static_cast<int>(m % Q);
      const int p = static_cast<int>((m / Q) % P);
      const int b = static_cast<int>(m / (static_cast<int64_t>(P) * Q));
      const int ih = p * stride - pad + r, iw = q * stride - pad + s;
      if (ih >= 0 && ih < H && iw >= 0 && iw < W) v = x[((static_cast<int64_t>(b) * H + ih) * W + iw) * Cin + c];
    }
    out[i] = v;
  }
}

}  // namespace dev
}  // namespace gmb
