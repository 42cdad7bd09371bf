// The space-time super-kernel for sm_100a.
//
// One persistent launch executes every tile of a space-time plan: the
// members are independent tenants' conv / GEMM operators, each with its own
// shape, weights and batch (the reference's SuperKernel, scheduler.hpp:37-42;
// the paper's batched-SGEMM super-kernel).  The CTA walks a
// tile-dispatch table (member, m-tile, n-tile) built by the host planner.
//
// Per CTA (256 threads, 1 CTA per SM), templated on the N tile (128 | 256):
//   warp 0    TMA producer: A tile (2-D tiled map, or 4-D im2col map for
//             implicit-GEMM conv) + B tile (weights, K-major) into a ring of
//             128B-swizzled smem stages; boxes are sized per member, so a
//             small-M or small-N member moves only its real bytes
//   warp 1    MMA issuer: one thread issues tcgen05.mma (kind::f16,
//             bf16 x bf16 -> fp32, M=128, N = the member's box) into a
//             double-buffered TMEM accumulator
//   warp 2    TMEM allocator (2 x BN columns)
//   warps 4-7 epilogue: tcgen05.ld 32x32b -> bf16 -> 64B-swizzled smem
//             staging -> TMA bulk store (coalesced, clipped at M/N edges)
// Pipelines: smem full/empty mbarriers (TMA <-> MMA; tcgen05.commit frees a
// stage), TMEM full/empty mbarriers (MMA <-> epilogue), bulk-group waits on
// the double-buffered store staging.  Launches chain with programmatic
// dependent launch: the weights of the first stages stream before
// griddepcontrol.wait, activations after it.
#pragma once

#include <cuda.h>
#include <cuda_bf16.h>
#include <stdint.h>

#include <type_traits>

namespace gmb {
namespace dev {

constexpr int kBM = 128;  // UMMA M; == b200 DeviceSpec.tile_m
constexpr int kIdentN = 256;  // identity matrix side (the widest N tile): residual k-blocks' B operand
constexpr int kBK = 64;   // 64 bf16 = 128 B = one SWIZZLE_128B row
constexpr int kThreads = 384;  // 4 control warps + 2 epilogue warpgroups
constexpr int kABytes = kBM * kBK * 2;
constexpr int kEpiChunk = 32;                         // columns per store box
constexpr int kEpiBufBytes = 32 * kEpiChunk * 2;      // 32 rows x 32 cols bf16
#ifndef GMB_EPI_BUFS
#define GMB_EPI_BUFS 2
#endif
#ifndef GMB_WIDE_STAGES
#define GMB_WIDE_STAGES 4
#endif
constexpr int kEpiBufs = GMB_EPI_BUFS;                // store staging buffers per epilogue warp
constexpr int kEpiBytes = 8 * kEpiBufs * kEpiBufBytes;  // 8 epilogue warps

template <int BN>
struct Cfg {
  static_assert(BN == 128 || BN == 256, "N tile must be 128 or 256");
  static constexpr int kStages = BN == 256 ? GMB_WIDE_STAGES : 6;
  static constexpr int kBBytes = BN * kBK * 2;
  static constexpr int kStageBytes = kABytes + kBBytes;
  static constexpr int kTmemCols = 2 * BN;
  static constexpr int kSmemBytes = kStages * kStageBytes + kEpiBytes + 1024 /*align*/ + 1024 /*barriers, tile ring*/;
  // Two ring layouts over the same bytes: wide (kStages slots of kStageBytes)
  // and narrow (32 KB slots) for members whose stage fits in 32 KB (N tile
  // <= 128), which then keep more k-blocks in flight -- their k-block rate
  // is set by operand latency.  Switching layout drains the ring.
  static constexpr int kNarrowBytes = 32768;
  static constexpr int kNarrowSlots = kStages * kStageBytes / kNarrowBytes;
  static constexpr int kMaxSlots = kNarrowSlots > kStages ? kNarrowSlots : kStages;
  // A tall tile's stage: two 128-row A boxes and a <= 128-row B box; its second
  // accumulator half starts at column 128 of the tile's BN-column buffer.
  static constexpr bool kTallFits = 2 * kABytes + 128 * kBK * 2 <= kStageBytes && 128 + 128 <= BN;
};
static_assert(Cfg<256>::kTallFits, "tall tiles need the 256-column ring slot");

// A-operand modes: 2-D tiled box; TMA im2col (C_in % 64 == 0: one 128 B
// channel block per k-block, SW128); narrow-channel TMA im2col (input pixel
// pitch of 8 channels: eight 16 B tap columns per k-block, SWIZZLE_NONE).
// Row-folded mode (S * C_in <= 32, e.g. the 7x7 RGB stem): a pre-pass folds
// each output column's horizontal window into one 32-channel "pixel"
// (X'[b, h, q, s*C_in + c]); the conv becomes R x 1 with vertical stride,
// two 64 B (SW64) TMA im2col columns per k-block.
enum : int32_t { kATiled = 0, kAIm2col = 1, kAIm2colNarrow = 2, kAIm2colFold = 3, kDepthwise = 4, kMaxPool = 5,
                 kAvgPool = 6 };
// Modes >= kDepthwise are CUDA-core tile types (no TMA / MMA pipeline): the
// eight epilogue warps compute them.  Max / average pooling (ResNet's stem
// maxpool and global avgpool, VGG's 2x2 pools, MobileNet-v2's avgpool) sit
// between convs on a tenant's dataflow chain, so they are tiles of the same
// persistent launch, gated on the same dependency counters.
__host__ __device__ constexpr bool cuda_core_mode(int32_t m) { return m >= kDepthwise; }
// Epilogue activations (applied after the residual add).
enum : int32_t { kActNone = 0, kActRelu = 1, kActRelu6 = 2, kActGelu = 3 };
// Depthwise conv (MobileNet-v2) is a CUDA-core tile type inside the same
// persistent kernel (tensor cores do not apply: one filter per channel).  Its
// tiles skip the TMA/MMA pipeline; the eight epilogue warps compute them
// directly (kDwPixW output pixels each x kDwTileC channels, 4 channels per
// lane).  Tiles are short (kDwTileM pixels) so a layer spreads over many SMs:
// a depthwise layer sits on its tenant's chain, its latency is one tile's.
constexpr int kDwTileC = 128;
constexpr int kDwPixW = 4;               // output pixels per epilogue warp
constexpr int kDwTileM = 8 * kDwPixW;    // output pixels per depthwise tile
constexpr int kDwMaxTaps = 9;
constexpr int kNarrowC = 8;                     // channels per pixel of a narrow-im2col input
constexpr int kNarrowTaps = kBK / kNarrowC;     // filter taps per k-block
constexpr int kNarrowTapBytes = kBM * kNarrowC * 2;  // one tap column: 128 pixels x 16 B
constexpr int kFoldC = 32;                      // channels per folded pixel (64 B)
constexpr int kFoldTaps = kBK / kFoldC;         // filter rows per k-block
constexpr int kFoldTapBytes = kBM * kFoldC * 2;  // one filter-row column: 128 pixels x 64 B

// Device-resident descriptor of one registered (tenant, layer) operator.
struct alignas(128) MemberDesc {
  CUtensorMap a;        // A operand: [M, K] tiled, or NHWC im2col
  CUtensorMap b;        // B operand: weights [N, K], K-major
  CUtensorMap c;        // output [M, N] row-major, store box 32 x 32
  // Fused residual add as extra k-blocks of the same MMA: y = [A | R] [W ; I]
  // over the tile's columns.  r: the residual [M, N] as an A operand (box 64
  // columns x A-box rows, SW128); id: a bf16 identity as the B operand (box 64
  // x B-box rows).  ceil(cols / 64) extra k-blocks per tile add R exactly in
  // the fp32 accumulator, streamed by TMA through the operand ring.
  CUtensorMap r;
  CUtensorMap id;
  int32_t m, n;
  int32_t k_blocks;     // ceil(K / kBK)
  uint32_t idesc;       // tcgen05 instruction descriptor (N = B box rows)
  uint32_t tx_bytes;    // A box + B box bytes per k-block
  int32_t a_mode;
  int32_t pq, q;        // im2col: output pixels per image, output width
  int32_t stride, pad;
  int32_t s_taps;       // filter width S
  int32_t c_blocks;     // Cin / kBK
  int32_t act;          // kAct*: fused activation
  int32_t n_tile;       // output columns per tile (<= BN): narrower for few-tile members
  int32_t taps;         // narrow im2col: R*S filter taps
  int32_t images;       // narrow im2col: batch (an out-of-range image zero-fills a box)
  // Tall tile (N tile <= 128, tiled / im2col A only): 256 output rows as two
  // 128-row halves sharing one B box -- two A boxes per k-block, two UMMAs
  // per K step into accumulator columns [0, n_tile) and [n_tile, 2 n_tile).
  // Doubles the work per k-block of a narrow tile, whose k-block rate is set
  // by operand latency, not by the tensor pipe.
  int32_t tall;
  int32_t ring_narrow;  // 1: the stage (A region + B box) fits a 32 KB narrow-layout slot
  // depthwise members: raw operands and geometry (x NHWC [b, H, W, C],
  // w [C, ldw] with R*S taps per row, y [b*P*Q, C])
  const __nv_bfloat16* dx;
  const __nv_bfloat16* dw;
  __nv_bfloat16* dy;
  int32_t h_in, w_in, ch, r_taps, ldw;
  // fused residual add (ResNet's identity / downsample add, MobileNet-v2's
  // inverted-residual add, BERT's skip connections): y = act(acc + res), res
  // [M, N] row-major bf16 with row stride ldr; null = none.  The residual is
  // an earlier layer of the same tenant, complete by the dependency chain the
  // producer gates on; it enters the accumulator through maps r / id.
  const __nv_bfloat16* res;
  int32_t ldr;
  // Staged CUDA-core tiles (pools, depthwise; 0 = register path): output rows
  // per tile.  The producer lands a tile's whole input window -- box
  // {n_tile channels, (q-1)*stride+S columns, (cc_rows-1)*stride+R rows, 1
  // image} of the NHWC input through map `a` -- in one operand-ring stage
  // (tx_bytes; ring_narrow when it fits a 32 KB slot), so the loads of later
  // tiles stream while one epilogue warpgroup computes this one from smem.
  int32_t cc_rows;
  const __nv_bfloat16* dwt;  // staged depthwise: the filters tap-major [R*S][ch] (16-byte channel groups)
};

// Device tile-table entry; `member` is the registered slot index.
// In a round program (one persistent launch for a whole space-time round),
// every output row block (m-tile) of a member instance has a completion
// counter: `done` is the tile's.  A tile's activations are loaded only once
// the producer m-tiles holding its input rows are stored: counters
// [dep, dep + dep_n) (its input's producing layer) and [rdep, rdep + rdep_n)
// (its residual's), -1 = none.  So consecutive layers overlap row block by
// row block instead of meeting at a per-layer barrier.
//
// Split-K (round programs, few-tile long-K members): `splits` > 1 tiles each
// cover k-blocks [kb_begin, kb_end) of output tile `ws`; they reduce-add fp32
// partials into a workspace tile with TMA, and the last split to arrive
// converts the sum to bf16, stores it, clears the workspace and publishes.
struct TileEntry {
  uint16_t member, splits, m_tile, n_tile;
  int32_t done, dep;
  uint16_t kb_begin, kb_end;  // kb_end == 0: the whole K
  int32_t ws;                 // split workspace tile (-1 = not split)
  int32_t rdep;
  uint16_t dep_n, rdep_n;
};

// The producer's per-tile inputs: the tile entry and the member's scalar
// fields (a copy of MemberDesc m .. ring_narrow, plus cc_rows and whether a
// residual is fused).  The scheduler lane fills one per claimed tile in shared
// memory, so the producer -- the single issuing thread that paces narrow
// tiles -- reads its tile's setup from smem instead of two dependent L2 round
// trips (tile entry, then descriptor) per tile.
struct MemberScalars {
  int32_t m, n, k_blocks;
  uint32_t idesc, tx_bytes;
  int32_t a_mode, pq, q, stride, pad, s_taps, c_blocks, act, n_tile, taps, images, tall, ring_narrow;
};
static_assert(sizeof(MemberScalars) == 72, "MemberScalars mirrors MemberDesc m .. ring_narrow");
struct alignas(16) TileRec {
  TileEntry te;
  MemberScalars ms;
  int32_t cc_rows;
  int32_t has_res;
  // im2col start of the tile (tall: of each 128-row half) and the K walk's
  // first (channel block, filter column, filter row); staged CUDA-core tiles:
  // the input window's image and first row
  int32_t img, h0, w0, img1, h1, w1, cb, r_, s_;
};
static_assert(offsetof(MemberDesc, ring_narrow) - offsetof(MemberDesc, m) == sizeof(MemberScalars) - 4,
              "MemberScalars must match MemberDesc's scalar block");

__device__ __forceinline__ void load_tile_rec(const TileEntry* __restrict__ tiles, const MemberDesc* __restrict__ slots,
                                              int t, TileRec& r) {
  r.te = tiles[t];
  const MemberDesc* md = slots + r.te.member;
  r.ms = *reinterpret_cast<const MemberScalars*>(&md->m);
  r.cc_rows = md->cc_rows;
  r.has_res = md->res != nullptr;
  // the producer's integer divisions, done here (off the issuing thread)
  const MemberScalars& ms = r.ms;
  const TileEntry& te = r.te;
  r.img = r.h0 = r.w0 = r.img1 = r.h1 = r.w1 = r.cb = r.r_ = r.s_ = 0;
  if (cuda_core_mode(ms.a_mode)) {
    if (r.cc_rows > 0) {
      const int m0 = te.m_tile * r.cc_rows * ms.q;
      r.img = m0 / ms.pq;
      r.h0 = (m0 - r.img * ms.pq) / ms.q * ms.stride - ms.pad;
    }
  } else if (ms.a_mode != kATiled) {
    const bool fold = ms.a_mode == kAIm2colFold;
    const int m0 = te.m_tile * (kBM << ms.tall);
    r.img = m0 / ms.pq;
    int rem = m0 - r.img * ms.pq;
    int p = rem / ms.q;
    int q = rem - p * ms.q;
    r.h0 = p * ms.stride - ms.pad;
    r.w0 = fold ? q : q * ms.stride - ms.pad;  // folded columns are already strided
    if (ms.tall) {
      const int m1 = m0 + kBM;
      r.img1 = m1 / ms.pq;
      rem = m1 - r.img1 * ms.pq;
      p = rem / ms.q;
      q = rem - p * ms.q;
      r.h1 = p * ms.stride - ms.pad;
      r.w1 = fold ? q : q * ms.stride - ms.pad;
    }
    if (ms.a_mode == kAIm2col) {
      const int kb_lo = te.kb_end ? te.kb_begin : 0;
      const int tap = kb_lo / ms.c_blocks;
      r.cb = kb_lo - tap * ms.c_blocks;
      r.r_ = tap / ms.s_taps;
      r.s_ = tap - r.r_ * ms.s_taps;
    }
  }
}

// Wait until every counter of [first, first + n) reached its target (acquire).
__device__ __forceinline__ void wait_range(const uint32_t* counters, const uint32_t* targets, int32_t first, int n,
                                           uint32_t sleep_ns);
// Whether every counter of [first, first + n) reached its target (no wait).
__device__ __forceinline__ bool range_ready(const uint32_t* counters, const uint32_t* targets, int32_t first, int n);

// Round-program side state (all null for a plain super-kernel launch).
//
// Dynamic scheduling (round programs): the tiles are grouped into one work
// queue per tenant (tiles [qbeg[q], qbeg[q] + qlen[q]) in that tenant's plan
// order).  A CTA claims the head of any queue whose head tile's dependency is
// already satisfied (atomicCAS on heads[q]), so a tenant blocked at a layer
// boundary never idles SMs another tenant could use and tenants desynchronise
// instead of running in lock-step.  Claimed tiles never wait, so the claim
// order cannot deadlock.  heads == nullptr selects the static schedule.
struct RoundArgs {
  uint32_t* counters;         // per member instance: tile-quarters stored
  const uint32_t* targets;
  const CUtensorMap* ws_map;  // (unused; kept for ABI stability of the struct)
  float* ws;                  // split-K workspace, lane-major fp32
  uint32_t* split_ctr;        // per workspace tile and quarter: splits arrived
  uint64_t* trace;            // 6 %globaltimer stamps per tile (profiling)
  uint32_t* heads;            // per queue: next unclaimed position
  const int32_t* qbeg;
  const int32_t* qlen;
  int32_t nq;
  uint32_t* next_tile;        // greedy schedule: one global in-order claim counter (null = static / queues)
  uint32_t* exit_ctr;         // CTAs finished; the last one zeroes counters[0, n_reset) for the next launch
  int32_t n_reset;
};

constexpr int kTileQ = 8;   // claimed-tile ring between producer and consumers
constexpr int kDwTag = 1 << 30;  // tile-ring tag: a depthwise tile (no TMA / MMA work)
constexpr int kStagedTag = 1 << 29;  // with kDwTag: a staged CUDA-core tile (one ring stage, no MMA)
constexpr int kSchedQ = 2;  // scheduler look-ahead: tiles claimed (and their records loaded) before the producer needs them
constexpr int kPubQ = 4;    // per epilogue warpgroup: staged-tile publishes queued for the publisher warp

__device__ __forceinline__ bool elect_one() {
  uint32_t p = 0;
  asm volatile("{\n\t.reg .pred P;\n\telect.sync _|P, 0xffffffff;\n\tselp.b32 %0, 1, 0, P;\n\t}" : "=r"(p));
  return p != 0;
}

__device__ __forceinline__ uint64_t globaltimer() {
  uint64_t t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

__device__ __forceinline__ uint32_t ld_acquire(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// Wait until *ctr >= want (acquire).  A dependency that never resolves (a
// broken launch program) traps after ~4 s instead of hanging the GPU.
__device__ __forceinline__ void wait_counter(const uint32_t* ctr, uint32_t want, uint32_t sleep_ns) {
  uint32_t spins = 0;
  uint64_t t0 = 0;
  while (ld_acquire(ctr) < want) {
    __nanosleep(sleep_ns);
    if ((++spins & 4095u) == 0) {
      const uint64_t now = globaltimer();
      if (t0 == 0)
        t0 = now;
      else if (now - t0 > 4000000000ull)
        __trap();
    }
  }
}

__device__ __forceinline__ void wait_range(const uint32_t* counters, const uint32_t* targets, int32_t first, int n,
                                           uint32_t sleep_ns) {
  for (int i = 0; i < n; ++i) wait_counter(counters + first + i, targets[first + i], sleep_ns);
}

__device__ __forceinline__ bool range_ready(const uint32_t* counters, const uint32_t* targets, int32_t first, int n) {
  for (int i = 0; i < n; ++i)
    if (ld_acquire(counters + first + i) < targets[first + i]) return false;
  return true;
}

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

__device__ __forceinline__ bool mbar_test(uint64_t* bar, uint32_t parity) {
  uint32_t done = 0;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(done)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return done != 0;
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

// 4-D tiled box {c, w, h, n} (signed start; out-of-bounds elements zero-fill).
__device__ __forceinline__ void tma_load_4d(void* dst, const CUtensorMap* map, uint64_t* bar, int32_t c, int32_t w,
                                            int32_t h, int32_t n) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5, %6}], "
      "[%2];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c), "r"(w), "r"(h), "r"(n)
      : "memory");
}

// Release-add on a round counter (orders the prior writes this thread observed,
// including those of threads it synchronised with through a barrier).
__device__ __forceinline__ void red_release_add(uint32_t* p, uint32_t v) {
  asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

__device__ __forceinline__ void named_barrier(int id, int threads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(threads) : "memory");
}

__device__ __forceinline__ void tma_store_2d(const CUtensorMap* map, const void* src, int32_t c0, int32_t c1) {
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];" ::"l"(
                   reinterpret_cast<uint64_t>(map)),
               "r"(smem_u32(src)), "r"(c0), "r"(c1)
               : "memory");
}

// Bulk L2 prefetch of one tensor box (no smem destination, no completion).
__device__ __forceinline__ void prefetch_box_l2(const CUtensorMap* map, int32_t c0, int32_t c1) {
  asm volatile("cp.async.bulk.prefetch.tensor.2d.L2.global.tile [%0, {%1, %2}];" ::"l"(
                   reinterpret_cast<uint64_t>(map)),
               "r"(c0), "r"(c1)
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

// SWIZZLE_64B K-major descriptor: 64 B rows, SBO = 512 B between 8-row groups.
__device__ __forceinline__ uint64_t sw64_desc(uint32_t smem_addr) {
  uint64_t d = 0;
  d |= static_cast<uint64_t>((smem_addr >> 4) & 0x3FFFu);
  d |= static_cast<uint64_t>(1u) << 16;
  d |= static_cast<uint64_t>(512u >> 4) << 32;
  d |= static_cast<uint64_t>(1u) << 46;
  d |= static_cast<uint64_t>(4u) << 61;
  return d;
}

// SWIZZLE_NONE K-major descriptor: 8-row x 16 B core matrices contiguous,
// SBO = 128 B to the next 8 rows, LBO = one narrow tap column to the next 8
// K elements.
__device__ __forceinline__ uint64_t interleave_desc(uint32_t smem_addr) {
  uint64_t d = 0;
  d |= static_cast<uint64_t>((smem_addr >> 4) & 0x3FFFu);
  d |= static_cast<uint64_t>(kNarrowTapBytes >> 4) << 16;
  d |= static_cast<uint64_t>(128u >> 4) << 32;
  d |= static_cast<uint64_t>(1u) << 46;
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

// Activations: relu / relu6 are a clamp [lo, hi] applied while packing
// (branch-free, two instructions); GELU runs out of line over a whole chunk
// before packing (its erf would otherwise be inlined into every unrolled
// packing site and bloat the kernel's instruction footprint).
struct Clamp {
  float lo, hi;
};
__device__ __forceinline__ Clamp clamp_of(int act) {
  return Clamp{act == kActRelu || act == kActRelu6 ? 0.f : -INFINITY, act == kActRelu6 ? 6.f : INFINITY};
}

// GELU, erf form (BERT's FFN): erf by Abramowitz-Stegun 7.1.26 (|error| <=
// 1.5e-7, far below bf16 rounding) -- one reciprocal and one exp2 on the SFU
// plus five FMAs, instead of a call to erff per element.
__device__ __forceinline__ float gelu_f(float x) {
  const float u = fabsf(x) * 0.70710678118654752f;
  const float t = __fdividef(1.f, fmaf(0.3275911f, u, 1.f));
  float p = fmaf(1.061405429f, t, -1.453152027f);
  p = fmaf(p, t, 1.421413741f);
  p = fmaf(p, t, -0.284496736f);
  p = fmaf(p, t, 0.254829592f);
  const float erf_u = 1.f - p * t * __expf(-u * u);
  return 0.5f * x * (1.f + copysignf(erf_u, x));
}

// Two fp32 -> bf16x2 (round to nearest even) in one instruction; the .relu
// form clamps negatives to 0 in the same instruction.
__device__ __forceinline__ uint32_t cvt_bf16x2(float lo, float hi) {
  uint32_t r;
  asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo));
  return r;
}
__device__ __forceinline__ uint32_t cvt_bf16x2_relu(float lo, float hi) {
  uint32_t r;
  asm("cvt.rn.relu.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo));
  return r;
}

__device__ __forceinline__ uint32_t pack_bf16(uint32_t lo_bits, uint32_t hi_bits, Clamp k) {
  const float lo = fminf(fmaxf(__uint_as_float(lo_bits), k.lo), k.hi);
  const float hi = fminf(fmaxf(__uint_as_float(hi_bits), k.lo), k.hi);
  __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&v);
}


// Depthwise tile (CUDA cores): epilogue warp `ew` (0..7) computes output
// pixels [m_tile*128 + ew*16, +16) x channels [n_tile*kDwTileC + 4*lane, +4)
// in fp32 from bf16 NHWC input and [C, R*S] filters; one 8-byte load per tap
// and pixel per lane (a warp reads 256 contiguous bytes of channels).
__device__ __forceinline__ void depthwise_tile(const MemberDesc* __restrict__ md, const TileEntry& te, int ew, int lane) {
  const int M = md->m, C = md->ch, H = md->h_in, W = md->w_in;
  // lanes -> (channel group of 4, pixel): a narrow channel tile packs several
  // pixels per warp instruction instead of idling lanes
  const int cbase = te.n_tile * kDwTileC;
  const int g = min(kDwTileC, C - cbase) >> 2;  // channel groups in this tile
  const int gp = g <= 8 ? 8 : (g <= 16 ? 16 : 32);
  const int pp = 32 / gp;  // pixels per pass
  const int cg = lane & (gp - 1), sub = lane / gp;
  if (cg >= g) return;
  const int c = cbase + cg * 4;
  const int taps = md->r_taps, S = md->s_taps, st = md->stride, pad = md->pad, PQ = md->pq, Q = md->q;
  const Clamp ck = clamp_of(md->act);  // depthwise activations: none / relu / relu6
  float wv[4][kDwMaxTaps];
#pragma unroll
  for (int j = 0; j < 4; ++j)
#pragma unroll
    for (int k = 0; k < kDwMaxTaps; ++k)
      wv[j][k] = k < taps ? __bfloat162float(md->dw[static_cast<int64_t>(c + j) * md->ldw + k]) : 0.f;
  // kDwPixW pixels per warp: this lane's are m_base + pp * i.  Tap-major over
  // groups of kG pixels keeps kG independent loads in flight per tap.
  constexpr int kG = 4;
  const int m_base = te.m_tile * kDwTileM + ew * kDwPixW + sub;
  const int npx = (kDwPixW + pp - 1) / pp;
  for (int i0 = 0; i0 < npx; i0 += kG) {
    int bb[kG], hh[kG], ww[kG];
    float acc[kG][4];
#pragma unroll
    for (int j = 0; j < kG; ++j) {
      const int m = m_base + pp * (i0 + j);
      const bool ok = i0 + j < npx && m < M;
      const int b = ok ? m / PQ : -1;
      const int rem = m - b * PQ;
      const int p = rem / Q;
      bb[j] = b;
      hh[j] = p * st - pad;
      ww[j] = (rem - p * Q) * st - pad;
      acc[j][0] = acc[j][1] = acc[j][2] = acc[j][3] = 0.f;
    }
#pragma unroll
    for (int k = 0; k < kDwMaxTaps; ++k) {
      if (k >= taps) break;
      const int r = k / S, s = k - r * S;
      uint2 raw[kG];
#pragma unroll
      for (int j = 0; j < kG; ++j) {
        const int ih = hh[j] + r, iw = ww[j] + s;
        raw[j] = make_uint2(0u, 0u);
        if (bb[j] >= 0 && ih >= 0 && ih < H && iw >= 0 && iw < W)
          raw[j] = __ldcg(reinterpret_cast<const uint2*>(md->dx + ((static_cast<int64_t>(bb[j]) * H + ih) * W + iw) * C + c));
      }
#pragma unroll
      for (int j = 0; j < kG; ++j) {
        const __nv_bfloat162 x01 = *reinterpret_cast<const __nv_bfloat162*>(&raw[j].x);
        const __nv_bfloat162 x23 = *reinterpret_cast<const __nv_bfloat162*>(&raw[j].y);
        acc[j][0] = fmaf(__low2float(x01), wv[0][k], acc[j][0]);
        acc[j][1] = fmaf(__high2float(x01), wv[1][k], acc[j][1]);
        acc[j][2] = fmaf(__low2float(x23), wv[2][k], acc[j][2]);
        acc[j][3] = fmaf(__high2float(x23), wv[3][k], acc[j][3]);
      }
    }
#pragma unroll
    for (int j = 0; j < kG; ++j) {
      if (bb[j] < 0) continue;
      uint2 o;
      o.x = pack_bf16(__float_as_uint(acc[j][0]), __float_as_uint(acc[j][1]), ck);
      o.y = pack_bf16(__float_as_uint(acc[j][2]), __float_as_uint(acc[j][3]), ck);
      *reinterpret_cast<uint2*>(md->dy + static_cast<int64_t>(m_base + pp * (i0 + j)) * C + c) = o;
    }
  }
}

// Pool tile (CUDA cores): max or average over an R x S window, kPoolTileM
// output pixels x kDwTileC channels.  Each lane owns 8 channels (16-byte
// loads); a warp pass covers 32 / (channel groups) pixels, spread over the 8
// epilogue warps first (a global pool's few pixels still use every warp).
// Two pixels per lane are processed together with up to 9 taps each
// unrolled, so 18 independent loads are in flight per lane: the op is
// load-latency bound.  Max pooling skips padded taps (torch MaxPool2d, via a
// -inf fill); average pooling divides by R*S (the global pools it serves have
// no padding).
constexpr int kPoolTileM = 128;
constexpr int kPoolTapChunk = 9;

__device__ __forceinline__ void pool_tile(const MemberDesc* __restrict__ md, const TileEntry& te, int ew, int lane) {
  const int M = md->m, C = md->ch, H = md->h_in, W = md->w_in;
  const int cbase = te.n_tile * kDwTileC;
  const int g = min(kDwTileC, C - cbase) >> 3;  // 8-channel groups in this tile
  const int gp = g <= 4 ? 4 : (g <= 8 ? 8 : 16);
  const int pp = 32 / gp;  // pixels per warp pass
  const int cg = lane & (gp - 1), sub = lane / gp;
  if (cg >= g) return;
  const int c = cbase + cg * 8;
  const int taps = md->r_taps, S = md->s_taps, st = md->stride, pad = md->pad, PQ = md->pq, Q = md->q;
  const bool mx = md->a_mode == kMaxPool;
  const uint32_t fill = mx ? 0xFF80FF80u : 0u;  // bf16x2 -inf (max) or 0 (sum)
  const float scale = mx ? 1.f : 1.f / static_cast<float>(taps);
  const int passes = kPoolTileM / (8 * pp);
  for (int ps = 0; ps < passes; ps += 2) {
    int mm[2], bb[2], hh[2], ww[2];
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      mm[j] = te.m_tile * kPoolTileM + ((ps + j) * 8 + ew) * pp + sub;
      const bool ok = ps + j < passes && mm[j] < M;
      bb[j] = ok ? mm[j] / PQ : -1;
      const int rem = mm[j] - bb[j] * PQ;
      const int p = rem / Q;
      hh[j] = p * st - pad;
      ww[j] = (rem - p * Q) * st - pad;
    }
    if (bb[0] < 0 && bb[1] < 0) break;
    float acc[2][8];
#pragma unroll
    for (int j = 0; j < 2; ++j)
#pragma unroll
      for (int e = 0; e < 8; ++e) acc[j][e] = mx ? -INFINITY : 0.f;
    for (int t0 = 0; t0 < taps; t0 += kPoolTapChunk) {
      uint4 raw[2][kPoolTapChunk];
#pragma unroll
      for (int k = 0; k < kPoolTapChunk; ++k) {
        const int tap = t0 + k;
        const int r = tap / S, s = tap - (tap / S) * S;
#pragma unroll
        for (int j = 0; j < 2; ++j) {
          const int ih = hh[j] + r, iw = ww[j] + s;
          raw[j][k] = make_uint4(fill, fill, fill, fill);
          if (tap < taps && bb[j] >= 0 && ih >= 0 && ih < H && iw >= 0 && iw < W)
            raw[j][k] = __ldcg(reinterpret_cast<const uint4*>(md->dx + ((static_cast<int64_t>(bb[j]) * H + ih) * W + iw) * C + c));
        }
      }
#pragma unroll
      for (int k = 0; k < kPoolTapChunk; ++k)
#pragma unroll
        for (int j = 0; j < 2; ++j) {
          const uint32_t w4[4] = {raw[j][k].x, raw[j][k].y, raw[j][k].z, raw[j][k].w};
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const __nv_bfloat162 v = *reinterpret_cast<const __nv_bfloat162*>(&w4[e]);
            if (mx) {
              acc[j][2 * e] = fmaxf(acc[j][2 * e], __low2float(v));
              acc[j][2 * e + 1] = fmaxf(acc[j][2 * e + 1], __high2float(v));
            } else {
              acc[j][2 * e] += __low2float(v);
              acc[j][2 * e + 1] += __high2float(v);
            }
          }
        }
    }
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      if (bb[j] < 0) continue;
      uint4 o;
      const Clamp ck = clamp_of(md->act);
      o.x = pack_bf16(__float_as_uint(acc[j][0] * scale), __float_as_uint(acc[j][1] * scale), ck);
      o.y = pack_bf16(__float_as_uint(acc[j][2] * scale), __float_as_uint(acc[j][3] * scale), ck);
      o.z = pack_bf16(__float_as_uint(acc[j][4] * scale), __float_as_uint(acc[j][5] * scale), ck);
      o.w = pack_bf16(__float_as_uint(acc[j][6] * scale), __float_as_uint(acc[j][7] * scale), ck);
      *reinterpret_cast<uint4*>(md->dy + static_cast<int64_t>(mm[j]) * C + c) = o;
    }
  }
}

// Staged CUDA-core tiles.  The tile is output rows [p0, p0 + cc_rows) x all
// q columns of one image, channels [c0, c0 + n_tile); its input window sits in
// shared memory as [Hb][Wb][n_tile] bf16 (the TMA box, zero outside the
// image).  128 threads (one epilogue warpgroup): each owns one 8-channel group
// (16 B) of a pixel and keeps it across pixels (n_tile / 8 <= 32 groups per
// pixel; 128 mod groups threads idle).  Max pooling skips taps outside the image (torch
// MaxPool2d); average pooling and depthwise convs sum the zero fill (the
// reference divides by R*S).  fp32 accumulation, fused activation, bf16 out.
struct StagedGeom {
  int cc, Q, st, S, R, Wb, m0, h0, w0, c;
  int cg, px0, pstep;  // this thread's channel group, first pixel, pixel step (px0 >= pstep: idle)
};

__device__ __forceinline__ StagedGeom staged_geom(const MemberDesc* __restrict__ md, const TileEntry& te, int gt) {
  StagedGeom g;
  g.cc = md->n_tile;
  const int L = g.cc >> 3;  // 8-channel groups per pixel (<= 32)
  g.cg = gt % L;
  g.px0 = gt / L;
  g.pstep = 128 / L;
  g.Q = md->q;
  g.st = md->stride;
  g.S = md->s_taps;
  g.R = md->r_taps / g.S;
  g.Wb = (g.Q - 1) * g.st + g.S;
  g.m0 = te.m_tile * md->cc_rows * g.Q;
  const int img = g.m0 / md->pq;
  g.h0 = (g.m0 - img * md->pq) / g.Q * g.st - md->pad;
  g.w0 = -md->pad;
  g.c = te.n_tile * g.cc + g.cg * 8;
  return g;
}

__device__ __forceinline__ void bf16x8_to_f32(const uint4 v, float (&f)[8]) {
  const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    f[2 * e] = __uint_as_float(w[e] << 16);
    f[2 * e + 1] = __uint_as_float(w[e] & 0xFFFF0000u);
  }
}

__device__ __forceinline__ void store_bf16x8(__nv_bfloat16* dst, const float (&a)[8], float scale, Clamp ck) {
  uint4 o;
  o.x = pack_bf16(__float_as_uint(a[0] * scale), __float_as_uint(a[1] * scale), ck);
  o.y = pack_bf16(__float_as_uint(a[2] * scale), __float_as_uint(a[3] * scale), ck);
  o.z = pack_bf16(__float_as_uint(a[4] * scale), __float_as_uint(a[5] * scale), ck);
  o.w = pack_bf16(__float_as_uint(a[6] * scale), __float_as_uint(a[7] * scale), ck);
  *reinterpret_cast<uint4*>(dst) = o;
}

__device__ __forceinline__ void staged_pool_tile(const MemberDesc* __restrict__ md, const TileEntry& te,
                                                 const uint8_t* src, int gt, int bar_id) {
  const StagedGeom g = staged_geom(md, te, gt);
  const int H = md->h_in, W = md->w_in, C = md->ch;
  const int npix = md->cc_rows * g.Q;
  const Clamp ck = clamp_of(md->act);
  const int row_bytes = g.Wb * g.cc * 2, px_bytes = g.cc * 2;
  const uint8_t* base0 = src + g.cg * 16;
  const int px_first = g.px0 < g.pstep ? g.px0 : npix;
  if (md->a_mode == kMaxPool) {
    // max is exact in bf16: packed bf16x2 max over the taps inside the image
    // (taps in the padding are skipped, as torch MaxPool2d does)
    const __nv_bfloat162 ninf = __float2bfloat162_rn(-INFINITY);
    for (int px = px_first; px < npix; px += g.pstep) {
      const int pr = px / g.Q, qc = px - pr * g.Q;
      const int ih0 = g.h0 + pr * g.st, iw0 = g.w0 + qc * g.st;
      const uint8_t* base = base0 + pr * g.st * row_bytes + qc * g.st * px_bytes;
      __nv_bfloat162 m[4] = {ninf, ninf, ninf, ninf};
      for (int r = 0; r < g.R; ++r) {
        if (ih0 + r < 0 || ih0 + r >= H) continue;
        const uint8_t* rowp = base + r * row_bytes;
#pragma unroll 3
        for (int s = 0; s < g.S; ++s) {
          const uint4 v = *reinterpret_cast<const uint4*>(rowp + s * px_bytes);
          const bool ok = iw0 + s >= 0 && iw0 + s < W;
          const uint32_t w4[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
          for (int e = 0; e < 4; ++e)
            m[e] = ok ? __hmax2(m[e], *reinterpret_cast<const __nv_bfloat162*>(&w4[e])) : m[e];
        }
      }
      float acc[8];
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        acc[2 * e] = __low2float(m[e]);
        acc[2 * e + 1] = __high2float(m[e]);
      }
      store_bf16x8(md->dy + static_cast<int64_t>(g.m0 + px) * C + g.c, acc, 1.f, ck);
    }
    return;
  }
  // average: fp32 sum of every tap (the zero fill counts), / R*S
  const float scale = 1.f / static_cast<float>(md->r_taps);
  if (npix <= g.pstep / 2) {
    // few pixels (global pools: one per image): the idle pixel slots of the
    // group split each pixel's rows of taps, then one slot adds the partial
    // sums through the (consumed) input slot
    // partial-sum parts per pixel: the group's spare pixel slots, at most one
    // per filter row, and the other parts' sums must fit the input slot
    const int per_part = npix * (g.cc >> 3) * 32;  // bytes of one part's partial sums
    const int reps = min(min(g.pstep / npix, g.R), 1 + static_cast<int>(md->tx_bytes) / per_part);
    const int px = g.px0 % npix, part = g.px0 / npix;
    const bool active = g.px0 < g.pstep && part < reps;
    float acc[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) acc[e] = 0.f;
    if (active) {
      const int pr = px / g.Q, qc = px - pr * g.Q;
      const uint8_t* base = base0 + pr * g.st * row_bytes + qc * g.st * px_bytes;
      for (int r = part; r < g.R; r += reps) {
        const uint8_t* rowp = base + r * row_bytes;
#pragma unroll 4
        for (int s = 0; s < g.S; ++s) {
          float f[8];
          bf16x8_to_f32(*reinterpret_cast<const uint4*>(rowp + s * px_bytes), f);
#pragma unroll
          for (int e = 0; e < 8; ++e) acc[e] += f[e];
        }
      }
    }
    // every thread of the group has read its taps: reuse the slot's first bytes
    named_barrier(bar_id, 128);
    float* scratch = reinterpret_cast<float*>(const_cast<uint8_t*>(src));
    if (active && part > 0)
#pragma unroll
      for (int e = 0; e < 8; ++e) scratch[((part - 1) * npix * (g.cc >> 3) + px * (g.cc >> 3) + g.cg) * 8 + e] = acc[e];
    named_barrier(bar_id, 128);
    if (active && part == 0) {
      for (int p2 = 1; p2 < reps; ++p2)
#pragma unroll
        for (int e = 0; e < 8; ++e) acc[e] += scratch[((p2 - 1) * npix * (g.cc >> 3) + px * (g.cc >> 3) + g.cg) * 8 + e];
      store_bf16x8(md->dy + static_cast<int64_t>(g.m0 + px) * C + g.c, acc, scale, ck);
    }
    return;
  }
  for (int px = px_first; px < npix; px += g.pstep) {
    const int pr = px / g.Q, qc = px - pr * g.Q;
    const uint8_t* base = base0 + pr * g.st * row_bytes + qc * g.st * px_bytes;
    float acc[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) acc[e] = 0.f;
    for (int r = 0; r < g.R; ++r) {
      const uint8_t* rowp = base + r * row_bytes;
#pragma unroll 4
      for (int s = 0; s < g.S; ++s) {
        float f[8];
        bf16x8_to_f32(*reinterpret_cast<const uint4*>(rowp + s * px_bytes), f);
#pragma unroll
        for (int e = 0; e < 8; ++e) acc[e] += f[e];
      }
    }
    store_bf16x8(md->dy + static_cast<int64_t>(g.m0 + px) * C + g.c, acc, scale, ck);
  }
}

__device__ __forceinline__ void staged_dw_tile(const MemberDesc* __restrict__ md, const TileEntry& te,
                                               const uint8_t* src, int gt) {
  const StagedGeom g = staged_geom(md, te, gt);
  const int C = md->ch;
  const int npix = md->cc_rows * g.Q;
  const Clamp ck = clamp_of(md->act);
  const int row_bytes = g.Wb * g.cc * 2;
  const uint8_t* base0 = src + g.cg * 16;
  const __nv_bfloat16* wp = md->dw + static_cast<int64_t>(g.c) * md->ldw;
  if (g.R == 3 && g.S == 3) {
    // 3x3 (every depthwise layer of MobileNet-v2): this thread's 8 channels x
    // 9 taps in registers (one 16-byte load per tap), taps unrolled
    float wv[9][8];
#pragma unroll
    for (int k = 0; k < 9; ++k)
      bf16x8_to_f32(__ldg(reinterpret_cast<const uint4*>(md->dwt + static_cast<int64_t>(k) * C + g.c)), wv[k]);
    for (int px = g.px0 < g.pstep ? g.px0 : npix; px < npix; px += g.pstep) {
      const int pr = px / g.Q, qc = px - pr * g.Q;
      const uint8_t* base = base0 + pr * g.st * row_bytes + qc * g.st * g.cc * 2;
      float acc[8];
#pragma unroll
      for (int e = 0; e < 8; ++e) acc[e] = 0.f;
#pragma unroll
      for (int r = 0; r < 3; ++r)
#pragma unroll
        for (int s = 0; s < 3; ++s) {
          float f[8];
          bf16x8_to_f32(*reinterpret_cast<const uint4*>(base + r * row_bytes + s * g.cc * 2), f);
#pragma unroll
          for (int e = 0; e < 8; ++e) acc[e] = fmaf(f[e], wv[r * 3 + s][e], acc[e]);
        }
      store_bf16x8(md->dy + static_cast<int64_t>(g.m0 + px) * C + g.c, acc, 1.f, ck);
    }
    return;
  }
  // other filter shapes: weights re-read per tap (L1)
  for (int px = g.px0 < g.pstep ? g.px0 : npix; px < npix; px += g.pstep) {
    const int pr = px / g.Q, qc = px - pr * g.Q;
    const uint8_t* base = base0 + pr * g.st * row_bytes + qc * g.st * g.cc * 2;
    float acc[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) acc[e] = 0.f;
    for (int r = 0; r < g.R; ++r)
      for (int s = 0; s < g.S; ++s) {
        float f[8];
        bf16x8_to_f32(*reinterpret_cast<const uint4*>(base + r * row_bytes + s * g.cc * 2), f);
        const int k = r * g.S + s;
#pragma unroll
        for (int e = 0; e < 8; ++e) acc[e] = fmaf(f[e], __bfloat162float(wp[e * md->ldw + k]), acc[e]);
      }
    store_bf16x8(md->dy + static_cast<int64_t>(g.m0 + px) * C + g.c, acc, 1.f, ck);
  }
}

// ---------------------------------------------------------------- kernel

template <int BN>
__global__ void __launch_bounds__(kThreads, 1)
    superkernel(const MemberDesc* __restrict__ slots, const TileEntry* __restrict__ tiles, int n_tiles,
                const RoundArgs ra) {
  using C = Cfg<BN>;
  uint32_t* __restrict__ counters = ra.counters;
  const uint32_t* __restrict__ targets = ra.targets;
  uint64_t* __restrict__ trace = ra.trace;
  constexpr uint32_t kStages = C::kStages;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* ring = smem;                                // kStages x (A | B)
  uint8_t* epi = smem + kStages * C::kStageBytes;     // store staging
  uint64_t* full = reinterpret_cast<uint64_t*>(epi + kEpiBytes);
  uint64_t* empty = full + C::kMaxSlots;
  uint64_t* acc_full = empty + C::kMaxSlots;
  uint64_t* acc_empty = acc_full + 2;
  uint64_t* tq_full = acc_empty + 2;     // claimed-tile ring: producer -> consumers
  uint64_t* tq_empty = tq_full + kTileQ;
  uint64_t* sq_full = tq_empty + kTileQ;  // scheduler -> producer (claim look-ahead)
  uint64_t* sq_empty = sq_full + kSchedQ;
  uint64_t* pub_full = sq_empty + kSchedQ;  // [2][kPubQ]: epilogue warpgroup -> publisher warp
  uint64_t* pub_empty = pub_full + 2 * kPubQ;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(pub_empty + 2 * kPubQ);
  volatile int32_t* tq = reinterpret_cast<volatile int32_t*>(tmem_slot + 1);
  volatile int32_t* sq = tq + kTileQ;
  volatile uint32_t* tq_aux = reinterpret_cast<volatile uint32_t*>(sq + kSchedQ);  // staged tiles: ring slot
  volatile int32_t* pub_q = reinterpret_cast<volatile int32_t*>(tq_aux + kTileQ);    // [2][kPubQ] counter indices
  TileRec* srec = reinterpret_cast<TileRec*>((reinterpret_cast<uintptr_t>(pub_q + 2 * kPubQ) + 15) & ~uintptr_t(15));

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  // trace (debug): per CTA after the tile stamps, SM clock64 cycles: entry,
  // setup done, producer loop done, all roles done (warp 2 past the final
  // barrier), TMEM released, exit
  uint64_t* cta_trace = trace ? trace + 6 * n_tiles + 6 * blockIdx.x : nullptr;
  if (cta_trace && threadIdx.x == 0) cta_trace[0] = clock64();
  // Static schedule: this CTA's first tile is blockIdx.x.  While thread 0 and
  // warp 2 set up barriers and TMEM, the idle scheduler lane pulls that
  // tile's entry, member descriptor and tensor maps toward the SM, so the
  // producer's and MMA warp's first reads hit L1 instead of L2.
  if (warp == 3 && lane == 0 && !ra.heads && !ra.next_tile && static_cast<int>(blockIdx.x) < n_tiles) {
    const MemberDesc* md0 = slots + tiles[blockIdx.x].member;
    const char* p0 = reinterpret_cast<const char*>(md0);
#pragma unroll
    for (int i = 0; i < static_cast<int>(sizeof(MemberDesc)); i += 128)
      asm volatile("prefetch.global.L1 [%0];" ::"l"(p0 + i));
    prefetch_tmap(&md0->a);
    prefetch_tmap(&md0->b);
  }

  if (threadIdx.x == 0) {
    for (int s = 0; s < C::kMaxSlots; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&acc_full[a], 1);
      mbar_init(&acc_empty[a], 128);
    }
    for (int q = 0; q < kTileQ; ++q) {
      mbar_init(&tq_full[q], 1);
      mbar_init(&tq_empty[q], 1 + 8);  // the MMA thread + one lane per epilogue warp
    }
    for (int q = 0; q < kSchedQ; ++q) {
      mbar_init(&sq_full[q], 1);
      mbar_init(&sq_empty[q], 1);
    }
    for (int q = 0; q < 2 * kPubQ; ++q) {
      mbar_init(&pub_full[q], 1);
      mbar_init(&pub_empty[q], 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(C::kTmemCols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  if (cta_trace && threadIdx.x == 0) cta_trace[1] = clock64();
  // Let the next launch in the stream (programmatic dependent launch) start
  // its prologue on SMs this grid frees; it waits in griddepcontrol.wait.
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");

  if (warp == 0) {
    if (lane == 0) {
      // ------------------------------------------------ TMA producer
      // ring: current layout, next slot, per-slot use parity, last issued
      uint32_t stage = 0, ubits = 0, nslots = kStages, sbytes = C::kStageBytes;
      int layout = 0;
      auto advance = [&]() {
        ubits ^= 1u << stage;
        stage = stage + 1 == nslots ? 0 : stage + 1;
      };
      auto wait_free = [&]() { mbar_wait(&empty[stage], ((ubits >> stage) & 1u) ^ 1u); };
      auto set_layout = [&](int lay) {
        if (lay == layout) return;
        // drain every slot (staged CUDA-core slots are freed by the
        // epilogue, possibly before earlier MMA slots)
        for (uint32_t s = 0; s < nslots; ++s) mbar_wait(&empty[s], ((ubits >> s) & 1u) ^ 1u);
        layout = lay;
        nslots = layout ? C::kNarrowSlots : kStages;
        sbytes = layout ? C::kNarrowBytes : C::kStageBytes;
        stage = 0;
      };
      bool first = true;
      uint32_t qslot = 0, qphase = 0, sslot = 0, sphase = 0;
      // Greedy schedule: the producer claims its own tiles in table order
      // from one global counter, the next one as it starts a tile's loads (a
      // one-tile look-ahead instead of the static round-robin assignment).
      const bool greedy = ra.next_tile != nullptr;
      int next = 0;
      if (greedy) {
        // the claim counter is reset by the previous launch's last CTA
        asm volatile("griddepcontrol.wait;" ::: "memory");
        next = static_cast<int>(atomicAdd(ra.next_tile, 1u));
      }
      for (;;) {
        int t;
        TileRec rec;
        if (greedy) {
          t = next < n_tiles ? next : -1;
          if (t >= 0) load_tile_rec(tiles, slots, t, rec);
        } else {
          mbar_wait(&sq_full[sslot], sphase);  // next tile from the scheduler warp
          t = sq[sslot];
          if (t >= 0) rec = srec[sslot];  // copied before the slot is released
          mbar_arrive(&sq_empty[sslot]);
          if (++sslot == kSchedQ) {
            sslot = 0;
            sphase ^= 1;
          }
        }
        TileEntry te{};
        const MemberDesc* md = slots;  // tensor-map addresses only; scalars come from the record
        MemberScalars ms{};
        bool dw = false;
        if (t >= 0) {
          te = rec.te;
          md = slots + te.member;
          ms = rec.ms;
          dw = cuda_core_mode(ms.a_mode);
        }
        const bool staged = dw && rec.cc_rows > 0;
        if (staged) {
          // Name the slot to the consumers only once its previous use is
          // released: the epilogue's parity wait on it is then unambiguous
          // (one phase ahead at most), however far ahead of the ring it runs.
          set_layout(ms.ring_narrow);
          wait_free();
        }
        mbar_wait(&tq_empty[qslot], qphase ^ 1);
        // consumers skip / route a CUDA-core tile without loading it; a staged
        // one takes the next ring slot: slot | use parity << 4 | byte offset / 1 KB << 8
        tq[qslot] = dw ? (t | kDwTag | (staged ? kStagedTag : 0)) : t;
        if (staged) tq_aux[qslot] = stage | (((ubits >> stage) & 1u) << 4) | ((stage * sbytes) >> 10 << 8);
        mbar_arrive(&tq_full[qslot]);
        const uint32_t wslot = qslot, wphase = qphase;
        if (++qslot == kTileQ) {
          qslot = 0;
          qphase ^= 1;
        }
        if (t < 0) break;
        if (dw) {  // computed by the epilogue warps
          if (staged) {
            // gate like an activation load, then the whole input window as
            // one box into the next slot of the current ring layout
            const int img = rec.img, h0 = rec.h0;  // the window's image and first row (scheduler)
            if (trace) trace[6 * t + 0] = globaltimer();
            if (first) {
              asm volatile("griddepcontrol.wait;" ::: "memory");
              first = false;
            }
            if (te.dep >= 0 || te.rdep >= 0) {
              if (te.dep >= 0) wait_range(counters, targets, te.dep, te.dep_n, 32);
              if (te.rdep >= 0) wait_range(counters, targets, te.rdep, te.rdep_n, 32);
              asm volatile("fence.proxy.async.global;" ::: "memory");
            }
            if (trace) trace[6 * t + 1] = globaltimer();
            mbar_expect_tx(&full[stage], ms.tx_bytes);
            tma_load_4d(ring + stage * sbytes, &md->a, &full[stage], te.n_tile * ms.n_tile, -ms.pad, h0, img);
            advance();
          }
          if (greedy) {
            // claim the next tile only once every epilogue warp has taken this
            // one, so a CTA never hoards depthwise tiles other SMs could run
            mbar_wait(&tq_empty[wslot], wphase);
            next = static_cast<int>(atomicAdd(ra.next_tile, 1u));
          }
          continue;
        }
        if (greedy) {  // otherwise the scheduler lane prefetched them with the claim
          prefetch_tmap(&md->a);
          prefetch_tmap(&md->b);
        }
        set_layout(ms.ring_narrow);
        const int kb_lo = te.kb_end ? te.kb_begin : 0;
        const int k_blocks = te.kb_end ? te.kb_end : ms.k_blocks;
        const uint32_t tx = ms.tx_bytes;
        const int tall = ms.tall;
        const int m0 = te.m_tile * (kBM << tall);
        const int n0 = te.n_tile * ms.n_tile;
        const uint32_t b_off = static_cast<uint32_t>(kABytes << tall);
        const bool narrow = ms.a_mode == kAIm2colNarrow;
        const bool fold = ms.a_mode == kAIm2colFold;
        const bool im2col = ms.a_mode != kATiled;
        // im2col start coordinates (tall: both halves) and the K walk's first
        // position come precomputed with the tile record; they advance
        // incrementally (load_a runs in k-block order within a tile): no
        // integer divisions on the producer's path
        const int img = rec.img, h0 = rec.h0, w0 = rec.w0;
        const int img1 = rec.img1, h1 = rec.h1, w1 = rec.w1;
        const int c_blocks = im2col ? ms.c_blocks : 1, s_taps = im2col ? ms.s_taps : 1;
        int cb = rec.cb, s_ = rec.s_, r_ = rec.r_;
        const int taps = ms.taps, images = ms.images;
        const CUtensorMap* amap = &md->a;

        auto load_a = [&](int kb, uint32_t st) {
          uint8_t* a_dst = ring + st * sbytes;
          if (fold) {
            // two filter rows; a row past R re-reads row 0 (its weights are zero)
#pragma unroll
            for (int j = 0; j < kFoldTaps; ++j) {
              const int r = kb * kFoldTaps + j;
              tma_load_im2col(a_dst + j * kFoldTapBytes, amap, &full[st], 0, w0, h0, img, 0,
                              static_cast<uint16_t>(r < taps ? r : 0));
              if (tall)
                tma_load_im2col(a_dst + kABytes + j * kFoldTapBytes, amap, &full[st], 0, w1, h1, img1, 0,
                                static_cast<uint16_t>(r < taps ? r : 0));
            }
          } else if (narrow) {
            // eight 16 B tap columns; taps past R*S load an out-of-range image
            // so TMA zero-fills them (the weights there are zero too)
#pragma unroll 1
            for (int j = 0; j < kNarrowTaps; ++j) {
              const int tap = kb * kNarrowTaps + j;
              const bool real = tap < taps;
              const int r = real ? tap / s_taps : 0;
              const int s = real ? tap - r * s_taps : 0;
              tma_load_im2col(a_dst + j * kNarrowTapBytes, amap, &full[st], 0, w0, h0, real ? img : images,
                              static_cast<uint16_t>(s), static_cast<uint16_t>(r));
            }
          } else if (im2col) {
            // (tall: the map's box is 256 pixels, both halves in one load)
            tma_load_im2col(a_dst, amap, &full[st], cb * kBK, w0, h0, img, static_cast<uint16_t>(s_),
                            static_cast<uint16_t>(r_));
            if (++cb == c_blocks) {
              cb = 0;
              if (++s_ == s_taps) {
                s_ = 0;
                ++r_;
              }
            }
          } else {
            tma_load_2d(a_dst, amap, &full[st], kb * kBK, m0);  // tall: one 256-row box
          }
        };
        auto load_b = [&](int kb, uint32_t st) {
          tma_load_2d(ring + st * sbytes + b_off, &md->b, &full[st], kb * kBK, n0);
        };
        // Activation gate: the prerequisite grid (PDL) before the first tile,
        // and in a round program the tenant's previous layer (all its tiles
        // stored).  Weights never wait on either.
        auto gate = [&]() {
          if (first) asm volatile("griddepcontrol.wait;" ::: "memory");
          if (te.dep >= 0 || te.rdep >= 0) {
            if (te.dep >= 0) wait_range(counters, targets, te.dep, te.dep_n, 32);
            if (te.rdep >= 0) wait_range(counters, targets, te.rdep, te.rdep_n, 32);
            asm volatile("fence.proxy.async.global;" ::: "memory");
          }
        };
        if (trace) trace[6 * t + 0] = globaltimer();
        int kb = kb_lo;
        if (first) {
          // All slots are free (stage 0, fresh barriers): stream the first
          // stages' B tiles, then gate.
          const int pre = min(k_blocks - kb_lo, static_cast<int>(nslots));
          for (int j = 0; j < pre; ++j) {
            mbar_expect_tx(&full[j], tx);
            load_b(kb_lo + j, j);
          }
          gate();
          if (trace) trace[6 * t + 1] = globaltimer();
          first = false;
          for (int j = 0; j < pre; ++j) {
            load_a(kb_lo + j, j);
            advance();
          }
          kb = kb_lo + pre;
        } else if (te.dep >= 0 || te.rdep >= 0) {
          // weights do not wait on the dependency: stream B into the next
          // stages (up to the ring depth, as slots free up), then gate, then
          // the activations into the same stages
          const int pre = min(k_blocks - kb_lo, static_cast<int>(nslots) - 1);
          uint32_t st = stage;
          for (int j = 0; j < pre; ++j) {
            mbar_wait(&empty[st], ((ubits >> st) & 1u) ^ 1u);
            mbar_expect_tx(&full[st], tx);
            load_b(kb_lo + j, st);
            st = st + 1 == nslots ? 0 : st + 1;
          }
          gate();
          if (trace) trace[6 * t + 1] = globaltimer();
          for (int j = 0; j < pre; ++j) {
            load_a(kb_lo + j, stage);
            advance();
          }
          kb = kb_lo + pre;
        } else if (trace) {
          trace[6 * t + 1] = globaltimer();  // no gate
        }
        if (greedy) next = static_cast<int>(atomicAdd(ra.next_tile, 1u));  // latency hides under the loads
        // Steady state, specialised per A mode and tile height so the
        // per-k-block issue path (a single thread: it bounds narrow tiles)
        // carries no mode tests.
        auto steady = [&](auto mode_c, auto tall_c) {
          constexpr int kMode = decltype(mode_c)::value;
          constexpr int kTall = decltype(tall_c)::value;
          for (; kb < k_blocks; ++kb) {
            wait_free();
            uint64_t* bar = &full[stage];
            mbar_expect_tx(bar, tx);
            uint8_t* a_dst = ring + stage * sbytes;
            if constexpr (kMode == kATiled) {
              tma_load_2d(a_dst, amap, bar, kb * kBK, m0);  // tall: one 256-row box
            } else if constexpr (kMode == kAIm2colFold) {
              // two filter rows; a row past R re-reads row 0 (its weights are zero)
#pragma unroll
              for (int j = 0; j < kFoldTaps; ++j) {
                const int r = kb * kFoldTaps + j;
                const uint16_t rr = static_cast<uint16_t>(r < taps ? r : 0);
                tma_load_im2col(a_dst + j * kFoldTapBytes, amap, bar, 0, w0, h0, img, 0, rr);
                if constexpr (kTall) tma_load_im2col(a_dst + kABytes + j * kFoldTapBytes, amap, bar, 0, w1, h1, img1, 0, rr);
              }
            } else {
              tma_load_im2col(a_dst, amap, bar, cb * kBK, w0, h0, img, static_cast<uint16_t>(s_),
                              static_cast<uint16_t>(r_));  // tall: one 256-pixel box
              if (++cb == c_blocks) {
                cb = 0;
                if (++s_ == s_taps) {
                  s_ = 0;
                  ++r_;
                }
              }
            }
            tma_load_2d(a_dst + kABytes * (1 + kTall), &md->b, bar, kb * kBK, n0);
            advance();
          }
        };
        using I0 = std::integral_constant<int, 0>;
        using I1 = std::integral_constant<int, 1>;
        if (ms.a_mode == kATiled) {
          if (tall)
            steady(std::integral_constant<int, kATiled>{}, I1{});
          else
            steady(std::integral_constant<int, kATiled>{}, I0{});
        } else if (ms.a_mode == kAIm2col) {
          if (tall)
            steady(std::integral_constant<int, kAIm2col>{}, I1{});
          else
            steady(std::integral_constant<int, kAIm2col>{}, I0{});
        } else if (ms.a_mode == kAIm2colFold) {
          if (tall)
            steady(std::integral_constant<int, kAIm2colFold>{}, I1{});
          else
            steady(std::integral_constant<int, kAIm2colFold>{}, I0{});
        } else {
          for (; kb < k_blocks; ++kb) {
            wait_free();
            mbar_expect_tx(&full[stage], tx);
            load_a(kb, stage);
            load_b(kb, stage);
            advance();
          }
        }
        if (rec.has_res && k_blocks == ms.k_blocks) {
          // residual k-blocks (the tile, or the split holding the K tail):
          // A = residual columns [n0 + 64 j, +64) of the tile's rows, B = the
          // matching 64 columns of the identity
          const int rk = (min(ms.n_tile, ms.n - n0) + kBK - 1) / kBK;
          for (int j = 0; j < rk; ++j) {
            wait_free();
            uint64_t* bar = &full[stage];
            mbar_expect_tx(bar, tx);
            uint8_t* a_dst = ring + stage * sbytes;
            tma_load_2d(a_dst, &md->r, bar, n0 + j * kBK, m0);  // tall: one 256-row box
            tma_load_2d(a_dst + b_off, &md->id, bar, j * kBK, 0);
            advance();
          }
        }
      }
      if (first) asm volatile("griddepcontrol.wait;" ::: "memory");
    }
  } else if (warp == 1) {
    // ------------------------------------------------ MMA issuer
    // The whole warp runs the loop on warp-uniform values (tile fields are
    // broadcast from lane 0 with shfl), so the descriptor arithmetic lives in
    // uniform registers; one elected lane issues tcgen05.mma / commit.
    uint32_t stage = 0, fbits = 0, nslots = kStages, sbytes = C::kStageBytes, acc = 0, acc_phase = 0;
    int layout = 0;
    uint32_t qslot = 0, qphase = 0;
    const uint32_t ring_base = smem_u32(ring);
    for (;;) {
      mbar_wait(&tq_full[qslot], qphase);
      const int t = __shfl_sync(0xffffffffu, tq[qslot], 0);
      __syncwarp();
      if (lane == 0) mbar_arrive(&tq_empty[qslot]);
      if (++qslot == kTileQ) {
        qslot = 0;
        qphase ^= 1;
      }
      if (t < 0) break;
      if (t & kDwTag) {  // CUDA-core tile: no accumulator, the epilogue warps compute it
        if (t & kStagedTag) {  // its input took one ring slot, which the epilogue frees
          const int lay = __shfl_sync(0xffffffffu, slots[tiles[t & ~(kDwTag | kStagedTag)].member].ring_narrow, 0);
          if (lay != layout) {  // the producer drained the ring before switching
            layout = lay;
            nslots = lay ? C::kNarrowSlots : kStages;
            sbytes = lay ? C::kNarrowBytes : C::kStageBytes;
            stage = 0;
          }
          // Wait for the box to land even though no MMA reads it: a parity
          // wait only tells phases apart one use ahead, so skipping the slot
          // unwaited would let this warp lap the ring and take a still-pending
          // staged phase for its next GEMM use of the slot.
          mbar_wait(&full[stage], (fbits >> stage) & 1u);
          fbits ^= 1u << stage;
          stage = stage + 1 == nslots ? 0 : stage + 1;
        }
        continue;
      }
      const TileEntry te = tiles[t];
      const MemberDesc* md = slots + te.member;
      const int kb_lo = __shfl_sync(0xffffffffu, te.kb_end ? te.kb_begin : 0, 0);
      const int k_tail = te.kb_end ? te.kb_end : md->k_blocks;
      // residual k-blocks ride on the tile (or split) holding the K tail
      const int k_res = md->res && k_tail == md->k_blocks
                            ? (min(md->n_tile, md->n - te.n_tile * md->n_tile) + kBK - 1) / kBK
                            : 0;
      const int k_blocks = __shfl_sync(0xffffffffu, k_tail + k_res, 0);
      const uint32_t idesc = __shfl_sync(0xffffffffu, md->idesc, 0);
      const int lay = __shfl_sync(0xffffffffu, md->ring_narrow, 0);
      if (lay != layout) {  // the producer drained the ring before switching
        layout = lay;
        nslots = lay ? C::kNarrowSlots : kStages;
        sbytes = lay ? C::kNarrowBytes : C::kStageBytes;
        stage = 0;
      }
      const int a_mode = __shfl_sync(0xffffffffu, md->a_mode, 0);
      const int tall = __shfl_sync(0xffffffffu, md->tall, 0);
      const uint32_t d_half = static_cast<uint32_t>(__shfl_sync(0xffffffffu, md->n_tile, 0));  // tall: 2nd half's columns
      // Smem descriptors (SM100): lo = start >> 4 | LBO >> 4 << 16, hi = SBO
      // >> 4 | version 1 << 14 | swizzle << 29, built once per tile.  Per
      // UMMA_K step (16 bf16) the A start advances 32 B inside the 128 B
      // swizzle atom, or two narrow tap columns, or 32 B inside a folded
      // 64 B row (then the next column): k1..k3 in 16-byte units.
      uint32_t a_hi = (1024u >> 4) | (1u << 14) | (2u << 29), a_lbo = 1u << 16;
      uint32_t k1 = 2, k2 = 4, k3 = 6;
      if (a_mode == kAIm2colFold) {
        a_hi = (512u >> 4) | (1u << 14) | (4u << 29);
        k2 = kFoldTapBytes >> 4;
        k3 = k2 + 2;
      } else if (a_mode == kAIm2colNarrow) {
        a_hi = (128u >> 4) | (1u << 14);
        a_lbo = static_cast<uint32_t>(kNarrowTapBytes >> 4) << 16;
        k1 = (2 * kNarrowTapBytes) >> 4;
        k2 = 2 * k1;
        k3 = 3 * k1;
      }
      const uint64_t a_hi64 = static_cast<uint64_t>(a_hi) << 32;
      constexpr uint64_t b_hi64 = static_cast<uint64_t>((1024u >> 4) | (1u << 14) | (2u << 29)) << 32;
      mbar_wait(&acc_empty[acc], acc_phase ^ 1);
      tc_fence_after();
      const uint32_t d_tmem = tmem_base + acc * BN;
      // One k-block: wait for its stage, issue `halves` x 4 UMMA_K steps, free
      // the stage.  Two loop instances so the common path carries no test.
      auto kloop = [&](auto halves_c) {
        constexpr int kHalves = decltype(halves_c)::value;
        for (int kb = kb_lo; kb < k_blocks; ++kb) {
          mbar_wait(&full[stage], (fbits >> stage) & 1u);
          tc_fence_after();
          if (trace && kb == kb_lo && lane == 0) trace[6 * t + 2] = globaltimer();
          const uint32_t a_addr = ring_base + stage * sbytes;
          const uint32_t a_lo = ((a_addr >> 4) & 0x3FFFu) | a_lbo;
          const uint32_t b_lo = (((a_addr + (kABytes * kHalves)) >> 4) & 0x3FFFu) | (1u << 16);
          if (elect_one()) {
#pragma unroll
            for (int h = 0; h < kHalves; ++h) {
              // half h: A box at +16 KB * h, accumulator columns + n_tile * h
              const uint32_t ah = a_lo + h * (kABytes >> 4);
              const uint32_t dh = d_tmem + h * d_half;
              umma_bf16(dh, a_hi64 | ah, b_hi64 | b_lo, idesc, kb != kb_lo ? 1u : 0u);
              umma_bf16(dh, a_hi64 | (ah + k1), b_hi64 | (b_lo + 2), idesc, 1u);
              umma_bf16(dh, a_hi64 | (ah + k2), b_hi64 | (b_lo + 4), idesc, 1u);
              umma_bf16(dh, a_hi64 | (ah + k3), b_hi64 | (b_lo + 6), idesc, 1u);
            }
            umma_commit(&empty[stage]);  // frees the smem stage once these MMAs retire
          }
          __syncwarp();
          fbits ^= 1u << stage;
          stage = stage + 1 == nslots ? 0 : stage + 1;
        }
      };
      if (tall)
        kloop(std::integral_constant<int, 2>{});
      else
        kloop(std::integral_constant<int, 1>{});
      if (elect_one()) umma_commit(&acc_full[acc]);  // accumulator ready for the epilogue
      __syncwarp();
      if (trace && lane == 0) trace[6 * t + 3] = globaltimer();
      acc ^= 1;
      if (acc == 0) acc_phase ^= 1;
    }
  } else if (warp == 2) {
    if (lane == 0) {
      // ------------------------------------------------ publisher
      // Releases the round counters of staged CUDA-core tiles, so the
      // computing warpgroup does not stall on the release fence (which waits
      // for its stores).  Serves both groups' queues in arrival order per group.
      uint32_t ps[2] = {0, 0}, ph[2] = {0, 0};
      bool live[2] = {true, true};
      while (live[0] || live[1]) {
        bool any = false;
#pragma unroll
        for (int g = 0; g < 2; ++g) {
          if (!live[g] || !mbar_test(&pub_full[g * kPubQ + ps[g]], ph[g])) continue;
          any = true;
          const int d = pub_q[g * kPubQ + ps[g]];
          if (d < 0)
            live[g] = false;
          else
            red_release_add(counters + d, 1u);
          mbar_arrive(&pub_empty[g * kPubQ + ps[g]]);
          if (++ps[g] == kPubQ) {
            ps[g] = 0;
            ph[g] ^= 1;
          }
        }
        if (!any) __nanosleep(100);  // idle: leave the issue slots to the SM sub-partition's other warps
      }
    }
  } else if (warp == 3) {
    if (lane == 0 && !ra.next_tile) {  // greedy: the producer claims its own tiles
      // ------------------------------------------------ tile scheduler
      // Claims this CTA's next tile (static round-robin, or the head of a
      // ready per-tenant queue) up to kSchedQ tiles ahead of the producer, so
      // the claim's atomic round trip overlaps the producer's loads.
      if (ra.heads) asm volatile("griddepcontrol.wait;" ::: "memory");  // queue heads reset by the prior launch
      uint32_t sslot = 0, sphase = 0;
      int static_next = blockIdx.x;
      int rr = ra.nq > 0 ? static_cast<int>(blockIdx.x) % ra.nq : 0;
      auto claim = [&]() -> int {
        if (!ra.heads) {
          const int t = static_next < n_tiles ? static_next : -1;
          static_next += gridDim.x;
          return t;
        }
        for (;;) {
          bool pending = false;
          for (int i = 0; i < ra.nq; ++i) {
            const int q = rr + i < ra.nq ? rr + i : rr + i - ra.nq;
            const uint32_t len = static_cast<uint32_t>(ra.qlen[q]);
            const uint32_t h = *reinterpret_cast<volatile uint32_t*>(ra.heads + q);
            if (h >= len) continue;
            pending = true;
            // peek (no contention): skip a queue whose head is still blocked
            const TileEntry& head = tiles[ra.qbeg[q] + static_cast<int>(h)];
            if (head.dep >= 0 && !range_ready(counters, targets, head.dep, head.dep_n)) continue;
            if (head.rdep >= 0 && !range_ready(counters, targets, head.rdep, head.rdep_n)) continue;
            // claim with one fetch-and-add; a claim that overtook the peeked
            // head may land on a not-yet-ready tile, which the gate waits for
            // (queue order is a topological order, so this cannot deadlock)
            const uint32_t got = atomicAdd(ra.heads + q, 1u);
            if (got < len) {
              rr = q;
              return ra.qbeg[q] + static_cast<int>(got);
            }
          }
          if (!pending) return -1;
          __nanosleep(100);
        }
      };
      for (;;) {
        const int t = claim();
        if (t >= 0) {  // pull the claimed tile's entry and member descriptor toward the SM
          const char* p0 = reinterpret_cast<const char*>(slots + tiles[t].member);
#pragma unroll
          for (int i = 0; i < static_cast<int>(sizeof(MemberDesc)); i += 128)
            asm volatile("prefetch.global.L1 [%0];" ::"l"(p0 + i));
          prefetch_tmap(&reinterpret_cast<const MemberDesc*>(p0)->a);  // the producer's load maps
          prefetch_tmap(&reinterpret_cast<const MemberDesc*>(p0)->b);
          prefetch_tmap(&reinterpret_cast<const MemberDesc*>(p0)->c);  // the epilogue's store map
        }
        TileRec r;
        if (t >= 0) load_tile_rec(tiles, slots, t, r);  // global reads before the slot wait
        mbar_wait(&sq_empty[sslot], sphase ^ 1);
        sq[sslot] = t;
        if (t >= 0) srec[sslot] = r;
        mbar_arrive(&sq_full[sslot]);
        if (++sslot == kSchedQ) {
          sslot = 0;
          sphase ^= 1;
        }
        if (t < 0) break;
      }
    }
  } else if (warp >= 4) {
    // -------------------------------------------------- epilogue: 2 warpgroups
    // Warpgroup g drains accumulator buffer g, i.e. every other tile, so one
    // group's store-completion wait (needed before publishing a round
    // counter) overlaps the other group's TMEM drain.  (Draining every tile
    // with both groups halves a tile's drain latency but serialises the
    // publish waits; measured slower on the headline round.)
    const int quarter = warp & 3;  // the TMEM lane quarter this warp may access
    const uint32_t acc = static_cast<uint32_t>((warp - 4) >> 2);
    int mma_local = 0;  // accumulator tiles seen (depthwise tiles have none)
    uint8_t* stage_buf = epi + (warp - 4) * kEpiBufs * kEpiBufBytes;
    uint32_t acc_phase = 0, buf = 0;
    int issued = 0;
    uint32_t qslot = 0, qphase = 0;
    bool dw_gated = false;  // PDL wait done before this warp's first depthwise tile
    int cc_local = 0;       // staged CUDA-core tiles seen: warpgroup (cc_local & 1) computes each
    uint32_t pslot = 0, pphase = 0;  // this group's publish queue (its first lane pushes)
    for (;;) {
      int t = 0;
      uint32_t aux = 0;
      if (lane == 0) {
        mbar_wait(&tq_full[qslot], qphase);
        t = tq[qslot];
        aux = tq_aux[qslot];
        mbar_arrive(&tq_empty[qslot]);
      }
      t = __shfl_sync(0xffffffffu, t, 0);
      aux = __shfl_sync(0xffffffffu, aux, 0);
      if (++qslot == kTileQ) {
        qslot = 0;
        qphase ^= 1;
      }
      if (t < 0) {
        if ((warp & 3) == 0 && lane == 0) {  // end of this group's publish stream
          mbar_wait(&pub_empty[acc * kPubQ + pslot], pphase ^ 1);
          pub_q[acc * kPubQ + pslot] = -1;
          mbar_arrive(&pub_full[acc * kPubQ + pslot]);
        }
        break;
      }
      if ((t & (kDwTag | kStagedTag)) == (kDwTag | kStagedTag)) {
        // staged CUDA-core tile: one warpgroup computes it from its ring slot
        // (the two groups alternate, so one group's store / publish latency
        // overlaps the other's compute), frees the slot, publishes once
        if ((cc_local++ & 1) != static_cast<int>(acc)) continue;
        t &= ~(kDwTag | kStagedTag);
        const TileEntry te = tiles[t];
        const MemberDesc* md = slots + te.member;
        const uint32_t slot = aux & 15u;
        mbar_wait(&full[slot], (aux >> 4) & 1u);
        const int gt = (warp & 3) * 32 + lane;
        if (trace && gt == 0) {
          const uint64_t now = globaltimer();
          trace[6 * t + 2] = trace[6 * t + 3] = trace[6 * t + 4] = now;
        }
        const uint8_t* src = ring + ((aux >> 8) << 10);
        if (md->a_mode == kDepthwise)
          staged_dw_tile(md, te, src, gt);
        else
          staged_pool_tile(md, te, src, gt, 1 + static_cast<int>(acc));
        named_barrier(1 + static_cast<int>(acc), 128);  // the group's smem reads and global stores are issued
        if (gt == 0) {
          mbar_arrive(&empty[slot]);
          // the publisher warp releases the counter (its gpu-scope release
          // covers this group's stores: bar.sync, then mbarrier arrive/wait)
          if (te.done >= 0) {
            mbar_wait(&pub_empty[acc * kPubQ + pslot], pphase ^ 1);
            pub_q[acc * kPubQ + pslot] = te.done;
            mbar_arrive(&pub_full[acc * kPubQ + pslot]);
            if (++pslot == kPubQ) {
              pslot = 0;
              pphase ^= 1;
            }
          }
          if (trace) trace[6 * t + 5] = globaltimer();
        }
        continue;
      }
      if (t & kDwTag) {
        t &= ~kDwTag;
        const TileEntry te = tiles[t];
        const MemberDesc* md = slots + te.member;
        // all eight epilogue warps share the tile; gate on the PDL
        // prerequisite and the tenant's previous layer like the A producer
        if (!dw_gated) {
          asm volatile("griddepcontrol.wait;" ::: "memory");
          dw_gated = true;
        }
        if (te.dep >= 0) {
          if (lane == 0) wait_range(counters, targets, te.dep, te.dep_n, 32);
          __syncwarp();
        }
        if (trace && warp == 4 && lane == 0) {
          const uint64_t now = globaltimer();
          for (int j = 0; j < 5; ++j) trace[6 * t + j] = now;  // no load / MMA phases
        }
        if (md->a_mode == kDepthwise)
          depthwise_tile(md, te, warp - 4, lane);
        else
          pool_tile(md, te, warp - 4, lane);
        __syncwarp();
        if (trace && warp == 4 && lane == 0) trace[6 * t + 5] = globaltimer();
        if (te.done >= 0 && lane == 0) {
          __threadfence();
          atomicAdd(counters + te.done, 1u);
        }
        continue;
      }
      const bool mine = (mma_local & 1) == static_cast<int>(acc);
      ++mma_local;
      if (!mine) continue;
      const TileEntry te = tiles[t];
      const MemberDesc* md = slots + te.member;
      const int tall = md->tall;
      const int m0 = te.m_tile * (kBM << tall) + quarter * 32;
      const int n0 = te.n_tile * md->n_tile;
      const int cols = min(md->n_tile, md->n - n0);
      const int act = md->act;
      const Clamp ck = clamp_of(act);
      const int sw = (lane >> 1) & 3;  // SWIZZLE_64B: 16B chunk j of a 64 B row -> j ^ row[2:1]
      // Claim the next staging buffer once the store issued from it two
      // chunks ago has finished reading it.
      auto claim = [&]() -> uint8_t* {
        if (lane == 0 && issued >= kEpiBufs)
          asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(kEpiBufs - 1) : "memory");
        __syncwarp();
        return stage_buf + buf * kEpiBufBytes;
      };
      auto issue = [&]() {
        ++issued;
        buf = buf + 1 == kEpiBufs ? 0 : buf + 1;
      };
      // 32 fp32 accumulators of this lane's row (residual already added by
      // the MMA) -> activation -> bf16 -> one 32x32 store box.
      auto store_bf16 = [&](uint32_t (&v)[32], int c, int mrow) {
        if (act == kActGelu) {
#pragma unroll
          for (int i = 0; i < 32; ++i) v[i] = __float_as_uint(gelu_f(__uint_as_float(v[i])));
        }
        uint8_t* sbuf = claim();
        uint8_t* row = sbuf + lane * 64;
        // bf16 packing: one cvt per pair (the .relu form for relu; relu6 adds
        // its upper clamp first) -- the activation branch is warp-uniform
        auto pack4 = [&](auto cvt, int j) {
          uint4 pk;
          pk.x = cvt(__uint_as_float(v[8 * j + 0]), __uint_as_float(v[8 * j + 1]));
          pk.y = cvt(__uint_as_float(v[8 * j + 2]), __uint_as_float(v[8 * j + 3]));
          pk.z = cvt(__uint_as_float(v[8 * j + 4]), __uint_as_float(v[8 * j + 5]));
          pk.w = cvt(__uint_as_float(v[8 * j + 6]), __uint_as_float(v[8 * j + 7]));
          *reinterpret_cast<uint4*>(row + ((j ^ sw) << 4)) = pk;
        };
        if (act == kActRelu || act == kActRelu6) {
          if (act == kActRelu6) {
#pragma unroll
            for (int i = 0; i < 32; ++i) v[i] = __float_as_uint(fminf(__uint_as_float(v[i]), 6.f));
          }
#pragma unroll
          for (int j = 0; j < 4; ++j) pack4([](float a, float b) { return cvt_bf16x2_relu(a, b); }, j);
        } else {
#pragma unroll
          for (int j = 0; j < 4; ++j) pack4([](float a, float b) { return cvt_bf16x2(a, b); }, j);
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncwarp();
        if (lane == 0) {
          tma_store_2d(&md->c, sbuf, n0 + c, mrow);
          asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        }
        issue();
      };
      mbar_wait(&acc_full[acc], acc_phase);
      tc_fence_after();
      if (trace && quarter == 0 && lane == 0) trace[6 * t + 4] = globaltimer();
      const uint32_t taddr = tmem_base + (static_cast<uint32_t>(quarter * 32) << 16) + acc * BN;
      bool publish = te.done >= 0;
      if (te.splits > 1) {
        // ---- split-K partial: coalesced fp32 red.add into the workspace tile.
        // Lane-major layout: the 32 lanes' float4 of (chunk c, j) are 512
        // contiguous bytes, so each warp-wide REDG.F32x4 is fully coalesced.
        constexpr int kChunks = BN / kEpiChunk;
        float* wq = ra.ws + (static_cast<int64_t>(te.ws) * 4 + quarter) * (kChunks * 8 * 128);
        uint32_t* ctr = ra.split_ctr + te.ws * 4 + quarter;
        // Finisher: with two splits, whichever warp of the pair arrives
        // second (per TMEM lane quarter), so it never waits for its partner's
        // K loop, only for the partner's partial store (the first arrival
        // counts 1, its 32 lanes release 1 each after storing, the second
        // adds its own 1: 34); with more, the split holding the K tail waits
        // for every other split's lanes.
        bool finisher;
        uint32_t want;
        if (te.splits == 2) {
          uint32_t old = 0;
          if (lane == 0) old = atomicAdd(ctr, 1u);
          finisher = __shfl_sync(0xffffffffu, old, 0) != 0;
          want = 34u;
        } else {
          finisher = te.kb_end == md->k_blocks;
          want = static_cast<uint32_t>(te.splits - 1) * 32u;
        }
        if (!finisher) {
          // fire and forget: reduce-add the partial (two splits: the only
          // other writer is the finisher, so a plain store), then a release
          // arrival per lane (orders this lane's writes before it); no waiting
          const bool plain = te.splits == 2;
          for (int c = 0; c < cols; c += kEpiChunk) {
            uint32_t v[32];
            tmem_ld32(taddr + c, v);
            float* wc = wq + (c / kEpiChunk) * (8 * 128) + lane * 4;
            if (plain) {
#pragma unroll
              for (int j = 0; j < 8; ++j)
                __stcg(reinterpret_cast<float4*>(wc + j * 128),
                       make_float4(__uint_as_float(v[4 * j]), __uint_as_float(v[4 * j + 1]),
                                   __uint_as_float(v[4 * j + 2]), __uint_as_float(v[4 * j + 3])));
            } else {
#pragma unroll
              for (int j = 0; j < 8; ++j)
                asm volatile("red.relaxed.gpu.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(wc + j * 128),
                             "f"(__uint_as_float(v[4 * j])), "f"(__uint_as_float(v[4 * j + 1])),
                             "f"(__uint_as_float(v[4 * j + 2])), "f"(__uint_as_float(v[4 * j + 3]))
                             : "memory");
            }
          }
          tc_fence_before();
          mbar_arrive(&acc_empty[acc]);
          asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(ctr) : "memory");
          publish = false;
        } else {
          // finisher: wait for the other splits' lanes, add its own TMEM
          // partial to their sum, store bf16, clear the workspace
          wait_counter(ctr, want, 40);
          const bool clear_ws = te.splits > 2;  // a two-split partial is overwritten, not accumulated, next time
          // the other splits' sum for chunk c + 1 is loaded while chunk c is
          // packed and stored: one L2 round trip in flight behind the stores
          float4 f[8];
          auto load_part = [&](int c) {
            const float4* src = reinterpret_cast<const float4*>(wq + (c / kEpiChunk) * (8 * 128) + lane * 4);
#pragma unroll
            for (int j = 0; j < 8; ++j) f[j] = __ldcg(src + j * 32);
          };
          load_part(0);
          for (int c = 0; c < cols; c += kEpiChunk) {
            uint32_t v[32];
            tmem_ld32(taddr + c, v);
#pragma unroll
            for (int j = 0; j < 8; ++j) {
              v[4 * j] = __float_as_uint(__uint_as_float(v[4 * j]) + f[j].x);
              v[4 * j + 1] = __float_as_uint(__uint_as_float(v[4 * j + 1]) + f[j].y);
              v[4 * j + 2] = __float_as_uint(__uint_as_float(v[4 * j + 2]) + f[j].z);
              v[4 * j + 3] = __float_as_uint(__uint_as_float(v[4 * j + 3]) + f[j].w);
            }
            if (clear_ws) {
              float4* dst = reinterpret_cast<float4*>(wq + (c / kEpiChunk) * (8 * 128) + lane * 4);
#pragma unroll
              for (int j = 0; j < 8; ++j) __stcg(dst + j * 32, make_float4(0.f, 0.f, 0.f, 0.f));
            }
            if (c + kEpiChunk < cols) load_part(c + kEpiChunk);
            if (m0 < md->m) store_bf16(v, c, m0);
          }
          tc_fence_before();
          mbar_arrive(&acc_empty[acc]);
          __syncwarp();
          if (lane == 0) *ctr = 0;  // next round (kernel boundary orders it)
        }
      } else {
        // one or two (tall tile) 128-row halves; this warp's 32 rows of each
        for (int h = 0; h <= tall; ++h) {
          const int mrow = m0 + h * kBM;
          if (mrow >= md->m) break;  // warp-uniform: no real row left in this quarter
          const uint32_t tcol = taddr + h * md->n_tile;
          for (int c = 0; c < cols; c += kEpiChunk) {
            uint32_t v[32];
            tmem_ld32(tcol + c, v);
            store_bf16(v, c, mrow);
          }
        }
        tc_fence_before();
        mbar_arrive(&acc_empty[acc]);
      }
      acc_phase ^= 1;
      if (trace && quarter == 0 && lane == 0) trace[6 * t + 5] = globaltimer();
      if (publish && te.splits > 1) {
        // split finisher (chosen per lane quarter): this warp publishes its
        // own stores -- complete, ordered before generic-proxy accesses,
        // released with the counter increment itself
        if (lane == 0) {
          asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
          asm volatile("fence.proxy.async.global;" ::: "memory");
          red_release_add(counters + te.done, 1u);
        }
      } else if (publish) {
        // whole-tile publish: each warp's stores complete (its lane 0 issued
        // them all), the warpgroup meets, and one release increment covers
        // the four warps' stores (cumulative through the barrier): one
        // MEMBAR.GPU per tile instead of one per warp
        if (lane == 0) {
          asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
          asm volatile("fence.proxy.async.global;" ::: "memory");
        }
        named_barrier(1 + static_cast<int>(acc), 128);
        if (quarter == 0 && lane == 0) red_release_add(counters + te.done, 1u);
      }
    }
    if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  }

  // (ptxas may hoist this stamp above the barrier: it reads as the
  // producer's loop end; warp 2's stamp below is the barrier release)
  if (cta_trace && threadIdx.x == 0) cta_trace[2] = clock64();
  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    if (cta_trace && lane == 0) cta_trace[3] = clock64();
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(C::kTmemCols)
                 : "memory");
    if (cta_trace && lane == 0) cta_trace[4] = clock64();
  }
  // Round programs reset their own completion counters: the last CTA to
  // finish zeroes them, so a replay needs no memset node before the kernel.
  // The next launch touches counters only after griddepcontrol.wait, i.e.
  // after this grid (and the reset) completed.
  if (ra.exit_ctr) {
    if (threadIdx.x == 0) {
      __threadfence();
      *tmem_slot = atomicAdd(ra.exit_ctr, 1u) == gridDim.x - 1 ? 1u : 0u;
    }
    __syncthreads();
    if (*tmem_slot) {
      __threadfence();
      for (int i = threadIdx.x; i < ra.n_reset; i += blockDim.x) ra.counters[i] = 0;
      if (threadIdx.x == 0) *ra.exit_ctr = 0;
    }
  }
  if (cta_trace && threadIdx.x == 0) cta_trace[5] = clock64();
}

// Registration-time repack of narrow-channel conv weights: KRSC rows with
// C_in channels per tap -> kNarrowC channels per tap (zero padded), the K order
// of the narrow im2col A operand.
__global__ void pad_narrow_weights(const __nv_bfloat16* __restrict__ src, int64_t ldw, __nv_bfloat16* __restrict__ dst,
                                   int cout, int taps, int cin) {
  const int row = taps * kNarrowC;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < cout * row; i += gridDim.x * blockDim.x) {
    const int o = i / row;
    const int rem = i - o * row;
    const int tap = rem / kNarrowC;
    const int c = rem - tap * kNarrowC;
    dst[i] = c < cin ? src[static_cast<int64_t>(o) * ldw + tap * cin + c] : __float2bfloat16(0.f);
  }
}

// Depthwise filters [C, ldw] (R*S taps per row) -> tap-major [R*S, C].
__global__ void dw_tap_major(const __nv_bfloat16* __restrict__ src, int64_t ldw, __nv_bfloat16* __restrict__ dst, int ch,
                             int taps) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < ch * taps; i += gridDim.x * blockDim.x) {
    const int k = i / ch, c = i - k * ch;
    dst[i] = src[static_cast<int64_t>(c) * ldw + k];
  }
}

// Row-folded weights: dst[o, r*kFoldC + j] = src[o, r*S*Cin + j] for
// j < S*Cin and r < R, zero elsewhere (rows r in [R, rpad) pad K to whole k-blocks).
__global__ void fold_weights(const __nv_bfloat16* __restrict__ src, int64_t ldw, __nv_bfloat16* __restrict__ dst,
                             int cout, int R, int sc, int rpad) {
  const int row = rpad * kFoldC;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < cout * row; i += gridDim.x * blockDim.x) {
    const int o = i / row;
    const int rem = i - o * row;
    const int r = rem / kFoldC, j = rem - r * kFoldC;
    dst[i] = (r < R && j < sc) ? src[static_cast<int64_t>(o) * ldw + r * sc + j] : __float2bfloat16(0.f);
  }
}

// Row-fold pre-pass: X'[b, h, q, j] = X[b, h, q*stride - pad + j / Cin, j % Cin]
// for j < S*Cin (zero outside the image and for j >= S*Cin).  One thread per
// folded pixel (64 B: four 16 B stores); blockIdx.y selects the job.
struct FoldJob {
  const __nv_bfloat16* x;
  __nv_bfloat16* out;
  int batch, H, W, Cin, S, stride, pad, Q;
};
struct FoldBatch {
  FoldJob job[16];
};

__global__ void __launch_bounds__(128) fold_rows(const __grid_constant__ FoldBatch fb) {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  const FoldJob& j = fb.job[blockIdx.y];
  const unsigned short* xs = reinterpret_cast<const unsigned short*>(j.x);
  const int sc = j.S * j.Cin;
  const int total = j.batch * j.H * j.Q;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < total; i += gridDim.x * blockDim.x) {
    const int q = i % j.Q;
    const int bh = i / j.Q;  // b * H + h
    const int iw0 = q * j.stride - j.pad;
    const unsigned short* row = xs + static_cast<int64_t>(bh) * j.W * j.Cin;
    uint32_t packed[kFoldC / 2];
    int s = 0, c = 0;
#pragma unroll
    for (int e = 0; e < kFoldC; ++e) {
      uint32_t v = 0;
      if (e < sc) {
        const int iw = iw0 + s;
        if (iw >= 0 && iw < j.W) v = __ldg(row + iw * j.Cin + c);
        if (++c == j.Cin) {
          c = 0;
          ++s;
        }
      }
      if (e & 1)
        packed[e >> 1] |= v << 16;
      else
        packed[e >> 1] = v;
    }
    uint4* dst = reinterpret_cast<uint4*>(j.out + static_cast<int64_t>(i) * kFoldC);
#pragma unroll
    for (int u = 0; u < kFoldC / 8; ++u)
      dst[u] = make_uint4(packed[4 * u], packed[4 * u + 1], packed[4 * u + 2], packed[4 * u + 3]);
  }
}

// One thread per (row m, 8-element chunk of k): 32-bit index math, one
// coalesced 16-byte store per thread; ldk % 8 == 0.  Explicit im2col for
// convs whose Cin does not fill a 128 B TMA channel box (the 3-channel stem).
__global__ void im2col_prepass(const __nv_bfloat16* __restrict__ x, __nv_bfloat16* __restrict__ out, int batch, int H,
                               int W, int Cin, int R, int S, int stride, int pad, int P, int Q, int ldk) {
  const int chunks = ldk >> 3;
  const int rows = batch * P * Q;
  const int K = R * S * Cin;
  const unsigned short* xs = reinterpret_cast<const unsigned short*>(x);
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < rows * chunks; i += gridDim.x * blockDim.x) {
    const int m = i / chunks;
    const int k0 = (i - m * chunks) << 3;
    const int q = m % Q;
    const int t = m / Q;
    const int p = t % P;
    const int b = t / P;
    const int h0 = p * stride - pad, w0 = q * stride - pad;
    int c = k0 % Cin;
    int tap = k0 / Cin;
    int s = tap % S, r = tap / S;
    uint32_t packed[4];
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      unsigned short v = 0;
      if (k0 + j < K) {
        const int ih = h0 + r, iw = w0 + s;
        if (ih >= 0 && ih < H && iw >= 0 && iw < W) v = __ldg(xs + ((b * H + ih) * W + iw) * Cin + c);
      }
      if (j & 1)
        packed[j >> 1] |= static_cast<uint32_t>(v) << 16;
      else
        packed[j >> 1] = v;
      if (++c == Cin) {
        c = 0;
        if (++s == S) {
          s = 0;
          ++r;
        }
      }
    }
    *reinterpret_cast<uint4*>(out + static_cast<int64_t>(m) * ldk + k0) =
        make_uint4(packed[0], packed[1], packed[2], packed[3]);
  }
}

}  // namespace dev
}  // namespace gmb
