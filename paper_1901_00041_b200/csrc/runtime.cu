// B200 runtime: per-GPU context, tenant registration (member descriptors with
// TMA maps), plan preparation (device tile tables, cached per member list) and
// super-kernel launch.  C-ABI entry points for the device side live here.
#include <functional>
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstring>
#include <deque>
#include <condition_variable>
#include <map>
#include <mutex>
#include <random>
#include <set>
#include <string>
#include <thread>
#include <unordered_map>
#include <vector>

#include "abi.hpp"
#include "superkernel.cuh"

namespace gmb {

namespace {

void cuda_check(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw CudaError(std::string(what) + ": " + cudaGetErrorString(e));
}

using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                   const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                   CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
using EncodeIm2colFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                    const cuuint64_t*, const int*, const int*, cuuint32_t, cuuint32_t,
                                    const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                    CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

void* driver_entry(const char* name) {
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  cuda_check(cudaGetDriverEntryPoint(name, &fn, cudaEnableDefault, &q), name);
  if (q != cudaDriverEntryPointSuccess || !fn) throw CudaError(std::string("driver entry point missing: ") + name);
  return fn;
}

// tcgen05 kind::f16 instruction descriptor: D fp32, A/B bf16, both K-major,
// N>>3 at [17,23), M>>4 at [24,29).
uint32_t make_idesc(int umma_n) {
  return (1u << 4) | (1u << 7) | (1u << 10) | (static_cast<uint32_t>(umma_n >> 3) << 17) |
         (static_cast<uint32_t>(dev::kBM >> 4) << 24);
}

// Box rows per member: only real rows move (a small-M member's A box and a
// small-N member's B box shrink; the MMA's extra A rows are discarded).
int a_box_rows(int64_t m) { return static_cast<int>(std::min<int64_t>(dev::kBM, (m + 7) / 8 * 8)); }
int b_box_rows(int64_t n, int bn) { return static_cast<int>(std::min<int64_t>(bn, (n + 15) / 16 * 16)); }

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

// Operators computed on CUDA cores inside the persistent kernel (no tensor-core tile).
bool cuda_core_kind(int kind) {
  return kind == GM_LAYER_DWCONV || kind == GM_LAYER_MAXPOOL || kind == GM_LAYER_AVGPOOL;
}
// Output rows per tile of a CUDA-core operator.
int64_t cuda_core_rows(int kind) { return kind == GM_LAYER_DWCONV ? dev::kDwTileM : dev::kPoolTileM; }


}  // namespace

// One registered (tenant, layer) operator.
struct Operator {
  int kind = GM_LAYER_GEMM;
  Shape shape;      // the GEMM the planner sees (m includes batch)
  Conv conv;
  int batch = 1;
  int slot = -1;    // index into the device MemberDesc array
  int tenant = -1, layer = -1;
  int n_tile = 256;  // output columns per tile (the kernel's BN)
  // narrower-N variants of the same operator (descriptor slots), chosen per
  // plan when the plan's full-width tiles cannot fill the SMs
  int narrow_slot[2] = {-1, -1};
  int narrow_w[2] = {0, 0};
  int tall_slot = -1;  // 256-row x <=128-column variant (tiled / im2col A, M >= 256, N <= 128)
  const void* b_ptr = nullptr;  // weights as the B operand (for the variants' maps)
  int64_t b_k = 0, b_ld = 0;
  bool prepass = false;
  bool fold = false;        // the pre-pass is the row fold (kAIm2colFold)
  const void* x = nullptr;
  void* scratch = nullptr;  // explicit-im2col rows [M, ldk], or the folded input [b, H, Q, 32]
  int64_t ldk = 0;
  void* wpad = nullptr;     // narrow-channel conv: weights repacked to 8 channels per tap
  int64_t kernel_k = 0;     // K the kernel iterates (0 = shape.k)
  // dataflow (gm_layer_desc.src / res_src): producing layers of x and of the
  // residual within the tenant (-1 = external), and this layer's output range
  int src = -1, res_src = -1;
  const char* y = nullptr;
  int64_t y_bytes = 0;
  int64_t x_bytes = 0;           // extent of the input x (gm_request_io copies)
  int64_t x_pitch = 0;           // elements per input row (GEMM) or pixel (windowed ops)
  const char* res = nullptr;     // residual base and row stride (elements)
  int64_t ldr = 0;
  int64_t cc_rows = 0;  // staged CUDA-core tile: output pixels per tile (0 = register-path tile)
};

// Rows (output pixels) per tile of an operator's descriptor variant.
int64_t tile_rows_of(const Operator& op, bool tall) {
  if (cuda_core_kind(op.kind)) return op.cc_rows > 0 ? op.cc_rows : cuda_core_rows(op.kind);
  return int64_t{dev::kBM} << (tall ? 1 : 0);
}

struct Prepared {
  dev::TileEntry* tiles = nullptr;
  int n_tiles = 0;
  std::vector<int> prepass_ops;  // indices into Runtime::flat
  // round programs only: one completion counter per member instance
  uint32_t* counters = nullptr;
  uint32_t* targets = nullptr;
  int n_counters = 0;
  // split-K workspace: fp32 [n_ws * 128, bn] + per (tile, quarter) arrivals
  float* ws = nullptr;
  CUtensorMap* ws_map = nullptr;  // device copy, 64 B aligned
  uint32_t* split_ctr = nullptr;
  int n_ws = 0;
  std::vector<uint16_t> tile_plan;  // round programs: plan index of every tile (profiling)
  // dynamic schedule: per-tenant work queues (heads live after the counters)
  uint32_t* heads = nullptr;
  int32_t* qinfo = nullptr;  // [nq] begins then [nq] lengths
  int nq = 0;
  bool self_reset = true;  // round programs: counters in use, the last CTA resets them
  double measured_s = 0;   // serving: EWMA of this program's device time when a dispatch ran it alone
  bool greedy = false;  // greedy in-order claiming (one claim counter after the counters and queue heads)
  // input-gated round programs (end-to-end serving): per tenant, a counter
  // (target 1) its first layer depends on, set by a 4-byte DMA after the
  // tenant's H2D copy (and layer-0 pre-pass) on a side stream
  std::vector<std::pair<int, int>> gates;  // (tenant, counter index)
  std::vector<int> gated_prepass;          // layer-0 pre-pass ops, run per tenant on the copy stream

  void release() {
    cudaFree(qinfo);
    cudaFree(tiles);
    cudaFree(counters);
    cudaFree(targets);
    cudaFree(ws);
    cudaFree(ws_map);
    cudaFree(split_ctr);
  }
};

// One gm_dispatch awaiting gm_poll_completions: events bracket the
// super-kernel (execution time) and the whole dispatch (copy-out included).
struct InFlight {
  cudaEvent_t exec0 = nullptr, exec1 = nullptr, done = nullptr;
  std::vector<Request> members;
  int64_t dispatch_ns = 0;
};

struct Runtime {
  std::vector<gm_dispatch_event> serve_trace;
  std::deque<InFlight> inflight;     // gm_dispatch -> gm_poll_completions
  std::vector<cudaEvent_t> ev_pool;  // recycled timing events  // the last gm_serve's dispatches (gm_serve_trace)
  int device = -1;
  int sms = 0;
  int driver_version = 0;
  EncodeTiledFn encode_tiled = nullptr;
  EncodeIm2colFn encode_im2col = nullptr;
  std::vector<std::vector<int>> tenant_ops;  // tenant -> indices into flat
  std::vector<double> tenant_slo;            // seconds per pass
  std::vector<std::vector<gm_layer_desc>> tenant_layers;  // registration descriptors (gm_migrate_tenant)
  std::vector<int32_t> tenant_conc;
  std::vector<void*> owned;                  // device buffers this runtime allocated (migrated tenants)
  std::vector<Operator> flat;
  std::vector<int> slot_op;  // descriptor slot -> index into flat
  std::vector<dev::MemberDesc> host_desc;
  dev::MemberDesc* d_desc = nullptr;
  std::vector<dev::MemberDesc*> retired_desc;  // outgrown descriptor arrays (captured graphs may point at them)
  size_t d_cap = 0;
  std::unordered_map<std::string, Prepared> prepared;
  std::unordered_map<std::string, Prepared> rounds;
  std::recursive_mutex rounds_mu;
  // serving: EWMA of measured / planned device time of single-tenant and of
  // multi-tenant round programs (the planner's b200 profile is a roofline;
  // few-tile rounds run latency-bound)
  double serve_ratio[2] = {1.0, 1.0};
  // Drop a round program from the cache; its device tables are freed once the
  // caller guarantees no launch of it is pending (returns false if unknown).
  bool forget_round(const Prepared* p, std::vector<Prepared>& graveyard) {
    std::lock_guard<std::recursive_mutex> lock(rounds_mu);
    for (auto it = rounds.begin(); it != rounds.end(); ++it)
      if (&it->second == p) {
        graveyard.push_back(std::move(it->second));
        rounds.erase(it);
        return true;
      }
    return false;
  }
  int64_t n_superkernels = 0, n_prepasses = 0, n_tiles = 0;
  bool pdl = true;      // programmatic dependent launch between consecutive super-kernels
  bool split_k = false;      // round programs split few-tile long-K members (opt-in)
  int64_t max_splits = 4;
  int64_t split_min_kb = 8;  // fewest k-blocks per split
  // Weight-streaming members (M <= 64 rows, >= skinny_min_mb MB of weights,
  // e.g. VGG's fc6/fc7): full-width tiles split over K so the weights stream
  // through (up to) every SM; their fp32 partials are few (M rows).  0 = off.
  int64_t skinny_min_mb = 64;
  int64_t skinny_max_splits = 8;
  int64_t narrow_min_tiles = 20;  // >0: in a plan that cannot fill the SMs, narrow a member's N tile
                                 // (256 -> 128 -> 64) until it has this many tiles
  int64_t split_wide_kb = 0;     // >0: a member narrowed below 128 columns with >= this many k-blocks keeps
                                 // 128-column tiles and splits K instead (same tile count, half the k-blocks each)
  bool row_fold = true;          // S*Cin <= 32 convs (RGB stems) use the row-folded im2col path
  bool staged_cc = true;         // pools / depthwise convs as staged CUDA-core tiles (applies at registration)
  bool dynamic_schedule = false;  // round programs: per-tenant ready queues (else static round-robin)
  bool greedy_schedule = false;   // round programs: greedy in-order tile claiming (else static round-robin)
  bool tall_tiles = true;         // 256-row tiles for narrow members of throughput-bound plans
  int ring_layouts = 1;           // narrow members use the 6 x 32 KB ring layout (applies at registration)
  int critical_order = -1;        // round programs: tile order 0 plan, 1 remaining chain work, 2 chain progress,
                                  // -1 auto (2: chain progress)
  int64_t tall_min_tiles = 0;     // concurrent same-shape tiles that make a member "throughput-bound" (0 = 2 x SMs)
  int bn = 256;     // N tile of the super-kernel (== DeviceSpec.tile_n)
  uint32_t* host_one = nullptr;  // pinned 4-byte 1: DMA source that opens an input gate
  void* ident = nullptr;         // bf16 identity [kIdentN, kIdentN]: B operand of residual k-blocks
  int smem_bytes = 0;
  const void* kernel = nullptr;

  ~Runtime() {
    if (device < 0) return;
    cudaSetDevice(device);
    cudaDeviceSynchronize();
    for (auto& [k, p] : prepared) p.release();
    for (auto& [k, p] : rounds) p.release();
    for (Operator& op : flat) {
      cudaFree(op.scratch);
      cudaFree(op.wpad);
    }
    cudaFree(d_desc);
    for (dev::MemberDesc* p : retired_desc) cudaFree(p);
    cudaFree(ident);
    for (void* p : owned) cudaFree(p);
    cudaFreeHost(host_one);
    for (InFlight& f : inflight)
      for (cudaEvent_t e : {f.exec0, f.exec1, f.done}) cudaEventDestroy(e);
    for (cudaEvent_t e : ev_pool) cudaEventDestroy(e);
  }

  cudaEvent_t take_event() {
    if (!ev_pool.empty()) {
      cudaEvent_t e = ev_pool.back();
      ev_pool.pop_back();
      return e;
    }
    cudaEvent_t e;
    cuda_check(cudaEventCreate(&e), "cudaEventCreate");
    return e;
  }

  void init(int dev_index, const Device& spec) {
    if (spec.tile_m != dev::kBM || (spec.tile_n != 128 && spec.tile_n != 256))
      throw std::invalid_argument("b200 runtime needs tile_m 128 and tile_n 128 or 256 (the super-kernel tile)");
    bn = static_cast<int>(spec.tile_n);
    int count = 0;
    if (cudaGetDeviceCount(&count) != cudaSuccess || count == 0) throw NoDevice("no CUDA device visible");
    if (dev_index >= count) throw NoDevice("CUDA device index out of range");
    cuda_check(cudaSetDevice(dev_index), "cudaSetDevice");
    cudaDeviceProp prop;
    cuda_check(cudaGetDeviceProperties(&prop, dev_index), "cudaGetDeviceProperties");
    if (prop.major != 10 || prop.minor != 0)
      throw NoDevice("super-kernel is built for sm_100a; device is sm_" + std::to_string(prop.major) +
                     std::to_string(prop.minor));
    device = dev_index;
    sms = prop.multiProcessorCount;
    cuda_check(cudaDriverGetVersion(&driver_version), "cudaDriverGetVersion");
    encode_tiled = reinterpret_cast<EncodeTiledFn>(driver_entry("cuTensorMapEncodeTiled"));
    encode_im2col = reinterpret_cast<EncodeIm2colFn>(driver_entry("cuTensorMapEncodeIm2col"));
    if (bn == 256) {
      kernel = reinterpret_cast<const void*>(&dev::superkernel<256>);
      smem_bytes = dev::Cfg<256>::kSmemBytes;
    } else {
      kernel = reinterpret_cast<const void*>(&dev::superkernel<128>);
      smem_bytes = dev::Cfg<128>::kSmemBytes;
    }
    cuda_check(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_bytes),
               "cudaFuncSetAttribute");
    cuda_check(cudaHostAlloc(&host_one, sizeof(uint32_t), cudaHostAllocDefault), "cudaHostAlloc");
    *host_one = 1;
    {
      std::vector<uint16_t> eye(static_cast<size_t>(dev::kIdentN) * dev::kIdentN, 0);
      for (int i = 0; i < dev::kIdentN; ++i) eye[static_cast<size_t>(i) * dev::kIdentN + i] = 0x3F80;  // bf16 1.0
      cuda_check(cudaMalloc(&ident, eye.size() * 2), "cudaMalloc(identity)");
      cuda_check(cudaMemcpy(ident, eye.data(), eye.size() * 2, cudaMemcpyHostToDevice), "upload identity");
    }
  }

  // Staged CUDA-core tile geometry (pools, depthwise convs): a tile is `ro`
  // whole output rows of one image x `cc` channels, and its input window --
  // box {cc, (Q-1)*stride+S, (ro-1)*stride+R, 1} of the NHWC input -- lands in
  // one ring slot by a single TMA load.  TMA moves a box one innermost row
  // (cc channels) at a time, so the longest rows win first: cc a multiple of
  // 8 dividing C, up to 128 channels (256-byte rows; at most 32 8-channel
  // groups); then the most output work per tile.  A box that fits a 32 KB
  // slot runs in the narrow ring layout, else in a wide (BN = 256: 48 KB) one.
  // Ops no box fits keep the register-path tile.
  void stage_cuda_core(Operator& op, dev::MemberDesc& md, const void* x) {
    op.cc_rows = 0;
    md.cc_rows = 0;
    if (!staged_cc) return;
    const Conv& c = op.conv;
    const int64_t C = c.in_channels, P = md.pq / md.q, Q = md.q;
    const int64_t Wb = (Q - 1) * c.stride + c.kernel_w;
    if (op.x_pitch % 8 != 0 || Wb > 256 || !aligned16(x)) return;
    const int64_t cap = bn == 256 ? dev::Cfg<256>::kStageBytes : dev::Cfg<128>::kStageBytes;
    int64_t best_cc = 0, best_ro = 0, best_work = 0, best_row = 0;
    for (int64_t cc = 8; cc <= std::min<int64_t>(C, 256); cc += 8) {
      if (C % cc != 0) continue;
      const int64_t row = std::min<int64_t>(cc, 128);
      for (int64_t ro = 1; ro <= P; ++ro) {
        if (P % ro != 0) continue;
        const int64_t Hb = (ro - 1) * c.stride + c.kernel_h;
        if (Hb > 256 || cc * Wb * Hb * 2 > cap) break;
        if (row > best_row || (row == best_row && ro * Q * cc > best_work)) {
          best_row = row;
          best_work = ro * Q * cc;
          best_cc = cc;
          best_ro = ro;
        }
      }
    }
    if (best_cc == 0) return;
    const int64_t Hb = (best_ro - 1) * c.stride + c.kernel_h;
    const cuuint64_t dims[4] = {static_cast<cuuint64_t>(C), static_cast<cuuint64_t>(c.image_w),
                                static_cast<cuuint64_t>(c.image_h), static_cast<cuuint64_t>(op.batch)};
    const cuuint64_t strides[3] = {static_cast<cuuint64_t>(op.x_pitch * 2),
                                   static_cast<cuuint64_t>(op.x_pitch * 2 * c.image_w),
                                   static_cast<cuuint64_t>(op.x_pitch * 2 * c.image_w * c.image_h)};
    const cuuint32_t box[4] = {static_cast<cuuint32_t>(best_cc), static_cast<cuuint32_t>(Wb),
                               static_cast<cuuint32_t>(Hb), 1};
    const cuuint32_t estr[4] = {1, 1, 1, 1};
    const CUresult r = encode_tiled(&md.a, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void*>(x), dims, strides, box,
                                    estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                    CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) throw CudaError("cuTensorMapEncodeTiled (staged CUDA-core input) failed (" +
                                           std::to_string(int(r)) + ")");
    if (op.kind == GM_LAYER_DWCONV) {
      const int taps = static_cast<int>(c.kernel_h * c.kernel_w);
      cuda_check(cudaMalloc(&op.wpad, static_cast<size_t>(taps * C * 2)), "cudaMalloc(depthwise filters)");
      dev::dw_tap_major<<<static_cast<int>(std::min<int64_t>((taps * C + 255) / 256, 4096)), 256>>>(
          md.dw, md.ldw, static_cast<__nv_bfloat16*>(op.wpad), static_cast<int>(C), taps);
      cuda_check(cudaGetLastError(), "launch dw_tap_major");
      cuda_check(cudaDeviceSynchronize(), "dw_tap_major");
      md.dwt = static_cast<const __nv_bfloat16*>(op.wpad);
    }
    op.n_tile = static_cast<int>(best_cc);
    op.cc_rows = best_ro * Q;
    md.cc_rows = static_cast<int32_t>(best_ro);
    md.tx_bytes = static_cast<uint32_t>(best_cc * Wb * Hb * 2);
  }

  // A member's k-block stage (A region + B box) fits a 32 KB narrow-layout slot.
  int ring_narrow_of(const dev::MemberDesc& md, int b_rows) const {
    if (ring_layouts == 0) return 0;
    if (md.cc_rows > 0) return md.tx_bytes <= 32768 ? 1 : 0;  // a staged CUDA-core tile's box
    const bool cols = md.a_mode == dev::kAIm2colNarrow || md.a_mode == dev::kAIm2colFold;
    const int a_bytes = cols ? dev::kABytes : a_box_rows(md.m) * dev::kBK * 2;
    return a_bytes + b_rows * dev::kBK * 2 <= 32768 ? 1 : 0;
  }

  // [rows, cols] bf16 row-major with row stride ld (elements), box kBK x box_rows.
  void tiled_map(CUtensorMap* map, const void* base, int64_t rows, int64_t cols, int64_t ld, int box_rows) {
    if (!aligned16(base)) throw std::invalid_argument("operand base must be 16-byte aligned");
    if ((ld * 2) % 16 != 0) throw std::invalid_argument("operand row stride must be a multiple of 8 elements");
    const cuuint64_t dims[2] = {static_cast<cuuint64_t>(cols), static_cast<cuuint64_t>(rows)};
    const cuuint64_t strides[1] = {static_cast<cuuint64_t>(ld * 2)};
    const cuuint32_t box[2] = {static_cast<cuuint32_t>(dev::kBK), static_cast<cuuint32_t>(box_rows)};
    const cuuint32_t estr[2] = {1, 1};
    const CUresult r = encode_tiled(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides,
                                    box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                    CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) throw CudaError("cuTensorMapEncodeTiled failed (" + std::to_string(int(r)) + ")");
  }

  // NHWC activation as an im2col source (fprop, dilation 1).  Corner arrays
  // are in {W, H} order (CUTLASS convention); all convs routed here are
  // square with symmetric padding, so the order is immaterial.
  // Output [rows, cols] row-major: 32 x 32 store boxes, 64 B swizzle (the
  // epilogue staging layout).
  void store_map(CUtensorMap* map, void* base, int64_t rows, int64_t cols) {
    if (!aligned16(base)) throw std::invalid_argument("register_tenant: output must be 16-byte aligned");
    const cuuint64_t dims[2] = {static_cast<cuuint64_t>(cols), static_cast<cuuint64_t>(rows)};
    const cuuint64_t strides[1] = {static_cast<cuuint64_t>(cols * 2)};
    const cuuint32_t box[2] = {static_cast<cuuint32_t>(dev::kEpiChunk), 32};
    const cuuint32_t estr[2] = {1, 1};
    const CUresult r = encode_tiled(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, base, dims, strides, box, estr,
                                    CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_64B,
                                    CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) throw CudaError("cuTensorMapEncodeTiled(store) failed (" + std::to_string(int(r)) + ")");
  }

  // `pitch` = channels per stored pixel (>= C_in); `box_c` channels per box
  // pixel: 64 (one SW128 row) for the regular mode, 8 (16 B, no swizzle) for
  // the narrow-channel mode.
  void im2col_map(CUtensorMap* map, const void* x, const Conv& c, int batch, int pixels, int64_t pitch = 0,
                  int box_c = dev::kBK, CUtensorMapSwizzle swz = CU_TENSOR_MAP_SWIZZLE_128B) {
    if (!aligned16(x)) throw std::invalid_argument("conv input must be 16-byte aligned");
    if (pitch <= 0) pitch = c.in_channels;
    const cuuint64_t dims[4] = {static_cast<cuuint64_t>(pitch), static_cast<cuuint64_t>(c.image_w),
                                static_cast<cuuint64_t>(c.image_h), static_cast<cuuint64_t>(batch)};
    const cuuint64_t strides[3] = {static_cast<cuuint64_t>(pitch * 2),
                                   static_cast<cuuint64_t>(c.image_w * pitch * 2),
                                   static_cast<cuuint64_t>(c.image_h * c.image_w * pitch * 2)};
    const int lower[2] = {static_cast<int>(-c.padding), static_cast<int>(-c.padding)};
    const int upper[2] = {static_cast<int>(c.padding - (c.kernel_w - 1)), static_cast<int>(c.padding - (c.kernel_h - 1))};
    const cuuint32_t estr[4] = {1, static_cast<cuuint32_t>(c.stride), static_cast<cuuint32_t>(c.stride), 1};
    const CUresult r = encode_im2col(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void*>(x), dims, strides,
                                     lower, upper, static_cast<cuuint32_t>(box_c), static_cast<cuuint32_t>(pixels),
                                     estr, CU_TENSOR_MAP_INTERLEAVE_NONE, swz, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) throw CudaError("cuTensorMapEncodeIm2col failed (" + std::to_string(int(r)) + ")");
    // Driver <= 13.1 mis-encodes im2col maps of tensors under 128 KiB; clear
    // the offending bit exactly as CUTLASS does (copy_traits_sm90_im2col.hpp).
    const int64_t bytes = static_cast<int64_t>(batch) * c.image_h * c.image_w * pitch * 2;
    if (driver_version <= 13010 && bytes < 131072) reinterpret_cast<uint64_t*>(map)[1] &= ~(1ull << 21);
  }

  // Folded input X' [b, H, Q, 32] as an R x 1 im2col source: vertical stride
  // and padding from the conv, horizontal already applied by the fold.
  void fold_map(CUtensorMap* map, const void* xf, const Conv& c, int64_t Q, int batch, int pixels) {
    const cuuint64_t dims[4] = {static_cast<cuuint64_t>(dev::kFoldC), static_cast<cuuint64_t>(Q),
                                static_cast<cuuint64_t>(c.image_h), static_cast<cuuint64_t>(batch)};
    const cuuint64_t strides[3] = {static_cast<cuuint64_t>(dev::kFoldC * 2),
                                   static_cast<cuuint64_t>(Q * dev::kFoldC * 2),
                                   static_cast<cuuint64_t>(c.image_h * Q * dev::kFoldC * 2)};
    const int lower[2] = {0, static_cast<int>(-c.padding)};
    const int upper[2] = {0, static_cast<int>(c.padding - (c.kernel_h - 1))};
    const cuuint32_t estr[4] = {1, 1, static_cast<cuuint32_t>(c.stride), 1};
    const CUresult r = encode_im2col(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void*>(xf), dims, strides,
                                     lower, upper, static_cast<cuuint32_t>(dev::kFoldC),
                                     static_cast<cuuint32_t>(pixels), estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                     CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) throw CudaError("cuTensorMapEncodeIm2col(fold) failed (" + std::to_string(int(r)) + ")");
    const int64_t bytes = static_cast<int64_t>(batch) * c.image_h * Q * dev::kFoldC * 2;
    if (driver_version <= 13010 && bytes < 131072) reinterpret_cast<uint64_t*>(map)[1] &= ~(1ull << 21);
  }

  int register_tenant(const gm_tenant_desc& t) {
    if (!t.layers || t.n_layers == 0) throw std::invalid_argument("register_tenant: tenant has no layers");
    std::vector<int> ops;
    std::vector<Operator> fresh;
    std::vector<dev::MemberDesc> descs;
    std::vector<int> slot_of_new;  // per new descriptor: its operator's index into flat
    for (size_t i = 0; i < t.n_layers; ++i) {
      const gm_layer_desc& L = t.layers[i];
      Operator op;
      dev::MemberDesc md;
      std::memset(&md, 0, sizeof(md));
      std::function<void(CUtensorMap*)> a_tall, r_tall;  // 256-row A / residual maps (tall variant)
      op.kind = L.kind;
      op.x = L.x;
      op.tenant = static_cast<int>(tenant_ops.size());
      op.layer = static_cast<int>(i);
      const bool pool = L.kind == GM_LAYER_MAXPOOL || L.kind == GM_LAYER_AVGPOOL;
      if (!L.x || (!L.w && !pool) || !L.y) throw std::invalid_argument("register_tenant: null operand pointer");
      if (!aligned16(L.y)) throw std::invalid_argument("register_tenant: output must be 16-byte aligned");
      if (L.act < GM_ACT_NONE || L.act > GM_ACT_GELU) throw std::invalid_argument("register_tenant: unknown activation");
      // dataflow: x (and the residual) must lie inside the named earlier layer's output
      auto inside = [&](int j, const void* p, const char* what) {
        if (j < 0) return;
        if (j >= static_cast<int>(i))
          throw std::invalid_argument(std::string("register_tenant: ") + what + " must name an earlier layer");
        const Operator& pr = fresh[j];
        const char* c = static_cast<const char*>(p);
        if (c < pr.y || c >= pr.y + pr.y_bytes)
          throw std::invalid_argument(std::string("register_tenant: ") + what + " does not point into layer " +
                                      std::to_string(j) + "'s output");
      };
      inside(L.src, L.x, "src");
      op.src = L.src < 0 ? -1 : L.src;
      if (L.res) {
        inside(L.res_src, L.res, "res_src");
        op.res_src = L.res_src < 0 ? -1 : L.res_src;
      } else if (L.res_src >= 0) {
        throw std::invalid_argument("register_tenant: res_src without a residual pointer");
      }
      if (L.kind == GM_LAYER_CONV) {
        op.conv = to_conv(L.conv);
        op.batch = L.batch < 1 ? 1 : L.batch;
        op.shape = with_batch(lower_conv(op.conv), op.batch);
        op.n_tile = bn;
        const Conv& c = op.conv;
        const int64_t K = op.shape.k;
        const int64_t ldw = L.ldw > 0 ? L.ldw : K;
        if (ldw < K) throw std::invalid_argument("register_tenant: ldw < R*S*Cin");
        tiled_map(&md.b, L.w, op.shape.n, K, ldw, b_box_rows(op.shape.n, op.n_tile));
        op.b_ptr = L.w;
        op.b_k = K;
        op.b_ld = ldw;
        const int64_t P = (c.image_h + 2 * c.padding - c.kernel_h) / c.stride + 1;
        const int64_t Q = (c.image_w + 2 * c.padding - c.kernel_w) / c.stride + 1;
        const bool pointwise = c.kernel_h == 1 && c.kernel_w == 1 && c.stride == 1 && c.padding == 0;
        if (pointwise && c.in_channels % 8 == 0) {
          md.a_mode = dev::kATiled;  // 1x1 stride-1 conv == GEMM over NHWC rows
          tiled_map(&md.a, L.x, op.shape.m, c.in_channels, c.in_channels, a_box_rows(op.shape.m));
          a_tall = [=, this](CUtensorMap* mp) { tiled_map(mp, L.x, op.shape.m, c.in_channels, c.in_channels, 2 * dev::kBM); };
        } else if (c.in_channels % dev::kBK == 0 && c.kernel_h == c.kernel_w && c.stride <= 8 &&
                   c.padding <= 127 && c.kernel_h - 1 - c.padding <= 128) {
          md.a_mode = dev::kAIm2col;  // implicit GEMM through the TMA im2col unit
          im2col_map(&md.a, L.x, c, op.batch, a_box_rows(op.shape.m));
          a_tall = [=, this](CUtensorMap* mp) { im2col_map(mp, L.x, c, op.batch, 2 * dev::kBM); };
          md.pq = static_cast<int32_t>(P * Q);
          md.q = static_cast<int32_t>(Q);
          md.stride = static_cast<int32_t>(c.stride);
          md.pad = static_cast<int32_t>(c.padding);
          md.s_taps = static_cast<int32_t>(c.kernel_w);
          md.c_blocks = static_cast<int32_t>(c.in_channels / dev::kBK);
        } else if (c.in_channels <= dev::kNarrowC && L.ldx == dev::kNarrowC && c.kernel_h == c.kernel_w &&
                   c.stride <= 8 && c.padding <= 127) {
          // narrow-channel implicit GEMM: the input stores 8 channels per
          // pixel; one 16 B TMA im2col column per filter tap, 8 taps per
          // k-block; weights repacked once to the same (tap, 8-channel) K order
          md.a_mode = dev::kAIm2colNarrow;
          im2col_map(&md.a, L.x, c, op.batch, a_box_rows(op.shape.m), dev::kNarrowC, dev::kNarrowC,
                     CU_TENSOR_MAP_SWIZZLE_NONE);
          const int taps = static_cast<int>(c.kernel_h * c.kernel_w);
          md.pq = static_cast<int32_t>(P * Q);
          md.q = static_cast<int32_t>(Q);
          md.stride = static_cast<int32_t>(c.stride);
          md.pad = static_cast<int32_t>(c.padding);
          md.s_taps = static_cast<int32_t>(c.kernel_w);
          md.taps = taps;
          md.images = op.batch;
          op.kernel_k = static_cast<int64_t>(taps) * dev::kNarrowC;
          const size_t wbytes = static_cast<size_t>(op.shape.n * op.kernel_k * 2);
          cuda_check(cudaMalloc(&op.wpad, wbytes), "cudaMalloc(narrow weights)");
          dev::pad_narrow_weights<<<static_cast<int>(std::min<int64_t>((op.shape.n * op.kernel_k + 255) / 256, 4096)),
                                    256>>>(static_cast<const __nv_bfloat16*>(L.w), ldw,
                                           static_cast<__nv_bfloat16*>(op.wpad), static_cast<int>(op.shape.n), taps,
                                           static_cast<int>(c.in_channels));
          cuda_check(cudaGetLastError(), "launch pad_narrow_weights");
          cuda_check(cudaDeviceSynchronize(), "pad_narrow_weights");
          tiled_map(&md.b, op.wpad, op.shape.n, op.kernel_k, op.kernel_k, b_box_rows(op.shape.n, op.n_tile));
          op.b_ptr = op.wpad;
          op.b_k = op.kernel_k;
          op.b_ld = op.kernel_k;
        } else if (row_fold && c.kernel_w * c.in_channels <= dev::kFoldC &&
                   (L.ldx <= 0 || L.ldx == c.in_channels) && c.stride <= 8 && c.padding <= 127 &&
                   c.kernel_h - 1 - c.padding <= 128) {
          // row-folded implicit GEMM: a pre-pass folds each output column's
          // horizontal window into a 32-channel pixel; R x 1 TMA im2col over it
          md.a_mode = dev::kAIm2colFold;
          op.prepass = op.fold = true;
          const size_t xbytes = static_cast<size_t>(op.batch * c.image_h * Q * dev::kFoldC * 2);
          cuda_check(cudaMalloc(&op.scratch, xbytes), "cudaMalloc(folded input)");
          fold_map(&md.a, op.scratch, c, Q, op.batch, a_box_rows(op.shape.m));
          md.pq = static_cast<int32_t>(P * Q);
          md.q = static_cast<int32_t>(Q);
          md.stride = static_cast<int32_t>(c.stride);
          md.pad = static_cast<int32_t>(c.padding);
          md.taps = static_cast<int32_t>(c.kernel_h);
          const int rpad = static_cast<int>((c.kernel_h + dev::kFoldTaps - 1) / dev::kFoldTaps * dev::kFoldTaps);
          op.kernel_k = static_cast<int64_t>(rpad) * dev::kFoldC;
          cuda_check(cudaMalloc(&op.wpad, static_cast<size_t>(op.shape.n * op.kernel_k * 2)),
                     "cudaMalloc(folded weights)");
          dev::fold_weights<<<static_cast<int>(std::min<int64_t>((op.shape.n * op.kernel_k + 255) / 256, 4096)), 256>>>(
              static_cast<const __nv_bfloat16*>(L.w), ldw, static_cast<__nv_bfloat16*>(op.wpad),
              static_cast<int>(op.shape.n), static_cast<int>(c.kernel_h),
              static_cast<int>(c.kernel_w * c.in_channels), rpad);
          cuda_check(cudaGetLastError(), "launch fold_weights");
          cuda_check(cudaDeviceSynchronize(), "fold_weights");
          tiled_map(&md.b, op.wpad, op.shape.n, op.kernel_k, op.kernel_k, b_box_rows(op.shape.n, op.n_tile));
          op.b_ptr = op.wpad;
          op.b_k = op.kernel_k;
          op.b_ld = op.kernel_k;
        } else {
          md.a_mode = dev::kATiled;  // explicit im2col pre-pass, then GEMM
          op.prepass = true;
          op.ldk = (K + 7) / 8 * 8;
          cuda_check(cudaMalloc(&op.scratch, static_cast<size_t>(op.shape.m * op.ldk * 2)), "cudaMalloc(im2col)");
          tiled_map(&md.a, op.scratch, op.shape.m, K, op.ldk, a_box_rows(op.shape.m));
          a_tall = [=, this](CUtensorMap* mp) { tiled_map(mp, op.scratch, op.shape.m, K, op.ldk, 2 * dev::kBM); };
        }
      } else if (pool) {
        // max / average pool: CUDA-core tile type; planned as a K = R*S GEMM
        // like a depthwise conv (the reference's model of per-channel ops,
        // proj/src/workload.cpp:66)
        op.conv = to_conv(L.conv);
        op.batch = L.batch < 1 ? 1 : L.batch;
        const Conv& c = op.conv;
        if (c.in_channels != c.out_channels) throw std::invalid_argument("register_tenant: pool needs Cin == Cout");
        if (c.in_channels % 8 != 0) throw std::invalid_argument("register_tenant: pool channels must be a multiple of 8");
        if (!aligned16(L.x)) throw std::invalid_argument("pool input must be 16-byte aligned");
        if (L.res) throw std::invalid_argument("register_tenant: pools take no residual");
        const int64_t P = (c.image_h + 2 * c.padding - c.kernel_h) / c.stride + 1;
        const int64_t Q = (c.image_w + 2 * c.padding - c.kernel_w) / c.stride + 1;
        if (P < 1 || Q < 1 || c.kernel_h < 1 || c.kernel_w < 1 || c.stride < 1 || c.padding < 0)
          throw std::invalid_argument("conv output dims must be positive");
        op.shape = Shape{op.batch * P * Q, c.out_channels, c.kernel_h * c.kernel_w};
        op.n_tile = dev::kDwTileC;
        md.a_mode = L.kind == GM_LAYER_MAXPOOL ? dev::kMaxPool : dev::kAvgPool;
        md.dx = static_cast<const __nv_bfloat16*>(L.x);
        md.dy = static_cast<__nv_bfloat16*>(L.y);
        md.h_in = static_cast<int32_t>(c.image_h);
        md.w_in = static_cast<int32_t>(c.image_w);
        md.ch = static_cast<int32_t>(c.in_channels);
        md.r_taps = static_cast<int32_t>(c.kernel_h * c.kernel_w);
        md.s_taps = static_cast<int32_t>(c.kernel_w);
        md.stride = static_cast<int32_t>(c.stride);
        md.pad = static_cast<int32_t>(c.padding);
        md.pq = static_cast<int32_t>(P * Q);
        md.q = static_cast<int32_t>(Q);
        md.images = op.batch;
      } else if (L.kind == GM_LAYER_DWCONV) {
        // depthwise conv: the reference models it as a K = R*S GEMM
        // (proj/src/workload.cpp:66); executed as the super-kernel's CUDA-core
        // tile type (one filter per channel, no tensor-core path)
        op.conv = to_conv(L.conv);
        op.batch = L.batch < 1 ? 1 : L.batch;
        const Conv& c = op.conv;
        if (c.in_channels != c.out_channels) throw std::invalid_argument("register_tenant: depthwise needs Cin == Cout");
        if (c.kernel_h * c.kernel_w > dev::kDwMaxTaps)
          throw std::invalid_argument("register_tenant: depthwise filter larger than 3x3");
        if (c.in_channels % 4 != 0) throw std::invalid_argument("register_tenant: depthwise channels must be a multiple of 4");
        const int64_t taps = c.kernel_h * c.kernel_w;
        const int64_t ldw = L.ldw > 0 ? L.ldw : taps;
        if (ldw < taps) throw std::invalid_argument("register_tenant: ldw < R*S");
        if (!aligned16(L.x)) throw std::invalid_argument("conv input must be 16-byte aligned");
        const int64_t P = (c.image_h + 2 * c.padding - c.kernel_h) / c.stride + 1;
        const int64_t Q = (c.image_w + 2 * c.padding - c.kernel_w) / c.stride + 1;
        if (P < 1 || Q < 1) throw std::invalid_argument("conv output dims must be positive");
        op.shape = Shape{op.batch * P * Q, c.out_channels, taps};
        op.n_tile = dev::kDwTileC;
        md.a_mode = dev::kDepthwise;
        md.dx = static_cast<const __nv_bfloat16*>(L.x);
        md.dw = static_cast<const __nv_bfloat16*>(L.w);
        md.dy = static_cast<__nv_bfloat16*>(L.y);
        md.h_in = static_cast<int32_t>(c.image_h);
        md.w_in = static_cast<int32_t>(c.image_w);
        md.ch = static_cast<int32_t>(c.in_channels);
        md.r_taps = static_cast<int32_t>(taps);
        md.ldw = static_cast<int32_t>(ldw);
        md.s_taps = static_cast<int32_t>(c.kernel_w);
        md.stride = static_cast<int32_t>(c.stride);
        md.pad = static_cast<int32_t>(c.padding);
        md.pq = static_cast<int32_t>(P * Q);
        md.q = static_cast<int32_t>(Q);
        md.images = op.batch;
      } else if (L.kind == GM_LAYER_GEMM) {
        op.shape = to_shape(L.gemm);
        op.n_tile = bn;
        if (!op.shape.valid()) throw std::invalid_argument("register_tenant: invalid GEMM shape");
        const int64_t ldx = L.ldx > 0 ? L.ldx : op.shape.k;
        const int64_t ldw = L.ldw > 0 ? L.ldw : op.shape.k;
        md.a_mode = dev::kATiled;
        tiled_map(&md.a, L.x, op.shape.m, op.shape.k, ldx, a_box_rows(op.shape.m));
        a_tall = [=, this](CUtensorMap* mp) { tiled_map(mp, L.x, op.shape.m, op.shape.k, ldx, 2 * dev::kBM); };
        tiled_map(&md.b, L.w, op.shape.n, op.shape.k, ldw, b_box_rows(op.shape.n, op.n_tile));
        op.b_ptr = L.w;
        op.b_k = op.shape.k;
        op.b_ld = ldw;
      } else {
        throw std::invalid_argument("register_tenant: unknown layer kind");
      }
      if (op.shape.n % 8 != 0) throw std::invalid_argument("register_tenant: output channels must be a multiple of 8");
      if (op.shape.m > int64_t(0xFFFF) * (cuda_core_kind(op.kind) ? dev::kDwTileM : dev::kBM) ||
          op.shape.m > INT32_MAX)
        throw std::invalid_argument("register_tenant: M too large for the tile table");
      store_map(&md.c, L.y, op.shape.m, op.shape.n);
      md.m = static_cast<int32_t>(op.shape.m);
      md.n = static_cast<int32_t>(op.shape.n);
      if (op.kernel_k == 0) op.kernel_k = op.shape.k;
      md.k_blocks = static_cast<int32_t>((op.kernel_k + dev::kBK - 1) / dev::kBK);
      md.idesc = make_idesc(b_box_rows(op.shape.n, op.n_tile));
      // one k-block moves an A box (rows x 64 channels, or 8 tap columns of
      // rows x 8 channels: the same bytes) plus a B box
      md.tx_bytes = static_cast<uint32_t>((a_box_rows(op.shape.m) + b_box_rows(op.shape.n, op.n_tile)) * dev::kBK * 2);
      md.act = L.act;
      if (L.res) {
        if (cuda_core_kind(op.kind)) throw std::invalid_argument("register_tenant: residual add needs a conv / GEMM");
        const int64_t ldr = L.ldr > 0 ? L.ldr : op.shape.n;
        if (ldr < op.shape.n || ldr % 8 != 0 || !aligned16(L.res))
          throw std::invalid_argument("register_tenant: residual rows must be 16-byte aligned (ldr % 8 == 0, ldr >= N)");
        // the add runs on the tensor core as extra k-blocks (A = residual
        // columns, B = identity): the member's A operand must be the SW128
        // K-major layout the residual box lands in
        if (md.a_mode != dev::kATiled && md.a_mode != dev::kAIm2col)
          throw std::invalid_argument("register_tenant: residual add needs a tiled or im2col A operand");
        md.res = static_cast<const __nv_bfloat16*>(L.res);
        md.ldr = static_cast<int32_t>(ldr);
        tiled_map(&md.r, L.res, op.shape.m, op.shape.n, ldr, a_box_rows(op.shape.m));
        r_tall = [=, this](CUtensorMap* mp) { tiled_map(mp, L.res, op.shape.m, op.shape.n, ldr, 2 * dev::kBM); };
        tiled_map(&md.id, ident, dev::kIdentN, dev::kIdentN, dev::kIdentN, b_box_rows(op.shape.n, op.n_tile));
      }
      op.y = static_cast<const char*>(L.y);
      op.y_bytes = op.shape.m * op.shape.n * 2;
      op.x_pitch = L.ldx > 0 ? L.ldx : (L.kind == GM_LAYER_GEMM ? op.shape.k : op.conv.in_channels);
      {
        const bool gemm = L.kind == GM_LAYER_GEMM;
        const int64_t rows = gemm ? op.shape.m : op.batch * op.conv.image_h * op.conv.image_w;
        op.x_bytes = ((rows - 1) * op.x_pitch + (gemm ? op.shape.k : op.conv.in_channels)) * 2;
      }
      if (L.res) {
        op.res = static_cast<const char*>(L.res);
        op.ldr = L.ldr > 0 ? L.ldr : op.shape.n;
      }
      if (cuda_core_kind(op.kind)) stage_cuda_core(op, md, L.x);
      md.n_tile = op.n_tile;
      md.ring_narrow = ring_narrow_of(md, b_box_rows(op.shape.n, op.n_tile));
      op.slot = static_cast<int>(host_desc.size() + descs.size());
      const int f_index = static_cast<int>(flat.size() + fresh.size());
      descs.push_back(md);
      slot_of_new.push_back(f_index);
      // narrower-N variants (same operands, smaller B box / UMMA N)
      if (!cuda_core_kind(op.kind) && op.b_ptr) {
        int v = 0;
        for (int w = bn / 2; w >= 64 && v < 2; w /= 2) {
          if (op.shape.n <= w) break;
          dev::MemberDesc md2 = md;
          tiled_map(&md2.b, op.b_ptr, op.shape.n, op.b_k, op.b_ld, b_box_rows(op.shape.n, w));
          md2.idesc = make_idesc(b_box_rows(op.shape.n, w));
          if (md2.res) tiled_map(&md2.id, ident, dev::kIdentN, dev::kIdentN, dev::kIdentN, b_box_rows(op.shape.n, w));
          md2.tx_bytes = static_cast<uint32_t>((a_box_rows(op.shape.m) + b_box_rows(op.shape.n, w)) * dev::kBK * 2);
          md2.n_tile = w;
          md2.ring_narrow = ring_narrow_of(md2, b_box_rows(op.shape.n, w));
          op.narrow_slot[v] = static_cast<int>(host_desc.size() + descs.size());
          op.narrow_w[v] = w;
          descs.push_back(md2);
          slot_of_new.push_back(f_index);
          ++v;
        }
      }
      // tall variant: two 128-row halves per tile sharing the B box
      // (needs the 256-column kernel: the second half's accumulator sits at
      // column 128 of a BN-column buffer, and the stage holds 2 A boxes + a
      // <= 128-row B box, which only the 48 KB BN = 256 ring slot fits)
      if (bn == 256 && !cuda_core_kind(op.kind) && op.b_ptr && op.shape.m >= 2 * dev::kBM && op.shape.n <= 128 &&
          (md.a_mode == dev::kATiled || md.a_mode == dev::kAIm2col || md.a_mode == dev::kAIm2colFold) &&
          a_box_rows(op.shape.m) == dev::kBM) {
        if (!dev::Cfg<256>::kTallFits || b_box_rows(op.shape.n, 128) > 128)
          throw std::logic_error("tall variant does not fit the ring slot / accumulator");
        dev::MemberDesc md3 = md;
        md3.tall = 1;
        // tiled / im2col A (and the residual): one 256-row box per k-block
        // (SW128 rows 128..255 land 16 KB on, where the second half's UMMA
        // reads them): one TMA issue instead of two on the producer thread.
        // The folded stem keeps two boxes per filter-row column.
        if (md.a_mode != dev::kAIm2colFold) {
          if (!a_tall) throw std::logic_error("tall variant: no 256-row A map for this operand mode");
          a_tall(&md3.a);
          if (md.res) r_tall(&md3.r);
        }
        md3.ring_narrow = 0;  // two A boxes: a wide-layout stage
        md3.n_tile = 128;  // the second half's accumulator starts at column 128 of the tile's buffer
        md3.tx_bytes = static_cast<uint32_t>((2 * dev::kBM + b_box_rows(op.shape.n, op.n_tile)) * dev::kBK * 2);
        op.tall_slot = static_cast<int>(host_desc.size() + descs.size());
        descs.push_back(md3);
        slot_of_new.push_back(f_index);
      }
      if (host_desc.size() + descs.size() > 0x10000)
        throw std::invalid_argument("register_tenant: too many registered operators");
      fresh.push_back(op);
    }
    // Commit: grow the device descriptor array and upload.
    const size_t need_n = host_desc.size() + descs.size();
    if (need_n > d_cap) {
      size_t cap = std::max<size_t>(64, d_cap * 2);
      while (cap < need_n) cap *= 2;
      dev::MemberDesc* nd = nullptr;
      cuda_check(cudaMalloc(&nd, cap * sizeof(dev::MemberDesc)), "cudaMalloc(descriptors)");
      // the old array stays alive (freed with the runtime): launch programs
      // captured before this registration keep reading their descriptors
      if (d_desc) retired_desc.push_back(d_desc);
      d_desc = nd;
      d_cap = cap;
      host_desc.insert(host_desc.end(), descs.begin(), descs.end());
      cuda_check(cudaMemcpy(d_desc, host_desc.data(), host_desc.size() * sizeof(dev::MemberDesc),
                            cudaMemcpyHostToDevice),
                 "upload descriptors");
    } else {
      const size_t off = host_desc.size();
      host_desc.insert(host_desc.end(), descs.begin(), descs.end());
      cuda_check(cudaMemcpy(d_desc + off, descs.data(), descs.size() * sizeof(dev::MemberDesc), cudaMemcpyHostToDevice),
                 "upload descriptors");
    }
    for (Operator& op : fresh) {
      ops.push_back(static_cast<int>(flat.size()));
      flat.push_back(op);
    }
    slot_op.insert(slot_op.end(), slot_of_new.begin(), slot_of_new.end());
    tenant_ops.push_back(std::move(ops));
    tenant_slo.push_back(t.slo_latency > 0 ? t.slo_latency : 0.1);
    tenant_layers.emplace_back(t.layers, t.layers + t.n_layers);
    tenant_conc.push_back(t.concurrency);
    return static_cast<int>(tenant_ops.size() - 1);
  }

  const Operator& op_of(int tenant, int layer) const {
    if (tenant < 0 || tenant >= static_cast<int>(tenant_ops.size()))
      throw std::invalid_argument("unknown tenant " + std::to_string(tenant));
    const auto& ops = tenant_ops[tenant];
    if (layer < 0 || layer >= static_cast<int>(ops.size()))
      throw std::invalid_argument("unknown layer " + std::to_string(layer) + " of tenant " + std::to_string(tenant));
    return flat[ops[layer]];
  }

  int flat_index(int tenant, int layer) const {
    op_of(tenant, layer);
    return tenant_ops[tenant][layer];
  }

  // (descriptor slot, N tile) of operator f inside a plan whose members have
  // plan_tiles full-width tiles: when the plan leaves most SMs idle, a member
  // with few tiles uses a narrower-N variant (256 -> 128 -> 64) until it has
  // narrow_min_tiles tiles -- more SMs share the plan's long K loops.
  std::pair<int, int> variant(int f, int64_t plan_tiles, int64_t concurrent = 0) const {
    const Operator& op = flat[f];
    int slot = op.slot, w = op.n_tile;
    // throughput-bound (many tiles of this shape run at once): tall tiles
    if (tall_tiles && op.tall_slot >= 0 && concurrent >= (tall_min_tiles > 0 ? tall_min_tiles : 2 * sms))
      return {op.tall_slot, w};
    if (narrow_min_tiles <= 0 || 2 * plan_tiles > sms) return {slot, w};  // the plan fills half the SMs already
    const int64_t mt = (op.shape.m + dev::kBM - 1) / dev::kBM;
    for (int i = 0; i < 2 && op.narrow_slot[i] >= 0; ++i) {
      if (mt * ((op.shape.n + w - 1) / w) >= narrow_min_tiles) break;
      slot = op.narrow_slot[i];
      w = op.narrow_w[i];
    }
    return {slot, w};
  }
  bool is_tall(int slot) const { return host_desc[slot].tall != 0; }
  int64_t full_tiles(int f) const {
    const Operator& op = flat[f];
    return ((op.shape.m + dev::kBM - 1) / dev::kBM) * ((op.shape.n + op.n_tile - 1) / op.n_tile);
  }

  // Device tile table for a member list (cached: the B200 meaning of a
  // SuperKernelCache hit is that descriptors and table are already resident).
  Prepared& prepare(const std::vector<int>& members) {
    std::string key;
    key.reserve(members.size() * 6);
    for (int f : members) {
      key += std::to_string(f);
      key += ',';
    }
    auto it = prepared.find(key);
    if (it != prepared.end()) return it->second;
    Prepared p;
    std::vector<dev::TileEntry> table;
    int64_t plan_tiles = 0;
    for (int f : members) plan_tiles += full_tiles(f);
    for (int f : members) {
      const Operator& op = flat[f];
      const auto [slot, w] = variant(f, plan_tiles, plan_tiles);
      const int64_t tm = tile_rows_of(op, is_tall(slot));
      const int64_t mt = (op.shape.m + tm - 1) / tm;
      const int64_t nt = (op.shape.n + w - 1) / w;
      for (int64_t a = 0; a < mt; ++a)
        for (int64_t b = 0; b < nt; ++b)
          table.push_back(dev::TileEntry{static_cast<uint16_t>(slot), 0, static_cast<uint16_t>(a),
                                         static_cast<uint16_t>(b), -1, -1, 0, 0, -1, -1, 0, 0});
      if (op.prepass) p.prepass_ops.push_back(f);
    }
    p.n_tiles = static_cast<int>(table.size());
    cuda_check(cudaMalloc(&p.tiles, std::max<size_t>(1, table.size()) * sizeof(dev::TileEntry)), "cudaMalloc(tiles)");
    cuda_check(cudaMemcpy(p.tiles, table.data(), table.size() * sizeof(dev::TileEntry), cudaMemcpyHostToDevice),
               "upload tile table");
    return prepared.emplace(key, std::move(p)).first->second;
  }

  // Rows [lo, hi] of producer `pr`'s output that consumer `c`'s output rows
  // [r0, r1) read: through its input x (a view into pr's y: a windowed op's
  // receptive field, or a GEMM's row slice) or, with `residual`, through its
  // residual (the same rows).  Conservative for windowed ops: whole input
  // image rows from the first output pixel's window to the last one's.
  std::pair<int64_t, int64_t> producer_rows(const Operator& c, const Operator& pr, bool residual, int64_t r0,
                                            int64_t r1) const {
    const int64_t np = pr.shape.n;
    int64_t lo, hi;
    if (residual) {
      const int64_t off = (c.res - pr.y) / 2;
      lo = (off + r0 * c.ldr) / np;
      hi = (off + (r1 - 1) * c.ldr + c.shape.n - 1) / np;
    } else if (c.kind == GM_LAYER_GEMM) {
      const int64_t off = (static_cast<const char*>(c.x) - pr.y) / 2;
      lo = (off + r0 * c.x_pitch) / np;
      hi = (off + (r1 - 1) * c.x_pitch + c.shape.k - 1) / np;
    } else {
      const Conv& v = c.conv;
      const int64_t P = (v.image_h + 2 * v.padding - v.kernel_h) / v.stride + 1;
      const int64_t Q = (v.image_w + 2 * v.padding - v.kernel_w) / v.stride + 1;
      auto pixel_row = [&](int64_t m, bool last) {
        const int64_t b = m / (P * Q), p = (m % (P * Q)) / Q;
        const int64_t ih = last ? std::min(v.image_h - 1, p * v.stride - v.padding + v.kernel_h - 1)
                                : std::max<int64_t>(0, p * v.stride - v.padding);
        return (b * v.image_h + ih) * v.image_w + (last ? v.image_w - 1 : 0);
      };
      const int64_t off = (static_cast<const char*>(c.x) - pr.y) / 2;
      lo = (off + pixel_row(r0, false) * c.x_pitch) / np;
      hi = (off + pixel_row(r1 - 1, true) * c.x_pitch + c.x_pitch - 1) / np;
    }
    return {std::max<int64_t>(0, lo), std::min(pr.shape.m - 1, hi)};
  }

  // Round program: every plan of a round, in plan order, as ONE persistent
  // launch.  Member instances get completion counters; a member depends on the
  // same tenant's previous layer when that layer ran earlier in the round.
  Prepared& prepare_round(const std::vector<std::vector<int>>& plans, bool gated = false) {
    std::lock_guard<std::recursive_mutex> lock(rounds_mu);  // gm_serve prepares member sets on a worker thread
    std::string key = gated ? "G" : "R";
    for (const auto& pl : plans) {
      for (int f : pl) {
        key += std::to_string(f);
        key += ',';
      }
      key += '|';
    }
    auto it = rounds.find(key);
    if (it != rounds.end()) return it->second;
    Prepared p;
    std::vector<dev::TileEntry> table;
    std::vector<uint32_t> targets;
    // flat op -> its instance in this round: counters [base, base + mt), one
    // per output row block of `rows` rows
    struct Instance {
      int base;
      int64_t rows, mt;
    };
    std::unordered_map<int, Instance> last_instance;
    int n_ws = 0;
    // Concurrency estimate per shape: tenants run their chains in step, so
    // all members of a shape across the round's plans are in flight together.
    std::map<Shape, int64_t> shape_tiles;
    for (const auto& pl : plans)
      for (int f : pl) shape_tiles[flat[f].shape] += full_tiles(f);
    for (const auto& pl : plans) {
      int64_t plan_tiles = 0;
      for (int f : pl) plan_tiles += full_tiles(f);
      for (int f : pl) {
        const Operator& op = flat[f];
        auto [slot, w] = variant(f, plan_tiles, shape_tiles[op.shape]);
        int skinny_splits = 1;
        if (skinny_min_mb > 0 && op.kind == GM_LAYER_GEMM && op.shape.m <= 64 &&
            op.shape.n * op.shape.k * 2 >= skinny_min_mb * (int64_t{1} << 20)) {
          const dev::MemberDesc& hd = host_desc[op.slot];
          const int64_t conc = std::max<int64_t>(1, shape_tiles[op.shape]);  // full-width tiles of the shape in the round
          const int64_t sp = std::min<int64_t>({hd.k_blocks / split_min_kb, sms / conc, skinny_max_splits});
          if (hd.a_mode == dev::kATiled && sp >= 2) {
            slot = op.slot;
            w = op.n_tile;
            skinny_splits = static_cast<int>(sp);
          }
        }
        // Wide split (option): a long-K member that narrowing took below 128
        // columns keeps 128-column tiles and splits its K loop over as many
        // tiles as the narrow variant had -- a narrow tile's k-block costs
        // about what a 128-column one does (MMA / TMA issue bound), so each
        // split runs a fraction of the K loop at the same per-k-block cost.
        int wide_splits = 1;
        if (split_wide_kb > 0 && skinny_splits == 1 && !is_tall(slot) && w < 128 &&
            (op.shape.k + dev::kBK - 1) / dev::kBK >= split_wide_kb) {
          int ws_slot = -1, ww = 0;
          if (op.n_tile == 128) {
            ws_slot = op.slot;
            ww = 128;
          } else {
            for (int i = 0; i < 2; ++i)
              if (op.narrow_slot[i] >= 0 && op.narrow_w[i] == 128) {
                ws_slot = op.narrow_slot[i];
                ww = 128;
              }
          }
          if (ws_slot >= 0) {
            const int64_t mt0 = (op.shape.m + dev::kBM - 1) / dev::kBM;
            const int64_t target = mt0 * ((op.shape.n + w - 1) / w);
            const int64_t wide = mt0 * ((op.shape.n + ww - 1) / ww);
            const int64_t sp = std::min<int64_t>({target / wide, max_splits,
                                                  host_desc[ws_slot].k_blocks / std::max<int64_t>(1, split_min_kb)});
            if (sp >= 2) {
              slot = ws_slot;
              w = ww;
              wide_splits = static_cast<int>(sp);
            }
          }
        }
        const bool tall = is_tall(slot);
        // Dependencies.  Dataflow layers wait on the producer row blocks
        // their rows read (input and residual); a layer without a producer in
        // the round but with an earlier layer in it (an operator list without
        // dataflow) waits on that whole layer, keeping the tenant's layer order
        // (sim.cpp:482-488); the first layer of a gated (e2e) round waits on
        // the tenant's input gate (target 1), opened after its H2D copy.
        const Instance* src_inst = nullptr;
        const Instance* res_inst = nullptr;
        const Operator* src_op = nullptr;
        const Operator* res_op = nullptr;
        const Instance* chain = nullptr;
        int gate = -1;
        if (op.src >= 0) {
          auto it2 = last_instance.find(tenant_ops[op.tenant][op.src]);
          if (it2 != last_instance.end()) {
            src_inst = &it2->second;
            src_op = &flat[it2->first];
          }
        } else if (op.layer > 0) {
          auto it2 = last_instance.find(tenant_ops[op.tenant][op.layer - 1]);
          if (it2 != last_instance.end()) chain = &it2->second;
        } else if (gated) {
          gate = static_cast<int>(targets.size());
          targets.push_back(1);
          p.gates.emplace_back(op.tenant, gate);
        }
        if (op.res_src >= 0) {
          auto it2 = last_instance.find(tenant_ops[op.tenant][op.res_src]);
          if (it2 != last_instance.end()) {
            res_inst = &it2->second;
            res_op = &flat[it2->first];
          }
        }
        const int64_t tm = tile_rows_of(op, tall);
        const int64_t mt = (op.shape.m + tm - 1) / tm;
        const int64_t nt = (op.shape.n + w - 1) / w;
        // this instance's counters come after any gate counter pushed above
        // (a tile never publishes to what it waits on)
        const int inst = static_cast<int>(targets.size());
        auto deps_of = [&](int64_t a, bool residual) -> std::pair<int32_t, uint16_t> {
          const Instance* in = residual ? res_inst : src_inst;
          if (!residual && !in) {
            if (chain) return {chain->base, static_cast<uint16_t>(chain->mt)};
            if (gate >= 0) return {gate, 1};
            return {-1, 0};
          }
          if (!in) return {-1, 0};
          const int64_t r0 = a * tm, r1 = std::min(op.shape.m, r0 + tm);
          const auto [lo, hi] = producer_rows(op, residual ? *res_op : *src_op, residual, r0, r1);
          const int64_t first = lo / in->rows, last = hi / in->rows;
          if (last - first + 1 > 0xFFFF) throw std::logic_error("round program: dependency range too long");
          return {static_cast<int32_t>(in->base + first), static_cast<uint16_t>(last - first + 1)};
        };
        const int kb = static_cast<int>((op.shape.k + dev::kBK - 1) / dev::kBK);
        // Split-K when the plan cannot fill the SMs and the K loop is long:
        // about two waves of tiles, at least 4 k-blocks per split.
        int splits = 1;
        if (skinny_splits > 1) {
          const int kbw = host_desc[slot].k_blocks;
          const int chunk = (kbw + skinny_splits - 1) / skinny_splits;
          splits = (kbw + chunk - 1) / chunk;
        } else if (wide_splits > 1) {
          const int kbw = host_desc[slot].k_blocks;
          const int chunk = (kbw + wide_splits - 1) / wide_splits;
          splits = (kbw + chunk - 1) / chunk;
        } else if (split_k && !tall && plan_tiles < sms && kb >= 2 * split_min_kb) {
          splits = static_cast<int>(
              std::min<int64_t>({kb / split_min_kb, (sms + plan_tiles - 1) / plan_tiles, max_splits}));
          const int chunk = (kb + splits - 1) / splits;
          splits = (kb + chunk - 1) / chunk;
        }
        // one counter per row block, nt tiles per block: a GEMM tile's
        // warpgroup publishes once (4 arrivals, one per epilogue warp, for a
        // split tile: each lane quarter's finisher is picked separately), a
        // register-path CUDA-core tile 8 (all eight warps compute it), a
        // staged one 1 (its warpgroup publishes once)
        const int per_tile = !cuda_core_kind(op.kind) ? (splits > 1 ? 4 : 1) : op.cc_rows > 0 ? 1 : 8;
        for (int64_t a = 0; a < mt; ++a) targets.push_back(static_cast<uint32_t>(nt * per_tile));
        for (int64_t a = 0; a < mt; ++a) {
          const auto [dep, dep_n] = deps_of(a, false);
          const auto [rdep, rdep_n] = deps_of(a, true);
          const int32_t done = inst + static_cast<int32_t>(a);
          if ((dep >= 0 && done >= dep && done < dep + dep_n) || (rdep >= 0 && done >= rdep && done < rdep + rdep_n))
            throw std::logic_error("round program: a tile waits on its own counter");
          for (int64_t b = 0; b < nt; ++b) {
            if (splits == 1) {
              table.push_back(dev::TileEntry{static_cast<uint16_t>(slot), 1, static_cast<uint16_t>(a),
                                             static_cast<uint16_t>(b), done, dep, 0, 0, -1, rdep, dep_n, rdep_n});
              continue;
            }
            const int kbt = host_desc[slot].k_blocks;  // the kernel's K loop (padded channels included)
            const int chunk = (kbt + splits - 1) / splits;
            for (int s = 0; s < splits; ++s)
              table.push_back(dev::TileEntry{static_cast<uint16_t>(slot), static_cast<uint16_t>(splits),
                                             static_cast<uint16_t>(a), static_cast<uint16_t>(b), done, dep,
                                             static_cast<uint16_t>(s * chunk),
                                             static_cast<uint16_t>(std::min(kbt, (s + 1) * chunk)), n_ws, rdep,
                                             dep_n, rdep_n});
            ++n_ws;
          }
        }
        last_instance[f] = Instance{inst, tm, mt};
        if (op.prepass && src_inst)
          throw std::invalid_argument("round program: operator " + std::to_string(op.layer) + " of tenant " +
                                      std::to_string(op.tenant) +
                                      " needs a pre-pass over an input produced inside the round");
        if (op.prepass) (gated && op.layer == 0 ? p.gated_prepass : p.prepass_ops).push_back(f);
      }
      p.tile_plan.resize(table.size(), static_cast<uint16_t>(&pl - plans.data()));
    }
    // Critical-path order (option): tiles sorted by their tenant's remaining
    // work from this layer on (FLOPs of the layer and every later layer),
    // longest first.  Remaining work strictly decreases along a chain, so the
    // order stays topological; with heterogeneous tenants the longest chain's
    // tiles reach the SMs first instead of following the virtual-clock plan.
    // auto (-1): progress order.  Round 1 kept the virtual-clock plan order
    // for mixed models; with row-block dependencies and staged CUDA-core
    // tiles the progress order is ahead there too (C3 mix b4 1046 -> 979 us,
    // b8 1537 -> 1506 us; homogeneous rounds +5-9% as before).
    const int order = critical_order < 0 ? 2 : critical_order;
    if (order && !table.empty()) {
      // mode 1: remaining FLOPs (longest chain first); mode 2: chain progress
      // (fraction of the tenant's FLOPs before this layer, ascending), which
      // keeps heterogeneous chains advancing together
      std::vector<double> tail(flat.size(), 0.0);
      for (const auto& ops : tenant_ops) {
        double acc = 0;
        for (auto it2 = ops.rbegin(); it2 != ops.rend(); ++it2) {
          const Shape& sh = flat[*it2].shape;
          acc += 2.0 * static_cast<double>(sh.m) * static_cast<double>(sh.n) * static_cast<double>(sh.k);
          tail[*it2] = acc;
        }
        if (order == 2)
          for (int f2 : ops) tail[f2] = tail[f2] / acc;  // 1 - progress: descending == progress ascending
      }
      std::vector<size_t> idx(table.size());
      for (size_t i = 0; i < idx.size(); ++i) idx[i] = i;
      std::stable_sort(idx.begin(), idx.end(), [&](size_t a, size_t b) {
        return tail[slot_op[table[a].member]] > tail[slot_op[table[b].member]];
      });
      std::vector<dev::TileEntry> sorted(table.size());
      std::vector<uint16_t> sorted_plan(table.size());
      for (size_t i = 0; i < idx.size(); ++i) {
        sorted[i] = table[idx[i]];
        sorted_plan[i] = p.tile_plan[idx[i]];
      }
      table.swap(sorted);
      p.tile_plan.swap(sorted_plan);
    }
    // Dynamic schedule: one work queue per tenant, its tiles in plan order.
    std::vector<int32_t> qbeg, qlen;
    if (dynamic_schedule && !table.empty()) {
      std::vector<size_t> idx(table.size());
      for (size_t i = 0; i < idx.size(); ++i) idx[i] = i;
      auto tenant_of = [&](size_t i) { return flat[slot_op[table[i].member]].tenant; };
      std::stable_sort(idx.begin(), idx.end(), [&](size_t a, size_t b) { return tenant_of(a) < tenant_of(b); });
      std::vector<dev::TileEntry> sorted(table.size());
      std::vector<uint16_t> sorted_plan(table.size());
      for (size_t i = 0; i < idx.size(); ++i) {
        sorted[i] = table[idx[i]];
        sorted_plan[i] = p.tile_plan[idx[i]];
      }
      table.swap(sorted);
      p.tile_plan.swap(sorted_plan);
      for (size_t i = 0; i < table.size(); ++i) {
        if (i == 0 || tenant_of(i) != tenant_of(i - 1)) {
          qbeg.push_back(static_cast<int32_t>(i));
          qlen.push_back(0);
        }
        ++qlen.back();
      }
    }
    p.nq = static_cast<int>(qbeg.size());
    // Members nothing waits on (each tenant's last layer of the round; every
    // member of a single-layer round) skip the publish -- store-completion
    // wait, fence and counter atomic on the tail of their chain.  A round
    // whose tiles neither publish nor wait needs no counters at all, so its
    // launch also skips the last-CTA reset (the exit counter).
    {
      std::vector<char> needed(targets.size(), 0);
      for (const auto& te : table) {
        for (int i = 0; te.dep >= 0 && i < te.dep_n; ++i) needed[te.dep + i] = 1;
        for (int i = 0; te.rdep >= 0 && i < te.rdep_n; ++i) needed[te.rdep + i] = 1;
      }
      bool used = greedy_schedule || p.nq > 0;
      for (auto& te : table) {
        if (te.splits <= 1 && te.done >= 0 && !needed[te.done]) te.done = -1;
        used = used || te.done >= 0 || te.dep >= 0 || te.rdep >= 0;
      }
      p.self_reset = used;
    }
    p.n_tiles = static_cast<int>(table.size());
    p.n_counters = static_cast<int>(targets.size());
    p.n_ws = n_ws;
    if (n_ws > 0) {
      const size_t ws_bytes = static_cast<size_t>(n_ws) * dev::kBM * bn * sizeof(float);
      cuda_check(cudaMalloc(&p.ws, ws_bytes), "cudaMalloc(split workspace)");
      cuda_check(cudaMemset(p.ws, 0, ws_bytes), "clear split workspace");
      cuda_check(cudaMalloc(&p.split_ctr, static_cast<size_t>(n_ws) * 4 * sizeof(uint32_t)), "cudaMalloc(split ctr)");
      cuda_check(cudaMemset(p.split_ctr, 0, static_cast<size_t>(n_ws) * 4 * sizeof(uint32_t)), "clear split ctr");
      alignas(64) CUtensorMap map;
      const cuuint64_t dims[2] = {static_cast<cuuint64_t>(bn), static_cast<cuuint64_t>(n_ws) * dev::kBM};
      const cuuint64_t strides[1] = {static_cast<cuuint64_t>(bn) * 4};
      const cuuint32_t box[2] = {16, 32};
      const cuuint32_t estr[2] = {1, 1};
      const CUresult r = encode_tiled(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, p.ws, dims, strides, box, estr,
                                      CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_64B,
                                      CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      if (r != CUDA_SUCCESS) throw CudaError("cuTensorMapEncodeTiled(workspace) failed (" + std::to_string(int(r)) + ")");
      cuda_check(cudaMalloc(&p.ws_map, sizeof(CUtensorMap)), "cudaMalloc(ws map)");
      cuda_check(cudaMemcpy(p.ws_map, &map, sizeof(CUtensorMap), cudaMemcpyHostToDevice), "upload ws map");
    }
    cuda_check(cudaMalloc(&p.tiles, std::max<size_t>(1, table.size()) * sizeof(dev::TileEntry)), "cudaMalloc(tiles)");
    cuda_check(cudaMemcpy(p.tiles, table.data(), table.size() * sizeof(dev::TileEntry), cudaMemcpyHostToDevice),
               "upload round tiles");
    // counters and queue heads share one allocation: one memset per launch resets both
    p.greedy = greedy_schedule && !dynamic_schedule;
    // completion counters | queue heads | greedy claim counter | exit counter: zeroed here once,
    // then by each launch's last CTA (no per-launch memset)
    cuda_check(cudaMalloc(&p.counters, (targets.size() + p.nq + 2) * sizeof(uint32_t)), "cudaMalloc(counters)");
    cuda_check(cudaMemset(p.counters, 0, (targets.size() + p.nq + 2) * sizeof(uint32_t)), "clear counters");
    if (p.nq > 0) {
      p.heads = p.counters + targets.size();
      std::vector<int32_t> qinfo(qbeg);
      qinfo.insert(qinfo.end(), qlen.begin(), qlen.end());
      cuda_check(cudaMalloc(&p.qinfo, qinfo.size() * sizeof(int32_t)), "cudaMalloc(queues)");
      cuda_check(cudaMemcpy(p.qinfo, qinfo.data(), qinfo.size() * sizeof(int32_t), cudaMemcpyHostToDevice),
                 "upload queues");
    }
    cuda_check(cudaMalloc(&p.targets, std::max<size_t>(1, targets.size()) * sizeof(uint32_t)), "cudaMalloc(targets)");
    cuda_check(cudaMemcpy(p.targets, targets.data(), targets.size() * sizeof(uint32_t), cudaMemcpyHostToDevice),
               "upload round targets");
    return rounds.emplace(key, std::move(p)).first->second;
  }

  // The plan's pre-passes: row folds are batched (up to 16 jobs per launch,
  // blockIdx.y = job); explicit im2col runs one launch per operator.
  static constexpr int kFoldJobs = 16;
  int prepass_launches(const std::vector<int>& ops) const {
    int folds = 0, other = 0;
    for (int f : ops) (flat[f].fold ? folds : other) += 1;
    return (folds + kFoldJobs - 1) / kFoldJobs + other;
  }
  int launch_prepasses(const Prepared& p, cudaStream_t stream, bool count) {
    return launch_prepass_ops(p.prepass_ops, stream, count);
  }
  int launch_prepass_ops(const std::vector<int>& ops, cudaStream_t stream, bool count) {
    int launches = 0;
    dev::FoldBatch fb{};
    int nj = 0, max_pixels = 0;
    auto flush = [&]() {
      if (!nj) return;
      // 128-thread blocks (~4K registers): small enough to co-reside with the
      // persistent super-kernel's CTAs when an e2e graph runs them beside it
      const int gx = std::min((max_pixels + 127) / 128, sms * 16);
      dev::fold_rows<<<dim3(static_cast<unsigned>(gx), static_cast<unsigned>(nj)), 128, 0, stream>>>(fb);
      cuda_check(cudaGetLastError(), "launch fold_rows");
      ++launches;
      if (count) ++n_prepasses;
      nj = 0;
      max_pixels = 0;
    };
    for (int f : ops) {
      const Operator& op = flat[f];
      const Conv& c = op.conv;
      const int H = static_cast<int>(c.image_h), W = static_cast<int>(c.image_w), Cin = static_cast<int>(c.in_channels);
      const int R = static_cast<int>(c.kernel_h), S = static_cast<int>(c.kernel_w);
      const int st = static_cast<int>(c.stride), pad = static_cast<int>(c.padding), ldk = static_cast<int>(op.ldk);
      const int P = static_cast<int>((c.image_h + 2 * c.padding - c.kernel_h) / c.stride + 1);
      const int Q = static_cast<int>((c.image_w + 2 * c.padding - c.kernel_w) / c.stride + 1);
      if (op.fold) {
        fb.job[nj] = dev::FoldJob{static_cast<const __nv_bfloat16*>(op.x), static_cast<__nv_bfloat16*>(op.scratch),
                                  op.batch, H, W, Cin, S, st, pad, Q};
        max_pixels = std::max(max_pixels, op.batch * H * Q);
        if (++nj == kFoldJobs) flush();
        continue;
      }
      const int64_t total = op.shape.m * (op.ldk / 8);
      const int grid = static_cast<int>(std::min<int64_t>((total + 127) / 128, int64_t(sms) * 32));
      dev::im2col_prepass<<<grid, 128, 0, stream>>>(static_cast<const __nv_bfloat16*>(op.x),
                                                     static_cast<__nv_bfloat16*>(op.scratch), op.batch, H, W, Cin, R,
                                                     S, st, pad, P, Q, ldk);
      cuda_check(cudaGetLastError(), "launch im2col_prepass");
      ++launches;
      if (count) ++n_prepasses;
    }
    flush();
    return launches;
  }

  // Enqueue one plan: explicit-im2col pre-passes (if any), then the
  // super-kernel.  `ev` (optional) brackets the super-kernel with external
  // event records so a captured graph can time it.  `count` is false while
  // capturing (the graph counts its launches per replay).
  int launch(Prepared& p, cudaStream_t stream, bool count = true, cudaEvent_t ev_begin = nullptr,
             cudaEvent_t ev_end = nullptr, uint64_t* trace = nullptr) {
    int launches = 0;
    if (ev_begin) cuda_check(cudaEventRecordWithFlags(ev_begin, stream, cudaEventRecordExternal), "event record");
    launches += launch_prepasses(p, stream, count);
    const int grid = std::max(1, std::min(p.n_tiles, sms));
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(dev::kThreads);
    cfg.dynamicSmemBytes = smem_bytes;
    cfg.stream = stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = pdl ? 1 : 0;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    const dev::MemberDesc* slots = d_desc;
    const dev::TileEntry* tiles = p.tiles;
    int n = p.n_tiles;
    uint32_t* counters = p.counters;
    const uint32_t* targets = p.targets;
    dev::RoundArgs ra{counters, targets, p.ws_map, p.ws, p.split_ctr, trace,
                      p.heads, p.qinfo, p.qinfo ? p.qinfo + p.nq : nullptr, p.nq,
                      p.greedy ? p.counters + p.n_counters + p.nq : nullptr,
                      p.counters && p.self_reset ? p.counters + p.n_counters + p.nq + 1 : nullptr,
                      p.n_counters + p.nq + 1};
    void* args[4] = {&slots, &tiles, &n, &ra};
    cuda_check(cudaLaunchKernelExC(&cfg, kernel, args), "launch superkernel");
    if (ev_end) cuda_check(cudaEventRecordWithFlags(ev_end, stream, cudaEventRecordExternal), "event record");
    ++launches;
    if (count) {
      ++n_superkernels;
      n_tiles += p.n_tiles;
    }
    return launches;
  }
};

namespace {

std::vector<int> members_of(const Runtime& rt, const Plan& plan) {
  std::vector<int> v;
  v.reserve(plan.members.size());
  for (const Request& r : plan.members) {
    const int f = rt.flat_index(r.tenant, r.layer);
    if (!(rt.flat[f].shape == r.shape))
      throw std::invalid_argument("dispatch: request shape " + key_of(r.shape) + " does not match tenant " +
                                  std::to_string(r.tenant) + " layer " + std::to_string(r.layer) + " (" +
                                  key_of(rt.flat[f].shape) + ")");
    v.push_back(f);
  }
  return v;
}

Runtime& runtime_of(gm_ctx* ctx) {
  if (!ctx) throw std::invalid_argument("null context");
  if (!ctx->rt) throw NoDevice("context has no CUDA device (created with cuda_device < 0)");
  return *ctx->rt;
}

}  // namespace
}  // namespace gmb

// A captured launch program (see gm_graph_* in the header).
struct gm_graph {
  gm_ctx* ctx = nullptr;
  cudaGraph_t graph = nullptr;
  cudaGraphExec_t exec = nullptr;
  std::vector<cudaEvent_t> events;  // begin/end pairs when timed
  std::vector<cudaStream_t> streams;
  std::vector<cudaEvent_t> joins;
  int32_t superkernels = 0, kernels = 0;
  int64_t tiles = 0;
  ~gm_graph() {
    if (exec) cudaGraphExecDestroy(exec);
    if (graph) cudaGraphDestroy(graph);
    for (cudaEvent_t e : events) cudaEventDestroy(e);
    for (cudaEvent_t e : joins) cudaEventDestroy(e);
    for (cudaStream_t s : streams) cudaStreamDestroy(s);
  }
};

namespace gmb {
namespace {

// Capture `body(stream, graph)` on a private stream (thread-local capture
// mode, so other host threads are unaffected) and instantiate it.
template <class Body>
gm_graph* capture(gm_ctx* ctx, Body body) {
  Runtime& rt = runtime_of(ctx);
  cuda_check(cudaSetDevice(rt.device), "cudaSetDevice");
  auto* g = new gm_graph();
  g->ctx = ctx;
  try {
    cudaStream_t cs;
    cuda_check(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking), "cudaStreamCreate");
    g->streams.push_back(cs);
    cuda_check(cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal), "cudaStreamBeginCapture");
    try {
      body(cs, *g);
    } catch (...) {
      cudaGraph_t junk = nullptr;
      cudaStreamEndCapture(cs, &junk);
      if (junk) cudaGraphDestroy(junk);
      throw;
    }
    cuda_check(cudaStreamEndCapture(cs, &g->graph), "cudaStreamEndCapture");
    cuda_check(cudaGraphInstantiate(&g->exec, g->graph, 0), "cudaGraphInstantiate");
  } catch (...) {
    delete g;
    throw;
  }
  return g;
}

std::pair<cudaEvent_t, cudaEvent_t> timing_pair(gm_graph& g, bool timed) {
  if (!timed) return {nullptr, nullptr};
  cudaEvent_t a, b;
  cuda_check(cudaEventCreate(&a), "cudaEventCreate");
  cuda_check(cudaEventCreate(&b), "cudaEventCreate");
  g.events.push_back(a);
  g.events.push_back(b);
  return {a, b};
}

}  // namespace
}  // namespace gmb

using namespace gmb;

extern "C" {

int gm_create(const gm_device_spec* d, const gm_batch_policy* p, const gm_detector* det, int cuda_device,
              gm_ctx** out) {
  GM_API_BEGIN
  if (!out) throw std::invalid_argument("null argument: out");
  auto* ctx = new gm_ctx();
  try {
    ctx->dev = d ? to_device(*d) : b200_device();
    ctx->dev.check();
    if (p) ctx->pol = to_policy(*p);
    if (det) ctx->det = to_detector(*det);
    ctx->cuda_device = cuda_device;
    ctx->clock0_ns = std::chrono::duration_cast<std::chrono::nanoseconds>(
                         std::chrono::steady_clock::now().time_since_epoch()).count();
    if (cuda_device >= 0) {
      ctx->rt = new Runtime();
      ctx->rt->init(cuda_device, ctx->dev);
    }
  } catch (...) {
    delete ctx->rt;
    ctx->rt = nullptr;
    delete ctx;
    throw;
  }
  *out = ctx;
  GM_API_END
}

void gm_destroy(gm_ctx* ctx) {
  if (!ctx) return;
  delete ctx->rt;
  delete ctx;
}

int gm_ctx_queue(gm_ctx* ctx, gm_queue** q) {
  GM_API_BEGIN
  if (!ctx || !q) throw std::invalid_argument("null argument");
  *q = &ctx->queue;
  GM_CTX_API_END(ctx)
}

int gm_ctx_cache(gm_ctx* ctx, gm_cache** c) {
  GM_API_BEGIN
  if (!ctx || !c) throw std::invalid_argument("null argument");
  *c = &ctx->cache;
  GM_CTX_API_END(ctx)
}

int gm_ctx_device_spec(const gm_ctx* ctx, gm_device_spec* out) {
  GM_API_BEGIN
  if (!ctx || !out) throw std::invalid_argument("null argument");
  *out = from_device(ctx->dev);
  GM_CTX_API_END(ctx)
}

int gm_ctx_set_option(gm_ctx* ctx, const char* name, int64_t value) {
  GM_API_BEGIN
  if (!name) throw std::invalid_argument("null argument: name");
  Runtime& rt = runtime_of(ctx);
  const std::string n(name);
  if (n == "pdl") {
    rt.pdl = value != 0;
  } else if (n == "split_k") {
    rt.split_k = value != 0;
  } else if (n == "split_wide_kb") {
    if (value < 0) throw std::invalid_argument("split_wide_kb must be >= 0");
    rt.split_wide_kb = value;  // applies to round programs prepared afterwards (0 = off)
  } else if (n == "max_splits") {
    if (value < 2 || value > 64) throw std::invalid_argument("max_splits must be in [2, 64]");
    rt.max_splits = value;
  } else if (n == "dynamic_schedule") {
    rt.dynamic_schedule = value != 0;  // applies to round programs prepared afterwards
  } else if (n == "skinny_min_mb") {
    if (value < 0) throw std::invalid_argument("skinny_min_mb must be >= 0");
    rt.skinny_min_mb = value;  // applies to round programs prepared afterwards
  } else if (n == "skinny_max_splits") {
    if (value < 2 || value > 64) throw std::invalid_argument("skinny_max_splits must be in [2, 64]");
    rt.skinny_max_splits = value;
  } else if (n == "split_min_kb") {
    if (value < 1 || value > 1024) throw std::invalid_argument("split_min_kb must be in [1, 1024]");
    rt.split_min_kb = value;
  } else if (n == "tall_min_tiles") {
    if (value < 0) throw std::invalid_argument("tall_min_tiles must be >= 0");
    rt.tall_min_tiles = value;
  } else if (n == "critical_order") {
    if (value < -1 || value > 2) throw std::invalid_argument("critical_order must be -1 (auto), 0, 1 or 2");
    rt.critical_order = static_cast<int>(value);  // applies to round programs prepared afterwards
  } else if (n == "ring_layouts") {
    rt.ring_layouts = value != 0 ? 1 : 0;  // applies to tenants registered afterwards
  } else if (n == "tall_tiles") {
    rt.tall_tiles = value != 0;  // applies to plans prepared afterwards
  } else if (n == "greedy_schedule") {
    rt.greedy_schedule = value != 0;  // applies to round programs prepared afterwards
  } else if (n == "narrow_min_tiles") {
    rt.narrow_min_tiles = value;  // applies to plans prepared afterwards (0 = always full width)
  } else if (n == "staged_cc") {
    rt.staged_cc = value != 0;  // applies to tenants registered afterwards

  } else if (n == "row_fold") {
    rt.row_fold = value != 0;  // applies to tenants registered afterwards
  } else {
    throw std::invalid_argument("unknown option " + n);
  }
  GM_CTX_API_END(ctx)
}

int gm_ctx_set_policy(gm_ctx* ctx, const gm_batch_policy* p) {
  GM_API_BEGIN
  if (!ctx || !p) throw std::invalid_argument("null argument");
  ctx->pol = to_policy(*p);
  GM_CTX_API_END(ctx)
}

int gm_register_tenant(gm_ctx* ctx, const gm_tenant_desc* t, int32_t* tenant_index) {
  GM_API_BEGIN
  if (!t) throw std::invalid_argument("null argument: tenant");
  Runtime& rt = runtime_of(ctx);
  cuda_check(cudaSetDevice(rt.device), "cudaSetDevice");
  const int idx = rt.register_tenant(*t);
  Health h;
  h.tenant = idx;
  h.alpha = ctx->det.ewma_alpha;
  ctx->health.push_back(h);
  if (tenant_index) *tenant_index = idx;
  GM_CTX_API_END(ctx)
}

int gm_layer_shape(gm_ctx* ctx, int32_t tenant, int32_t layer, gm_gemm_shape* out) {
  GM_API_BEGIN
  if (!out) throw std::invalid_argument("null argument: out");
  *out = from_shape(runtime_of(ctx).op_of(tenant, layer).shape);
  GM_CTX_API_END(ctx)
}

int gm_tenant_count(const gm_ctx* ctx, int32_t* n) {
  GM_API_BEGIN
  if (!ctx || !n) throw std::invalid_argument("null argument");
  *n = ctx->rt ? static_cast<int32_t>(ctx->rt->tenant_ops.size()) : 0;
  GM_CTX_API_END(ctx)
}

// Re-placement of a tenant on another GPU's context (the
// reference makes eviction terminal, scheduler.cpp:225-244, and names
// re-admission as the open extension): the destination allocates
// the tenant's buffers, its weights and external inputs move with
// cudaMemcpyPeerAsync (NVLink P2P when the devices can reach each other;
// the same device is a plain device copy), and the layers register there with
// the same dataflow (views into producers' outputs keep their offsets).
int gm_migrate_tenants(gm_ctx* src, const int32_t* tenants, size_t n, gm_ctx* dst, uint64_t stream,
                       int32_t* out_tenants) {
  GM_API_BEGIN
  if (!tenants || !out_tenants || n == 0) throw std::invalid_argument("null argument");
  Runtime& a = runtime_of(src);
  Runtime& b = runtime_of(dst);
  for (size_t t = 0; t < n; ++t) a.op_of(tenants[t], 0);
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  cuda_check(cudaSetDevice(b.device), "cudaSetDevice");
  if (a.device != b.device) {
    int can = 0;
    cuda_check(cudaDeviceCanAccessPeer(&can, b.device, a.device), "cudaDeviceCanAccessPeer");
    if (can) {
      const cudaError_t e = cudaDeviceEnablePeerAccess(a.device, 0);
      if (e == cudaErrorPeerAccessAlreadyEnabled)
        cudaGetLastError();
      else
        cuda_check(e, "cudaDeviceEnablePeerAccess");
    }
  }
  // Source byte ranges already placed on the destination: a buffer several of
  // the tenants reference (a tenant's batch variants share one set) moves once.
  struct Range {
    const char* lo;
    int64_t bytes;
    char* dst;
  };
  std::vector<Range> placed;
  auto find = [&](const void* p, int64_t bytes) -> char* {
    const char* c = static_cast<const char*>(p);
    for (const Range& r : placed)
      if (c >= r.lo && c + bytes <= r.lo + r.bytes) return r.dst + (c - r.lo);
    return nullptr;
  };
  auto place = [&](const void* p, int64_t bytes, bool copy) {
    if (char* d = find(p, bytes)) return d;
    void* q = nullptr;
    cuda_check(cudaMalloc(&q, static_cast<size_t>(std::max<int64_t>(bytes, 16))), "cudaMalloc(migrated tenant)");
    b.owned.push_back(q);
    if (copy)
      cuda_check(cudaMemcpyPeerAsync(q, b.device, p, a.device, static_cast<size_t>(bytes), st), "cudaMemcpyPeerAsync");
    placed.push_back(Range{static_cast<const char*>(p), bytes, static_cast<char*>(q)});
    return static_cast<char*>(q);
  };
  // largest first, so a variant's buffers (views of the largest's) translate
  std::vector<size_t> order(n);
  for (size_t t = 0; t < n; ++t) order[t] = t;
  auto footprint = [&](int32_t tn) {
    int64_t s = 0;
    for (int f : a.tenant_ops[tn]) s += a.flat[f].y_bytes + a.flat[f].x_bytes;
    return s;
  };
  std::stable_sort(order.begin(), order.end(),
                   [&](size_t x, size_t y) { return footprint(tenants[x]) > footprint(tenants[y]); });
  std::vector<std::vector<gm_layer_desc>> nds(n);
  for (size_t oi : order) {
    const int32_t tenant = tenants[oi];
    const std::vector<gm_layer_desc>& descs = a.tenant_layers.at(static_cast<size_t>(tenant));
    const std::vector<int>& ops = a.tenant_ops[tenant];
    std::vector<gm_layer_desc>& nd = nds[oi];
    nd = descs;
    for (size_t i = 0; i < descs.size(); ++i) {  // outputs first: inputs may be views of them
      const Operator& op = a.flat[ops[i]];
      nd[i].y = place(descs[i].y, op.y_bytes, false);
    }
    for (size_t i = 0; i < descs.size(); ++i) {
      const gm_layer_desc& L = descs[i];
      const Operator& op = a.flat[ops[i]];
      nd[i].x = place(L.x, op.x_bytes, L.src < 0);
      if (L.w) {
        int64_t rows = 0, k = 0;
        if (L.kind == GM_LAYER_GEMM) {
          rows = L.gemm.n;
          k = L.gemm.k;
        } else if (L.kind == GM_LAYER_DWCONV) {
          rows = L.conv.in_channels;
          k = L.conv.kernel_h * L.conv.kernel_w;
        } else {
          rows = L.conv.out_channels;
          k = L.conv.kernel_h * L.conv.kernel_w * L.conv.in_channels;
        }
        const int64_t ldw = L.ldw > 0 ? L.ldw : k;
        nd[i].w = place(L.w, ((rows - 1) * ldw + k) * 2, true);
      }
      if (L.res) {
        const int64_t ldr = L.ldr > 0 ? L.ldr : op.shape.n;
        nd[i].res = place(L.res, ((op.shape.m - 1) * ldr + op.shape.n) * 2, L.res_src < 0);
      }
    }
  }
  cuda_check(cudaStreamSynchronize(st), "cudaStreamSynchronize(migration)");
  for (size_t t = 0; t < n; ++t) {
    const std::string id = "migrated/" + std::to_string(tenants[t]);
    gm_tenant_desc td{id.c_str(), nds[t].data(), nds[t].size(), a.tenant_slo[tenants[t]], a.tenant_conc[tenants[t]], 0};
    const int idx = b.register_tenant(td);
    Health h;
    h.tenant = idx;
    h.alpha = dst->det.ewma_alpha;
    dst->health.push_back(h);
    out_tenants[t] = idx;
  }
  GM_CTX_API_END(src)
}

int gm_migrate_tenant(gm_ctx* src, int32_t tenant, gm_ctx* dst, uint64_t stream, int32_t* out_tenant) {
  return gm_migrate_tenants(src, &tenant, 1, dst, stream, out_tenant);
}

int gm_prepare(gm_ctx* ctx, const gm_plans* p, size_t i) {
  GM_API_BEGIN
  if (!p || i >= p->plans.size()) throw std::invalid_argument("plan index out of range");
  Runtime& rt = runtime_of(ctx);
  cuda_check(cudaSetDevice(rt.device), "cudaSetDevice");
  rt.prepare(members_of(rt, p->plans[i]));
  GM_CTX_API_END(ctx)
}

int gm_dispatch(gm_ctx* ctx, const gm_plans* p, size_t i, uint64_t stream, double* planned_s, int* cache_hit) {
  GM_API_BEGIN
  if (!p || i >= p->plans.size()) throw std::invalid_argument("plan index out of range");
  Runtime& rt = runtime_of(ctx);
  const Plan& plan = p->plans[i];
  const std::vector<int> ops = members_of(rt, plan);
  Prepared& prep = rt.prepare(ops);
  const int64_t misses = ctx->cache.c.misses;
  const double dur = charge(plan, ctx->cache.c, ctx->dev);
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  cudaStreamCaptureStatus capturing = cudaStreamCaptureStatusNone;
  cuda_check(cudaStreamIsCapturing(s, &capturing), "cudaStreamIsCapturing");
  const bool track = capturing == cudaStreamCaptureStatusNone;
  // request I/O (gm_enqueue): query inputs land right before the launch
  auto io_of = [&](const Request& r) -> const gm_request_io* {
    auto it = ctx->io.find(r.id);
    return it == ctx->io.end() ? nullptr : &it->second;
  };
  for (size_t j = 0; j < plan.members.size(); ++j)
    if (const gm_request_io* io = io_of(plan.members[j]); io && io->x && io->x_bytes)
      cuda_check(cudaMemcpyAsync(const_cast<void*>(rt.flat[ops[j]].x), io->x, io->x_bytes, cudaMemcpyDefault, s),
                 "request input copy");
  InFlight f;
  if (track) {
    f.exec0 = rt.take_event();
    f.exec1 = rt.take_event();
    f.done = rt.take_event();
    cuda_check(cudaEventRecord(f.exec0, s), "cudaEventRecord");
  }
  rt.launch(prep, s);
  if (track) cuda_check(cudaEventRecord(f.exec1, s), "cudaEventRecord");
  for (size_t j = 0; j < plan.members.size(); ++j)
    if (const gm_request_io* io = io_of(plan.members[j]); io && io->y && io->y_bytes)
      cuda_check(cudaMemcpyAsync(io->y, rt.flat[ops[j]].y, io->y_bytes, cudaMemcpyDefault, s), "request output copy");
  if (track) {
    cuda_check(cudaEventRecord(f.done, s), "cudaEventRecord");
    f.members = plan.members;
    f.dispatch_ns = gm_ctx_now_ns(ctx);
    rt.inflight.push_back(std::move(f));
  }
  if (planned_s) *planned_s = dur;
  if (cache_hit) *cache_hit = ctx->cache.c.misses == misses ? 1 : 0;
  GM_CTX_API_END(ctx)
}

int gm_enqueue(gm_ctx* ctx, const gm_kernel_request* r, const gm_request_io* io) {
  GM_API_BEGIN
  if (!ctx || !r) throw std::invalid_argument("null argument");
  const Request req = to_request(*r);
  const bool has_io = io && ((io->x && io->x_bytes) || (io->y && io->y_bytes));
  if (ctx->rt) {
    const Operator& op = ctx->rt->op_of(req.tenant, req.layer);
    if (req.shape.valid() && !(op.shape == req.shape))
      throw std::invalid_argument("enqueue: request shape " + key_of(req.shape) + " does not match tenant " +
                                  std::to_string(req.tenant) + " layer " + std::to_string(req.layer) + " (" +
                                  key_of(op.shape) + ")");
    if (has_io && io->x && static_cast<int64_t>(io->x_bytes) > op.x_bytes)
      throw std::invalid_argument("enqueue: input copy of " + std::to_string(io->x_bytes) +
                                  " bytes exceeds the layer's input (" + std::to_string(op.x_bytes) + ")");
    if (has_io && io->y && static_cast<int64_t>(io->y_bytes) > op.y_bytes)
      throw std::invalid_argument("enqueue: output copy of " + std::to_string(io->y_bytes) +
                                  " bytes exceeds the layer's output (" + std::to_string(op.y_bytes) + ")");
  } else if (has_io) {
    throw NoDevice("context has no CUDA device (created with cuda_device < 0): request I/O needs one");
  }
  ctx->queue.q.push(req);  // scheduler.cpp:8-16 (duplicate id / invalid shape texts)
  if (has_io) ctx->io[req.id] = *io;
  if (!ctx->rt && req.tenant >= 0)
    while (static_cast<int>(ctx->health.size()) <= req.tenant) {
      Health h;
      h.tenant = static_cast<int>(ctx->health.size());
      h.alpha = ctx->det.ewma_alpha;
      ctx->health.push_back(h);
    }
  GM_CTX_API_END(ctx)
}

int gm_poll_completions(gm_ctx* ctx, gm_completion* out, size_t cap, size_t* n) {
  GM_API_BEGIN
  if (!n) throw std::invalid_argument("null argument: n");
  Runtime& rt = runtime_of(ctx);
  *n = 0;
  size_t written = 0;
  for (auto it = rt.inflight.begin(); it != rt.inflight.end();) {
    const cudaError_t q = cudaEventQuery(it->done);
    if (q == cudaErrorNotReady) {
      ++it;
      continue;
    }
    cuda_check(q, "dispatch completion");
    if (written + it->members.size() > cap) {
      if (written == 0) throw RangeError("poll_completions: a finished dispatch has " +
                                         std::to_string(it->members.size()) + " members, cap " + std::to_string(cap));
      break;
    }
    float ms = 0;
    cuda_check(cudaEventElapsedTime(&ms, it->exec0, it->exec1), "cudaEventElapsedTime");
    const int64_t now = gm_ctx_now_ns(ctx);
    for (const Request& r : it->members) {
      gm_completion& c = out[written++];
      c.request_id = r.id;
      c.tenant_index = r.tenant;
      c.layer_index = r.layer;
      c.pass_index = r.pass;
      c.batch = r.batch;
      c.enqueue_time = r.enqueue;
      c.slo_deadline = r.deadline;
      c.dispatch_ns = it->dispatch_ns;
      c.complete_ns = now;
      c.exec_seconds = static_cast<double>(ms) * 1e-3;
      c.plan_members = static_cast<int32_t>(it->members.size());
      c.reserved0 = 0;
      ctx->io.erase(r.id);
    }
    for (cudaEvent_t e : {it->exec0, it->exec1, it->done}) rt.ev_pool.push_back(e);
    it = rt.inflight.erase(it);
  }
  *n = written;
  GM_CTX_API_END(ctx)
}

int gm_ctx_in_flight(const gm_ctx* ctx, size_t* n) {
  GM_API_BEGIN
  if (!ctx || !n) throw std::invalid_argument("null argument");
  *n = ctx->rt ? ctx->rt->inflight.size() : 0;
  GM_API_END
}

int gm_ctx_synchronize(gm_ctx* ctx) {
  GM_API_BEGIN
  Runtime& rt = runtime_of(ctx);
  for (const InFlight& f : rt.inflight) cuda_check(cudaEventSynchronize(f.done), "cudaEventSynchronize");
  GM_CTX_API_END(ctx)
}

int gm_launch_members(gm_ctx* ctx, const int32_t* tenants, const int32_t* layers, size_t n, uint64_t stream,
                      int32_t* launches) {
  GM_API_BEGIN
  if (n == 0 || !tenants || !layers) throw std::invalid_argument("empty dispatch");
  Runtime& rt = runtime_of(ctx);
  std::vector<int> members;
  for (size_t j = 0; j < n; ++j) members.push_back(rt.flat_index(tenants[j], layers[j]));
  const int l = rt.launch(rt.prepare(members), reinterpret_cast<cudaStream_t>(stream));
  if (launches) *launches = l;
  GM_CTX_API_END(ctx)
}

int gm_members_launch_count(gm_ctx* ctx, const int32_t* tenants, const int32_t* layers, size_t n, int32_t* launches) {
  GM_API_BEGIN
  if (n == 0 || !tenants || !layers || !launches) throw std::invalid_argument("empty dispatch");
  Runtime& rt = runtime_of(ctx);
  std::vector<int> ops;
  for (size_t j = 0; j < n; ++j)
    if (rt.op_of(tenants[j], layers[j]).prepass) ops.push_back(rt.flat_index(tenants[j], layers[j]));
  *launches = 1 + rt.prepass_launches(ops);
  GM_CTX_API_END(ctx)
}

int gm_plan_round(gm_ctx* ctx, const int32_t* tenants, size_t n, int64_t now, gm_plans** out) {
  GM_API_BEGIN
  if (!out || (n && !tenants)) throw std::invalid_argument("null argument");
  Runtime& rt = runtime_of(ctx);
  std::vector<RoundTenant> round;
  round.reserve(n);
  for (size_t j = 0; j < n; ++j) {
    const int t = tenants[j];
    rt.op_of(t, 0);
    if (ctx->health[t].evicted) continue;  // eviction is terminal (scheduler.cpp:225-244)
    RoundTenant rtn;
    rtn.tenant = t;
    for (int f : rt.tenant_ops[t]) rtn.layers.push_back(rt.flat[f].shape);
    rtn.slo_ns = to_ns(rt.tenant_slo[t]);
    round.push_back(std::move(rtn));
  }
  RoundResult res = plan_round(round, now, ctx->pol, ctx->dev, ctx->cache.c, ctx->next_request_id);
  auto* plans = new gm_plans();
  for (RoundDispatch& d : res.dispatches) {
    plans->plans.push_back(std::move(d.plan));
    plans->times.emplace_back(d.start, d.end);
  }
  *out = plans;
  GM_CTX_API_END(ctx)
}

int gm_plans_times(const gm_plans* p, size_t i, int64_t* start, int64_t* end) {
  GM_API_BEGIN
  if (!p || i >= p->times.size()) throw std::invalid_argument("plan index out of range");
  if (start) *start = p->times[i].first;
  if (end) *end = p->times[i].second;
  GM_API_END
}

int gm_prepare_plans(gm_ctx* ctx, const gm_plans* p) {
  GM_API_BEGIN
  if (!p) throw std::invalid_argument("null argument: plans");
  Runtime& rt = runtime_of(ctx);
  cuda_check(cudaSetDevice(rt.device), "cudaSetDevice");
  for (const Plan& plan : p->plans) rt.prepare(members_of(rt, plan));
  GM_CTX_API_END(ctx)
}

int gm_dispatch_plans(gm_ctx* ctx, const gm_plans* p, uint64_t stream, int32_t* launches) {
  GM_API_BEGIN
  if (!p) throw std::invalid_argument("null argument: plans");
  Runtime& rt = runtime_of(ctx);
  int l = 0;
  for (const Plan& plan : p->plans) l += rt.launch(rt.prepare(members_of(rt, plan)), reinterpret_cast<cudaStream_t>(stream));
  if (launches) *launches = l;
  GM_CTX_API_END(ctx)
}

int gm_graph_capture_plans(gm_ctx* ctx, const gm_plans* p, int timed, gm_graph** out) {
  GM_API_BEGIN
  if (!p || !out) throw std::invalid_argument("null argument");
  Runtime& rt = runtime_of(ctx);
  std::vector<Prepared*> preps;
  for (const Plan& plan : p->plans) preps.push_back(&rt.prepare(members_of(rt, plan)));
  *out = capture(ctx, [&](cudaStream_t cs, gm_graph& g) {
    for (Prepared* pr : preps) {
      auto ev = timing_pair(g, timed != 0);
      g.kernels += rt.launch(*pr, cs, false, ev.first, ev.second);
      g.superkernels += 1;
      g.tiles += pr->n_tiles;
    }
  });
  GM_CTX_API_END(ctx)
}

int gm_graph_capture_serial(gm_ctx* ctx, const int32_t* tenants, size_t n, int mode, int timed, gm_graph** out) {
  GM_API_BEGIN
  if (!out || (n && !tenants)) throw std::invalid_argument("null argument");
  if (mode != GM_MODE_TIME_ONLY && mode != GM_MODE_SPACE_ONLY) throw std::invalid_argument("unknown serial mode");
  Runtime& rt = runtime_of(ctx);
  std::vector<std::vector<Prepared*>> per_tenant;
  for (size_t j = 0; j < n; ++j) {
    rt.op_of(tenants[j], 0);
    std::vector<Prepared*> v;
    for (int f : rt.tenant_ops[tenants[j]]) v.push_back(&rt.prepare({f}));
    per_tenant.push_back(std::move(v));
  }
  *out = capture(ctx, [&](cudaStream_t cs, gm_graph& g) {
    if (mode == GM_MODE_TIME_ONLY) {
      for (auto& v : per_tenant)
        for (Prepared* pr : v) {
          auto ev = timing_pair(g, timed != 0);
          g.kernels += rt.launch(*pr, cs, false, ev.first, ev.second);
          g.superkernels += 1;
          g.tiles += pr->n_tiles;
        }
      return;
    }
    cudaEvent_t fork;
    cuda_check(cudaEventCreateWithFlags(&fork, cudaEventDisableTiming), "cudaEventCreate");
    g.joins.push_back(fork);
    cuda_check(cudaEventRecord(fork, cs), "cudaEventRecord");
    std::vector<cudaEvent_t> done;
    for (auto& v : per_tenant) {
      cudaStream_t s;
      cuda_check(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking), "cudaStreamCreate");
      g.streams.push_back(s);
      cuda_check(cudaStreamWaitEvent(s, fork, 0), "cudaStreamWaitEvent");
      for (Prepared* pr : v) {
        auto ev = timing_pair(g, timed != 0);
        g.kernels += rt.launch(*pr, s, false, ev.first, ev.second);
        g.superkernels += 1;
        g.tiles += pr->n_tiles;
      }
      cudaEvent_t e;
      cuda_check(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "cudaEventCreate");
      g.joins.push_back(e);
      cuda_check(cudaEventRecord(e, s), "cudaEventRecord");
      done.push_back(e);
    }
    for (cudaEvent_t e : done) cuda_check(cudaStreamWaitEvent(cs, e, 0), "cudaStreamWaitEvent");
  });
  GM_CTX_API_END(ctx)
}

int gm_dispatch_round(gm_ctx* ctx, const gm_plans* p, uint64_t stream, int32_t* launches) {
  GM_API_BEGIN
  if (!p) throw std::invalid_argument("null argument: plans");
  Runtime& rt = runtime_of(ctx);
  std::vector<std::vector<int>> plans;
  for (const Plan& plan : p->plans) plans.push_back(members_of(rt, plan));
  const int l = rt.launch(rt.prepare_round(plans), reinterpret_cast<cudaStream_t>(stream));
  if (launches) *launches = l;
  GM_CTX_API_END(ctx)
}

int gm_trace_round(gm_ctx* ctx, const gm_plans* p, uint64_t stream, uint64_t* out, size_t cap, size_t* n_tiles) {
  GM_API_BEGIN
  if (!p) throw std::invalid_argument("null argument: plans");
  Runtime& rt = runtime_of(ctx);
  std::vector<std::vector<int>> plans;
  for (const Plan& plan : p->plans) plans.push_back(members_of(rt, plan));
  Prepared& pr = rt.prepare_round(plans);
  if (n_tiles) *n_tiles = static_cast<size_t>(pr.n_tiles);
  const size_t words = static_cast<size_t>(pr.n_tiles) * 6;
  if (!out || cap < words) throw RangeError("output buffer too small");
  // the kernel also stamps 6 words per CTA after the tiles (SM cycles: entry,
  // setup, loops, barrier, TMEM released, exit); returned when the buffer has room
  const size_t all = words + 6 * static_cast<size_t>(std::max(1, std::min(pr.n_tiles, rt.sms)));
  const size_t copy = cap >= all ? all : words;
  uint64_t* d_trace = nullptr;
  cuda_check(cudaMalloc(&d_trace, all * sizeof(uint64_t)), "cudaMalloc(trace)");
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  cudaMemsetAsync(d_trace, 0, all * sizeof(uint64_t), s);
  rt.launch(pr, s, true, nullptr, nullptr, d_trace);
  cudaError_t e = cudaMemcpyAsync(out, d_trace, copy * sizeof(uint64_t), cudaMemcpyDeviceToHost, s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  cudaFree(d_trace);
  cuda_check(e, "trace copy");
  GM_CTX_API_END(ctx)
}

int gm_round_tiles(gm_ctx* ctx, const gm_plans* p, gm_tile* out, size_t cap, size_t* n) {
  GM_API_BEGIN
  if (!p) throw std::invalid_argument("null argument: plans");
  Runtime& rt = runtime_of(ctx);
  std::vector<std::vector<int>> plans;
  for (const Plan& plan : p->plans) plans.push_back(members_of(rt, plan));
  Prepared& pr = rt.prepare_round(plans);
  std::vector<dev::TileEntry> table(pr.n_tiles);
  cuda_check(cudaMemcpy(table.data(), pr.tiles, table.size() * sizeof(dev::TileEntry), cudaMemcpyDeviceToHost),
             "read round tiles");
  std::vector<gm_tile> v;
  for (size_t i = 0; i < table.size(); ++i)  // flags = plan index of the tile
    v.push_back(gm_tile{table[i].member, pr.tile_plan[i], table[i].m_tile, table[i].n_tile});
  if (n) *n = v.size();
  if (!out || cap < v.size()) throw RangeError("output buffer too small");
  std::copy(v.begin(), v.end(), out);
  GM_CTX_API_END(ctx)
}

int gm_round_tile_info(gm_ctx* ctx, const gm_plans* p, gm_round_tile* out, size_t cap, size_t* n) {
  GM_API_BEGIN
  if (!p) throw std::invalid_argument("null argument: plans");
  Runtime& rt = runtime_of(ctx);
  std::vector<std::vector<int>> plans;
  for (const Plan& plan : p->plans) plans.push_back(members_of(rt, plan));
  Prepared& pr = rt.prepare_round(plans);
  std::vector<dev::TileEntry> table(pr.n_tiles);
  cuda_check(cudaMemcpy(table.data(), pr.tiles, table.size() * sizeof(dev::TileEntry), cudaMemcpyDeviceToHost),
             "read round tiles");
  if (n) *n = table.size();
  if (!out || cap < table.size()) throw RangeError("output buffer too small");
  for (size_t i = 0; i < table.size(); ++i) {
    const dev::TileEntry& te = table[i];
    const Operator& op = rt.flat[rt.slot_op[te.member]];
    const dev::MemberDesc& md = rt.host_desc[te.member];
    gm_round_tile& o = out[i];
    o.tenant = op.tenant;
    o.layer = op.layer;
    o.m_tile = te.m_tile;
    o.n_tile = te.n_tile;
    o.rows = static_cast<int32_t>(tile_rows_of(op, md.tall != 0));
    o.cols = md.n_tile;
    o.splits = te.splits > 1 ? te.splits : 1;
    o.kb_begin = te.kb_begin;
    o.kb_end = te.kb_end;
    o.done = te.done;
    o.dep = te.dep;
    o.dep_n = te.dep >= 0 ? te.dep_n : 0;
    o.rdep = te.rdep;
    o.rdep_n = te.rdep >= 0 ? te.rdep_n : 0;
    o.plan = pr.tile_plan[i];
    o.cuda_core = dev::cuda_core_mode(md.a_mode) ? 1 : 0;
  }
  GM_CTX_API_END(ctx)
}

int gm_graph_capture_round(gm_ctx* ctx, const gm_plans* p, int timed, gm_graph** out) {
  GM_API_BEGIN
  if (!p || !out) throw std::invalid_argument("null argument");
  Runtime& rt = runtime_of(ctx);
  std::vector<std::vector<int>> plans;
  for (const Plan& plan : p->plans) plans.push_back(members_of(rt, plan));
  Prepared* pr = &rt.prepare_round(plans);
  *out = capture(ctx, [&](cudaStream_t cs, gm_graph& g) {
    auto ev = timing_pair(g, timed != 0);
    g.kernels += rt.launch(*pr, cs, false, ev.first, ev.second);
    g.superkernels += 1;
    g.tiles += pr->n_tiles;
  });
  GM_CTX_API_END(ctx)
}

int gm_graph_capture_round_e2e(gm_ctx* ctx, const gm_plans* p, size_t n, const int32_t* tenants,
                               const void* const* h_in, void* const* d_in, const size_t* in_bytes,
                               const void* const* d_out, void* const* h_out, const size_t* out_bytes,
                               gm_graph** out) {
  GM_API_BEGIN
  if (!p || !out || (n && (!tenants || !h_in || !d_in || !in_bytes || !d_out || !h_out || !out_bytes)))
    throw std::invalid_argument("null argument");
  Runtime& rt = runtime_of(ctx);
  std::vector<std::vector<int>> plans;
  for (const Plan& plan : p->plans) plans.push_back(members_of(rt, plan));
  // The copy branch's pre-pass blocks must fit beside a persistent CTA
  // (registers: the CTA's allocation plus one 128-thread pre-pass block);
  // otherwise gates could wait on work that cannot be scheduled, so the
  // program is captured serially instead (copies, round, results).
  auto regs_of = [](const void* fn) {
    cudaFuncAttributes a{};
    cuda_check(cudaFuncGetAttributes(&a, fn), "cudaFuncGetAttributes");
    return (a.numRegs + 7) / 8 * 8;
  };
  const int pre_regs = std::max(regs_of(reinterpret_cast<const void*>(&dev::fold_rows)),
                                regs_of(reinterpret_cast<const void*>(&dev::im2col_prepass)));
  const bool co_resident = regs_of(rt.kernel) * dev::kThreads + pre_regs * 128 <= 65536;
  if (!co_resident) {
    Prepared* sp = &rt.prepare_round(plans);
    *out = capture(ctx, [&](cudaStream_t cs, gm_graph& g) {
      for (size_t i = 0; i < n; ++i)
        if (in_bytes[i]) cuda_check(cudaMemcpyAsync(d_in[i], h_in[i], in_bytes[i], cudaMemcpyHostToDevice, cs), "H2D query");
      g.kernels += rt.launch(*sp, cs, false);
      g.superkernels += 1;
      g.tiles += sp->n_tiles;
      for (size_t i = 0; i < n; ++i)
        if (out_bytes[i])
          cuda_check(cudaMemcpyAsync(h_out[i], d_out[i], out_bytes[i], cudaMemcpyDeviceToHost, cs), "D2H result");
    });
    return GM_OK;
  }
  Prepared* pr = &rt.prepare_round(plans, true);
  for (size_t i = 0; i < n; ++i) {
    bool found = false;
    for (const auto& gt : pr->gates) found |= gt.first == tenants[i];
    if (!found) throw std::invalid_argument("e2e round: tenant " + std::to_string(tenants[i]) + " is not in the round");
  }
  // every gate of the round must be opened by this program, or the kernel
  // would spin on it until the device-side watchdog traps
  for (const auto& gt : pr->gates) {
    bool covered = false;
    for (size_t i = 0; i < n; ++i) covered |= gt.first == tenants[i];
    if (!covered)
      throw std::invalid_argument("e2e round: tenant " + std::to_string(gt.first) +
                                  " of the round has no host input (every round tenant needs one)");
  }
  *out = capture(ctx, [&](cudaStream_t cs, gm_graph& g) {
    // copy branch: each tenant's H2D, its layer-0 pre-pass, then the gate
    // DMA; the round kernel runs concurrently and starts a tenant's chain as
    // soon as its gate opens (the pre-pass blocks co-reside with the
    // persistent CTAs: 31 registers x 256 threads fit the SM's spare file)
    // (copies back to back on one stream; a tenant's layer-0 pre-pass and
    // gate on a second, so pre-passes do not hold up the next tenant's copy)
    cudaStream_t ss, sp;
    cuda_check(cudaStreamCreateWithFlags(&ss, cudaStreamNonBlocking), "cudaStreamCreate");
    cuda_check(cudaStreamCreateWithFlags(&sp, cudaStreamNonBlocking), "cudaStreamCreate");
    g.streams.push_back(ss);
    g.streams.push_back(sp);
    auto new_event = [&]() {
      cudaEvent_t e;
      cuda_check(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "cudaEventCreate");
      g.joins.push_back(e);
      return e;
    };
    cudaEvent_t fork = new_event(), join = new_event(), copies = new_event();
    cuda_check(cudaEventRecord(fork, cs), "cudaEventRecord");
    cuda_check(cudaStreamWaitEvent(ss, fork, 0), "cudaStreamWaitEvent");
    cuda_check(cudaStreamWaitEvent(sp, fork, 0), "cudaStreamWaitEvent");
    for (size_t i = 0; i < n; ++i) {
      cuda_check(cudaMemcpyAsync(d_in[i], h_in[i], in_bytes[i], cudaMemcpyHostToDevice, ss), "H2D query");
      std::vector<int> ops;
      for (int f : pr->gated_prepass)
        if (rt.flat[f].tenant == tenants[i]) ops.push_back(f);
      cudaStream_t gs = ss;
      if (!ops.empty()) {
        cudaEvent_t landed = new_event();
        cuda_check(cudaEventRecord(landed, ss), "cudaEventRecord");
        cuda_check(cudaStreamWaitEvent(sp, landed, 0), "cudaStreamWaitEvent");
        g.kernels += rt.launch_prepass_ops(ops, sp, false);
        gs = sp;
      }
      for (const auto& gt : pr->gates)
        if (gt.first == tenants[i])
          cuda_check(cudaMemcpyAsync(pr->counters + gt.second, rt.host_one, sizeof(uint32_t), cudaMemcpyHostToDevice, gs),
                     "open input gate");
    }
    cuda_check(cudaEventRecord(copies, ss), "cudaEventRecord");
    cuda_check(cudaStreamWaitEvent(sp, copies, 0), "cudaStreamWaitEvent");
    cuda_check(cudaEventRecord(join, sp), "cudaEventRecord");
    g.kernels += rt.launch(*pr, cs, false);
    g.superkernels += 1;
    g.tiles += pr->n_tiles;
    cuda_check(cudaStreamWaitEvent(cs, join, 0), "cudaStreamWaitEvent");
    for (size_t i = 0; i < n; ++i)
      cuda_check(cudaMemcpyAsync(h_out[i], d_out[i], out_bytes[i], cudaMemcpyDeviceToHost, cs), "D2H result");
  });
  GM_CTX_API_END(ctx)
}

int gm_serve_trace(gm_ctx* ctx, gm_dispatch_event* out, size_t cap, size_t* n) {
  GM_API_BEGIN
  Runtime& rt = runtime_of(ctx);
  if (n) *n = rt.serve_trace.size();
  if (!out) return GM_OK;
  if (cap < rt.serve_trace.size()) throw RangeError("output buffer too small");
  std::copy(rt.serve_trace.begin(), rt.serve_trace.end(), out);
  GM_CTX_API_END(ctx)
}

int gm_graph_launch(gm_graph* g, uint64_t stream) {
  GM_API_BEGIN
  if (!g) throw std::invalid_argument("null graph");
  Runtime& rt = runtime_of(g->ctx);
  cuda_check(cudaGraphLaunch(g->exec, reinterpret_cast<cudaStream_t>(stream)), "cudaGraphLaunch");
  rt.n_superkernels += g->superkernels;
  rt.n_prepasses += g->kernels - g->superkernels;
  rt.n_tiles += g->tiles;
  GM_API_END
}

int gm_graph_launch_count(const gm_graph* g, int32_t* superkernels, int32_t* kernels) {
  GM_API_BEGIN
  if (!g) throw std::invalid_argument("null graph");
  if (superkernels) *superkernels = g->superkernels;
  if (kernels) *kernels = g->kernels;
  GM_API_END
}

int gm_graph_kernel_times(gm_graph* g, float* ms, size_t cap, size_t* n) {
  GM_API_BEGIN
  if (!g) throw std::invalid_argument("null graph");
  const size_t pairs = g->events.size() / 2;
  if (n) *n = pairs;
  if (pairs == 0) return GM_OK;
  if (!ms || cap < pairs) throw RangeError("output buffer too small");
  cuda_check(cudaEventSynchronize(g->events.back()), "cudaEventSynchronize");
  for (size_t i = 0; i < pairs; ++i)
    cuda_check(cudaEventElapsedTime(&ms[i], g->events[2 * i], g->events[2 * i + 1]), "cudaEventElapsedTime");
  GM_API_END
}

void gm_graph_destroy(gm_graph* g) { delete g; }

int gm_ctx_launch_stats(const gm_ctx* ctx, int64_t* superkernels, int64_t* prepasses, int64_t* tiles) {
  GM_API_BEGIN
  if (!ctx) throw std::invalid_argument("null context");
  const Runtime* rt = ctx->rt;
  if (superkernels) *superkernels = rt ? rt->n_superkernels : 0;
  if (prepasses) *prepasses = rt ? rt->n_prepasses : 0;
  if (tiles) *tiles = rt ? rt->n_tiles : 0;
  GM_CTX_API_END(ctx)
}

}  // extern "C"

// ---------------------------------------------------------------------------
// Real-clock serving: the B200 form of run_space_time (proj/src/sim.cpp:398-581).
//
// Queries arrive per logical tenant (Poisson, or closed loop: a query re-arrives
// when the previous one completes).  The batcher keeps per-tenant pending
// queues and triggers a dispatch on the reference's three conditions
// (form_batches, scheduler.cpp:166-197): size (pending queries >= target,
// auto = live tenants as in sim.cpp:516-523), age (oldest >= max_wait) or SLO
// (some pending query's deadline minus the predicted round time has passed).
// A dispatch takes up to one max-batch of queries per tenant (the tenant's
// dynamic batch: the smallest registered batch variant that holds them) and
// runs them as one round program: the reference planner orders and packs every
// layer of every member (plan_round), one persistent super-kernel launch
// executes it with device-side layer dependencies.  Plans and device tables are
// cached per member set (the SuperKernelCache meaning on B200).  Completions
// come from CUDA events; each member tenant's monitor is fed the round's device
// time (execution time, sim.cpp:475-476), then stragglers are detected and
// evicted (terminal, scheduler.cpp:225-271).
namespace gmb {
namespace {

struct ServeQuery {
  int64_t arrival_ns;
  int64_t seq;  // per logical tenant: arrival order (its host I/O slot is seq % io_slots)
};

struct ServeRound {
  cudaEvent_t ev0 = nullptr, ev1 = nullptr, ev2 = nullptr;  // launch begin / end, copy-out end
  std::vector<std::pair<int, std::vector<ServeQuery>>> members;  // (logical tenant, its queries)
  std::vector<std::vector<int>> keys;  // cached member sets launched (one, or singles while the set is prepared)
  int64_t dispatch_ns = 0;
  double flops = 0;  // the members' queries' FLOPs (served work)
  int32_t tiles = 0;
  int32_t launches = 0;
};

int64_t since(std::chrono::steady_clock::time_point t0) {
  return std::chrono::duration_cast<std::chrono::nanoseconds>(std::chrono::steady_clock::now() - t0).count();
}

}  // namespace
}  // namespace gmb

extern "C" int gm_serve(gm_ctx* ctx, const gm_serve_tenant* tenants, size_t n, const gm_serve_config* cfg,
                        gm_serve_stats* out, double* latencies_ms, size_t cap, size_t* n_lat) {
  GM_API_BEGIN
  if (!tenants || n == 0 || !cfg || !out) throw std::invalid_argument("null argument");
  Runtime& rt = runtime_of(ctx);
  cuda_check(cudaSetDevice(rt.device), "cudaSetDevice");
  if (cfg->prewarm < 0) throw std::invalid_argument("serve: prewarm cap must be >= 0");
  if (cfg->plan_cache_cap < 0) throw std::invalid_argument("serve: plan cache cap must be >= 0");
  // degradation is off when degrade_slowdown == 0 (a zero-initialised config)
  const int deg_t = cfg->degrade_slowdown != 0.0 ? cfg->degrade_tenant : -1;
  if (deg_t >= static_cast<int>(n)) throw std::invalid_argument("serve: degradation names unknown tenant");
  if (deg_t >= 0 && cfg->degrade_slowdown < 1.0) throw std::invalid_argument("serve: degradation slowdown must be >= 1");
  const int64_t deg_start_ns = deg_t >= 0 ? to_ns(cfg->degrade_start) : 0;
  if (cfg->duration <= 0 || cfg->warmup < 0 || cfg->warmup >= cfg->duration)
    throw std::invalid_argument("serve: need 0 <= warmup < duration");
  const int depth = std::max(1, cfg->depth);
  const int64_t duration_ns = to_ns(cfg->duration), warmup_ns = to_ns(cfg->warmup);
  const int64_t max_wait_ns = to_ns(cfg->max_wait >= 0 ? cfg->max_wait : ctx->pol.max_wait);
  cudaStream_t stream = reinterpret_cast<cudaStream_t>(cfg->stream);

  struct T {
    std::vector<std::pair<int, int>> variants;  // (batch, runtime tenant), ascending batch
    double rate = 0, slo = 0.1;
    int conc = 0;
    int64_t flops = 0;
    std::deque<ServeQuery> pending;
    std::vector<int64_t> delayed;  // closed-loop re-arrivals after a degraded (delayed) completion
    int64_t next_arrival = 0, next_seq = 0;
    std::mt19937_64 rng;
    bool live = true;
    // per-query I/O (host_input != null): pinned host slots, the device query
    // input (layer 0's x) and output (last layer's y), bytes per query
    const char* hin = nullptr;
    char* hout = nullptr;
    int slots = 0;
    char* dx = nullptr;
    const char* dy = nullptr;
    int64_t in_q = 0, out_q = 0;
    void push(int64_t arrival) { pending.push_back(ServeQuery{arrival, next_seq++}); }
  };
  std::vector<T> ts(n);
  std::vector<Health> health(n);
  for (size_t i = 0; i < n; ++i) {
    const gm_serve_tenant& st = tenants[i];
    if (st.n_variants < 1 || !st.variant_tenant || !st.variant_batch)
      throw std::invalid_argument("serve: tenant needs at least one batch variant");
    for (int v = 0; v < st.n_variants; ++v) {
      rt.op_of(st.variant_tenant[v], 0);
      if (st.variant_batch[v] < 1) throw std::invalid_argument("serve: variant batch must be >= 1");
      ts[i].variants.emplace_back(st.variant_batch[v], st.variant_tenant[v]);
    }
    std::sort(ts[i].variants.begin(), ts[i].variants.end());
    if (st.rate_qps < 0 || (st.rate_qps == 0 && st.concurrency < 1))
      throw std::invalid_argument("serve: tenant needs a Poisson rate > 0 or a closed-loop concurrency >= 1");
    ts[i].rate = st.rate_qps;
    ts[i].conc = st.concurrency;
    ts[i].slo = st.slo_latency > 0 ? st.slo_latency : 0.1;
    ts[i].flops = st.flops_per_query;
    if (st.host_input || st.host_output) {
      if (!st.host_input || !st.host_output || st.io_slots < 1)
        throw std::invalid_argument("serve: per-query I/O needs host_input, host_output and io_slots >= 1");
      const auto [bmax, tid] = ts[i].variants.back();
      const Operator& first = rt.op_of(tid, 0);
      const Operator& last = rt.flat[rt.tenant_ops[tid].back()];
      const int64_t cols = first.kind == GM_LAYER_GEMM ? first.shape.k : first.conv.in_channels;
      ts[i].hin = static_cast<const char*>(st.host_input);
      ts[i].hout = static_cast<char*>(st.host_output);
      ts[i].slots = st.io_slots;
      ts[i].dx = const_cast<char*>(static_cast<const char*>(first.x));
      ts[i].dy = last.y;
      ts[i].in_q = (first.x_bytes + (first.x_pitch - cols) * 2) / bmax;  // rows of one query x pitch
      ts[i].out_q = last.y_bytes / bmax;
    }
    // per-tenant stream: splitmix-chained seed (hash, never XOR)
    uint64_t h = cfg->seed + 0x9E3779B97F4A7C15ull * (i + 1);
    h = (h ^ (h >> 30)) * 0xBF58476D1CE4E5B9ull;
    h = (h ^ (h >> 27)) * 0x94D049BB133111EBull;
    ts[i].rng.seed(h ^ (h >> 31));
    health[i].tenant = static_cast<int>(i);
    health[i].alpha = ctx->det.ewma_alpha;
  }
  auto draw = [](T& t) {
    std::exponential_distribution<double> e(t.rate);
    return static_cast<int64_t>(std::llround(e(t.rng) * 1e9));
  };
  for (T& t : ts) {
    if (t.rate > 0)
      t.next_arrival = draw(t);
    else
      for (int c = 0; c < t.conc; ++c) t.push(0);
  }

  // Plan + device-table cache per member set (the SuperKernelCache on B200),
  // bounded (plan_cache_cap > 0: least recently used sets not in flight are
  // dropped).  Single-tenant sets (every variant) are pinned: with async_plan a
  // set seen for the first time is planned and uploaded on a worker thread
  // while its dispatch runs as back-to-back round programs of cached
  // sub-sets (largest first, then single-tenant sets).
  struct Cached {
    Prepared* prep;
    double planned_s;
    uint64_t last_use;
    int inflight;
    bool pinned;
    size_t members;
  };
  std::map<std::vector<int>, Cached> cache;
  std::vector<Prepared> graveyard;  // evicted device tables, freed after the loop
  std::unordered_map<int, std::pair<int, int>> var_of;  // runtime tenant -> (logical tenant, batch)
  for (size_t i = 0; i < n; ++i)
    for (const auto& [b, id] : ts[i].variants) var_of[id] = {static_cast<int>(i), b};
  int64_t padded = 0;
  std::map<std::vector<int>, int> misses_of;  // async planning: sightings of not-yet-planned sets
  // a cached program's expected device time: measured (alone, this ctx), else
  // planned scaled by what measurements showed of the planner's estimates
  auto expect_s = [&](const Cached& c) {
    return c.prep->measured_s > 0 ? c.prep->measured_s : c.planned_s * rt.serve_ratio[c.members > 1 ? 1 : 0];
  };
  int64_t plan_hits = 0, plan_misses = 0, evictions = 0, fallbacks = 0;
  uint64_t use_clock = 0;
  auto plan_members = [&](const std::vector<int>& key) {
    std::vector<RoundTenant> round;
    for (int id : key) {
      RoundTenant rtn;
      rtn.tenant = id;
      for (int f : rt.tenant_ops[id]) rtn.layers.push_back(rt.flat[f].shape);
      rtn.slo_ns = to_ns(rt.tenant_slo[id]);
      round.push_back(std::move(rtn));
    }
    RoundResult res = plan_round(round, 0, ctx->pol, ctx->dev, ctx->cache.c, ctx->next_request_id);
    std::vector<std::vector<int>> plans;
    TimeNs end = 0;
    for (RoundDispatch& d : res.dispatches) {
      plans.push_back(members_of(rt, d.plan));
      end = std::max(end, d.end);
    }
    return std::make_pair(&rt.prepare_round(plans), to_seconds(end));
  };
  // round programs that existed before this call (other launch programs may
  // hold them) are never evicted
  std::set<const Prepared*> preexisting;
  {
    std::lock_guard<std::recursive_mutex> lock(rt.rounds_mu);
    for (const auto& [k, pr] : rt.rounds) preexisting.insert(&pr);
  }
  auto insert = [&](const std::vector<int>& key, std::pair<Prepared*, double> pp, bool pinned) {
    pinned = pinned || preexisting.count(pp.first) > 0;
    auto it = cache.emplace(key, Cached{pp.first, pp.second, ++use_clock, 0, pinned, key.size()}).first;
    if (cfg->plan_cache_cap > 0) {
      while (static_cast<int64_t>(cache.size()) > cfg->plan_cache_cap) {
        auto victim = cache.end();
        for (auto c = cache.begin(); c != cache.end(); ++c)
          if (!c->second.pinned && c->second.inflight == 0 && c != it &&
              (victim == cache.end() || c->second.last_use < victim->second.last_use))
            victim = c;
        if (victim == cache.end()) break;
        rt.forget_round(victim->second.prep, graveyard);
        cache.erase(victim);
        ++evictions;
      }
    }
    return it;
  };
  // Worker thread (async_plan): plans and uploads member sets off the
  // dispatch path; the loop picks them up between dispatches.
  std::mutex wmu;
  std::condition_variable wcv;
  std::deque<std::vector<int>> wtodo;
  std::vector<std::pair<std::vector<int>, std::pair<Prepared*, double>>> wdone;
  std::map<std::vector<int>, bool> wqueued;
  std::string werr;
  bool wstop = false;
  std::thread worker;
  if (cfg->async_plan) {
    worker = std::thread([&]() {
      try {
        cuda_check(cudaSetDevice(rt.device), "cudaSetDevice");
        for (;;) {
          std::vector<int> key;
          {
            std::unique_lock<std::mutex> lk(wmu);
            wcv.wait(lk, [&] { return wstop || !wtodo.empty(); });
            if (wstop) return;
            key = std::move(wtodo.front());
            wtodo.pop_front();
          }
          auto pp = plan_members(key);
          std::lock_guard<std::mutex> lk(wmu);
          wdone.emplace_back(std::move(key), pp);
        }
      } catch (const std::exception& e) {
        std::lock_guard<std::mutex> lk(wmu);
        werr = e.what();
      }
    });
  }
  struct StopWorker {
    std::thread& w;
    std::mutex& mu;
    std::condition_variable& cv;
    bool& stop;
    ~StopWorker() {
      if (!w.joinable()) return;
      {
        std::lock_guard<std::mutex> lk(mu);
        stop = true;
      }
      cv.notify_all();
      w.join();
    }
  } stop_worker{worker, wmu, wcv, wstop};
  // Pre-warm: every formable member set (one variant or none per tenant) when
  // there are at most cfg->prewarm of them -- the steady state the
  // reference's cache converges to ("cache super-kernels as
  // workloads stabilize") -- else the single-tenant sets and the full set.
  if (cfg->prewarm) {
    size_t combos = 1;
    for (const T& t : ts) combos = std::min<size_t>(combos * (t.variants.size() + 1), size_t{1} << 40);
    if (combos - 1 <= static_cast<size_t>(cfg->prewarm)) {
      for (size_t c = 1; c < combos; ++c) {
        size_t x = c;
        std::vector<int> key;
        for (size_t i = 0; i < n; ++i) {
          const size_t k = x % (ts[i].variants.size() + 1);
          x /= ts[i].variants.size() + 1;
          if (k) key.push_back(ts[i].variants[k - 1].second);
        }
        if (!cache.count(key)) insert(key, plan_members(key), true);
      }
    } else {
      std::vector<int> full;
      for (const T& t : ts) {
        for (const auto& [b, id] : t.variants)
          if (!cache.count({id})) insert({id}, plan_members({id}), true);
        full.push_back(t.variants.back().second);
      }
      if (!cache.count(full)) insert(full, plan_members(full), false);
    }
  } else if (cfg->async_plan) {
    for (const T& t : ts)
      for (const auto& [b, id] : t.variants)
        if (!cache.count({id})) insert({id}, plan_members({id}), true);
  }
  std::vector<cudaEvent_t> pool;
  auto get_event = [&]() {
    if (!pool.empty()) {
      cudaEvent_t e = pool.back();
      pool.pop_back();
      return e;
    }
    cudaEvent_t e;
    cuda_check(cudaEventCreate(&e), "cudaEventCreate");
    return e;
  };
  std::deque<ServeRound> inflight;
  std::vector<gm_dispatch_event> trace;
  std::vector<double> lat_ms;
  int64_t queries = 0, rounds = 0, dispatched_queries = 0, slo_miss = 0, flops_done = 0, h2d = 0, d2h = 0;
  double round_ms_sum = 0;
  double predicted_s = 0;  // EWMA of measured round device time (SLO trigger)
  int evicted = 0;
  uint64_t evicted_mask = 0;
  // contiguous runs of a tenant's query slots: copy(dev offset, host offset, bytes)
  auto for_runs = [](const T& t, const std::vector<ServeQuery>& qs, int64_t qbytes, auto&& copy) {
    size_t j = 0;
    while (j < qs.size()) {
      const int64_t slot0 = qs[j].seq % t.slots;
      size_t k = j + 1;
      while (k < qs.size() && qs[k].seq % t.slots == slot0 + static_cast<int64_t>(k - j)) ++k;
      copy(static_cast<int64_t>(j) * qbytes, slot0 * qbytes, static_cast<int64_t>(k - j) * qbytes);
      j = k;
    }
  };
  const auto t0 = std::chrono::steady_clock::now();

  for (;;) {
    int64_t now = since(t0);
    if (cfg->async_plan) {  // member sets the worker finished
      std::lock_guard<std::mutex> lk(wmu);
      if (!werr.empty()) throw std::runtime_error("serve: background planning failed: " + werr);
      for (auto& [key, pp] : wdone) {
        wqueued.erase(key);
        if (!cache.count(key)) insert(key, pp, false);
      }
      wdone.clear();
    }
    // arrivals (stop admitting at the end of the window)
    for (T& t : ts) {
      if (!t.delayed.empty() && t.live) {
        auto keep = t.delayed.begin();
        for (int64_t a : t.delayed)
          if (a <= now)
            t.push(a);
          else
            *keep++ = a;
        t.delayed.erase(keep, t.delayed.end());
      }
      if (!t.live || t.rate <= 0) continue;
      while (t.next_arrival <= now && t.next_arrival < duration_ns) {
        t.push(t.next_arrival);
        t.next_arrival += draw(t);
      }
    }
    // completions, in dispatch order
    while (!inflight.empty() && cudaEventQuery(inflight.front().ev2) == cudaSuccess) {
      ServeRound r = std::move(inflight.front());
      inflight.pop_front();
      const int64_t done = since(t0);
      float ms = 0;
      cuda_check(cudaEventElapsedTime(&ms, r.ev0, r.ev1), "cudaEventElapsedTime");
      for (cudaEvent_t e : {r.ev0, r.ev1, r.ev2})
        if (e) pool.push_back(e);
      {
        double planned = 0;
        bool singles = true;
        for (const auto& key : r.keys) {
          auto it = cache.find(key);
          if (it == cache.end()) continue;
          --it->second.inflight;
          planned += it->second.planned_s;
          singles = singles && key.size() == 1;
          if (r.keys.size() == 1) {  // a program timed alone
            Prepared& pr = *it->second.prep;
            pr.measured_s = pr.measured_s > 0 ? 0.7 * pr.measured_s + 0.3 * ms * 1e-3 : ms * 1e-3;
          }
        }
        if (planned > 0 && (r.keys.size() == 1 || singles)) {
          double& ratio = rt.serve_ratio[singles ? 0 : 1];
          ratio = 0.9 * ratio + 0.1 * (ms * 1e-3 / planned);
        }
      }
      round_ms_sum += ms;
      {
        gm_dispatch_event ev{};
        ev.start_ns = r.dispatch_ns;
        ev.end_ns = done;
        ev.device_ms = ms;
        ev.flops = r.flops;
        for (auto& m : r.members) ev.queries += static_cast<int32_t>(m.second.size());
        ev.tenants = static_cast<int32_t>(r.members.size());
        ev.launches = r.launches;
        ev.tiles = r.tiles;
        trace.push_back(ev);
      }
      predicted_s = rounds == 1 && predicted_s == 0 ? ms * 1e-3 : 0.8 * predicted_s + 0.2 * ms * 1e-3;
      for (auto& [ti, qs] : r.members) {
        T& t = ts[ti];
        // a degraded tenant's completion is observed exec x slowdown after its
        // dispatch (completion_with_degradation, sim.cpp:105-110)
        const bool deg = static_cast<int>(ti) == deg_t && r.dispatch_ns >= deg_start_ns && cfg->degrade_slowdown > 1.0;
        const double exec_s = ms * 1e-3 * (deg ? cfg->degrade_slowdown : 1.0);
        const int64_t seen = deg ? done + std::llround(ms * 1e6 * (cfg->degrade_slowdown - 1.0)) : done;
        for (const ServeQuery& q : qs) {
          const double l = (seen - q.arrival_ns) * 1e-6;
          if (q.arrival_ns >= warmup_ns && seen <= duration_ns) {
            lat_ms.push_back(l);
            ++queries;
            flops_done += t.flops;
            if (l * 1e-3 > t.slo) ++slo_miss;
          }
          if (t.rate <= 0 && t.live && seen < duration_ns) {  // closed loop: the next query
            if (seen <= done)
              t.push(seen);
            else
              t.delayed.push_back(seen);
          }
        }
        if (!health[ti].evicted) observe(health[ti], exec_s);
      }
      if (ctx->det.evict_stragglers) {
        for (int s : stragglers(health, ctx->det.threshold_ratio, ctx->det.min_observations)) {
          health[s].evicted = true;  // terminal (scheduler.cpp:225-244): pending queries are cancelled
          ts[s].live = false;
          ts[s].pending.clear();
          ts[s].delayed.clear();
          ++evicted;
          evicted_mask |= 1ull << std::min<int>(s, 63);
        }
      }
      now = since(t0);
    }
    size_t pending = 0, live = 0;
    int64_t oldest = INT64_MAX;
    bool slo_due = false;
    const int64_t pred_ns = to_ns(predicted_s * (1.0 + ctx->pol.slo_safety_margin));
    for (T& t : ts) {
      if (!t.live) continue;
      ++live;
      pending += t.pending.size();
      if (!t.pending.empty()) {
        oldest = std::min(oldest, t.pending.front().arrival_ns);
        if (t.pending.front().arrival_ns + to_ns(t.slo) - pred_ns <= now) slo_due = true;
      }
    }
    if (now >= duration_ns && inflight.empty() && (pending == 0 || now >= duration_ns + to_ns(1.0))) break;
    if (static_cast<int>(inflight.size()) < depth && pending > 0) {
      const size_t target = ctx->pol.target_batch > 0 ? static_cast<size_t>(ctx->pol.target_batch) : live;
      if (pending >= target || now - oldest >= max_wait_ns || slo_due || now >= duration_ns) {
        // dynamic batch per tenant: up to its largest variant, the smallest variant that holds them
        std::vector<int> key;
        ServeRound r;
        for (size_t i = 0; i < n; ++i) {
          T& t = ts[i];
          if (!t.live || t.pending.empty()) continue;
          const int bmax = t.variants.back().first;
          const int q = static_cast<int>(std::min<size_t>(t.pending.size(), static_cast<size_t>(bmax)));
          int rtid = t.variants.back().second;
          for (auto& [b, id] : t.variants)
            if (b >= q) {
              rtid = id;
              break;
            }
          key.push_back(rtid);
          std::vector<ServeQuery> qs(t.pending.begin(), t.pending.begin() + q);
          t.pending.erase(t.pending.begin(), t.pending.begin() + q);
          dispatched_queries += q;
          r.flops += static_cast<double>(q) * static_cast<double>(t.flops);
          r.members.emplace_back(static_cast<int>(i), std::move(qs));
        }
        // the member set's round program, or (async planning, first sighting)
        // its members' single-tenant rounds while the worker prepares it
        std::vector<Cached*> progs;
        auto it = cache.find(key);
        if (it != cache.end()) {
          ++plan_hits;
          progs.push_back(&it->second);
          r.keys.push_back(key);
        } else if (cfg->async_plan) {
          ++plan_misses;
          ++fallbacks;
          // admission on the second sighting (a set seen once rarely recurs
          // among many tenants; padding serves it meanwhile)
          if (++misses_of[key] >= 2) {
            {
              std::lock_guard<std::mutex> lk(wmu);
              if (!wqueued.count(key)) {
                wqueued[key] = true;
                wtodo.push_back(key);
              }
            }
            wcv.notify_one();
            misses_of.erase(key);
          }
          if (misses_of.size() > 4096) misses_of.clear();
          // Meanwhile: (a) the cached set expected shortest (measured device
          // time, else its plan scaled by the measured/planned ratio) among
          // those holding every member tenant at a batch variant >= its
          // queries (padding: other tenants and larger batches ride along;
          // only the members' rows are copied), or (b) a cover by cached
          // sub-sets, largest first, then single-tenant sets, back to back --
          // whichever is expected shorter.
          const std::vector<int>* pad = nullptr;
          double pad_s = 0;
          for (auto& [k2, c2] : cache) {
            if (pad && expect_s(c2) >= pad_s) continue;
            bool covers = true;
            for (int id : key) {
              const auto [lt, b] = var_of.at(id);
              bool held = false;
              for (int id2 : k2) {
                const auto [lt2, b2] = var_of.at(id2);
                if (lt2 == lt && b2 >= b) {
                  held = true;
                  break;
                }
              }
              if (!held) {
                covers = false;
                break;
              }
            }
            if (covers) {
              pad = &k2;
              pad_s = expect_s(c2);
            }
          }
          std::vector<const std::vector<int>*> cover;
          double cover_s = 0;
          std::vector<int> rest = key;
          std::vector<std::pair<size_t, const std::vector<int>*>> cand;
          for (auto& [k2, c2] : cache)
            if (k2.size() > 1 && k2.size() < key.size()) cand.emplace_back(k2.size(), &k2);
          std::sort(cand.begin(), cand.end(), [](const auto& a, const auto& b) { return a.first > b.first; });
          for (const auto& [sz, k2] : cand) {
            if (sz > rest.size()) continue;
            bool sub = true;
            for (int id : *k2)
              if (std::find(rest.begin(), rest.end(), id) == rest.end()) {
                sub = false;
                break;
              }
            if (!sub) continue;
            cover.push_back(k2);
            rest.erase(std::remove_if(rest.begin(), rest.end(),
                                      [&](int id) { return std::find(k2->begin(), k2->end(), id) != k2->end(); }),
                       rest.end());
          }
          for (int id : rest) cover.push_back(&cache.find({id})->first);
          for (const auto* k2 : cover) cover_s += expect_s(cache.at(*k2));
          if (pad && pad_s <= cover_s) {
            ++padded;
            progs.push_back(&cache.at(*pad));
            r.keys.push_back(*pad);
          } else {
            for (const auto* k2 : cover) {
              progs.push_back(&cache.at(*k2));
              r.keys.push_back(*k2);
            }
          }
        } else {
          ++plan_misses;
          auto it2 = insert(key, plan_members(key), false);
          progs.push_back(&it2->second);
          r.keys.push_back(key);
        }
        if (predicted_s == 0) predicted_s = progs.front()->planned_s;
        for (size_t m = 0; m < r.members.size(); ++m) {  // this dispatch's query inputs
          const T& t = ts[r.members[m].first];
          if (!t.hin) continue;
          for_runs(t, r.members[m].second, t.in_q, [&](int64_t doff, int64_t hoff, int64_t bytes) {
            cuda_check(cudaMemcpyAsync(t.dx + doff, t.hin + hoff, bytes, cudaMemcpyHostToDevice, stream), "H2D");
            h2d += bytes;
          });
        }
        r.ev0 = get_event();
        r.ev1 = get_event();
        r.ev2 = get_event();
        r.dispatch_ns = now;
        cuda_check(cudaEventRecord(r.ev0, stream), "cudaEventRecord");
        for (Cached* c : progs) {
          c->last_use = ++use_clock;
          ++c->inflight;
          r.tiles += c->prep->n_tiles;
          rt.launch(*c->prep, stream);
          ++r.launches;  // round programs (a layer-0 pre-pass rides with its program)
        }
        cuda_check(cudaEventRecord(r.ev1, stream), "cudaEventRecord");
        for (size_t m = 0; m < r.members.size(); ++m) {  // and results
          const T& t = ts[r.members[m].first];
          if (!t.hout) continue;
          for_runs(t, r.members[m].second, t.out_q, [&](int64_t doff, int64_t hoff, int64_t bytes) {
            cuda_check(cudaMemcpyAsync(t.hout + hoff, t.dy + doff, bytes, cudaMemcpyDeviceToHost, stream), "D2H");
            d2h += bytes;
          });
        }
        cuda_check(cudaEventRecord(r.ev2, stream), "cudaEventRecord");
        inflight.push_back(std::move(r));
        ++rounds;
        continue;
      }
    }
    // nothing to do right now: yield briefly (completion polling granularity)
    std::this_thread::yield();
  }
  cuda_check(cudaStreamSynchronize(stream), "cudaStreamSynchronize");
  for (cudaEvent_t e : pool) cudaEventDestroy(e);
  for (Prepared& p : graveyard) p.release();
  rt.serve_trace = std::move(trace);

  std::memset(out, 0, sizeof(*out));
  out->queries = queries;
  out->rounds = rounds;
  out->dispatched_queries = dispatched_queries;
  out->window_s = cfg->duration - cfg->warmup;
  out->tflops = static_cast<double>(flops_done) / out->window_s / 1e12;
  out->qps = static_cast<double>(queries) / out->window_s;
  if (!lat_ms.empty()) {
    out->p50_ms = nearest_rank(lat_ms, 50.0);
    out->p99_ms = nearest_rank(lat_ms, 99.0);
    out->max_ms = *std::max_element(lat_ms.begin(), lat_ms.end());
    double sum = 0;
    for (double l : lat_ms) sum += l;
    out->mean_ms = sum / static_cast<double>(lat_ms.size());
    out->slo_violation_frac = static_cast<double>(slo_miss) / static_cast<double>(lat_ms.size());
  }
  out->mean_queries_per_round = rounds ? static_cast<double>(dispatched_queries) / rounds : 0;
  out->mean_round_ms = rounds ? round_ms_sum / rounds : 0;
  out->plan_hits = plan_hits;
  out->plan_misses = plan_misses;
  out->evicted = evicted;
  out->evicted_mask = evicted_mask;
  out->plan_evictions = evictions;
  out->plan_fallbacks = fallbacks;
  out->plans_cached = static_cast<int64_t>(cache.size());
  out->plan_padded = padded;
  out->h2d_bytes = h2d;
  out->d2h_bytes = d2h;
  if (n_lat) *n_lat = lat_ms.size();
  if (latencies_ms && cap) std::copy(lat_ms.begin(), lat_ms.begin() + std::min(cap, lat_ms.size()), latencies_ms);
  GM_CTX_API_END(ctx)
}
