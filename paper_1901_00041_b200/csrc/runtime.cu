// B200 runtime: per-GPU context, tenant registration (member descriptors with
// TMA maps), plan preparation (device tile tables, cached per member list) and
// super-kernel launch.  C-ABI entry points for the device side live here.
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstring>
#include <string>
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
uint32_t make_idesc(int n) {
  const uint32_t umma_n = static_cast<uint32_t>(std::min(dev::kBN, (n + 15) / 16 * 16));
  return (1u << 4) | (1u << 7) | (1u << 10) | ((umma_n >> 3) << 17) | (static_cast<uint32_t>(dev::kBM >> 4) << 24);
}

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

}  // namespace

// One registered (tenant, layer) operator.
struct Operator {
  int kind = GM_LAYER_GEMM;
  Shape shape;      // the GEMM the planner sees (m includes batch)
  Conv conv;
  int batch = 1;
  int slot = -1;    // index into the device MemberDesc array
  bool prepass = false;
  const void* x = nullptr;
  void* scratch = nullptr;  // explicit-im2col rows [M, ldk]
  int64_t ldk = 0;
};

struct Prepared {
  dev::TileEntry* tiles = nullptr;
  int n_tiles = 0;
  std::vector<int> prepass_ops;  // indices into Runtime::flat
};

struct Runtime {
  int device = -1;
  int sms = 0;
  int driver_version = 0;
  EncodeTiledFn encode_tiled = nullptr;
  EncodeIm2colFn encode_im2col = nullptr;
  std::vector<std::vector<int>> tenant_ops;  // tenant -> indices into flat
  std::vector<double> tenant_slo;            // seconds per pass
  std::vector<Operator> flat;
  std::vector<dev::MemberDesc> host_desc;
  dev::MemberDesc* d_desc = nullptr;
  size_t d_cap = 0;
  std::unordered_map<std::string, Prepared> prepared;
  int64_t n_superkernels = 0, n_prepasses = 0, n_tiles = 0;

  ~Runtime() {
    if (device < 0) return;
    cudaSetDevice(device);
    cudaDeviceSynchronize();
    for (auto& [k, p] : prepared) cudaFree(p.tiles);
    for (Operator& op : flat) cudaFree(op.scratch);
    cudaFree(d_desc);
  }

  void init(int dev_index) {
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
    cuda_check(cudaFuncSetAttribute(dev::superkernel, cudaFuncAttributeMaxDynamicSharedMemorySize, dev::kSmemBytes),
               "cudaFuncSetAttribute");
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
  void im2col_map(CUtensorMap* map, const void* x, const Conv& c, int batch) {
    if (!aligned16(x)) throw std::invalid_argument("conv input must be 16-byte aligned");
    const cuuint64_t dims[4] = {static_cast<cuuint64_t>(c.in_channels), static_cast<cuuint64_t>(c.image_w),
                                static_cast<cuuint64_t>(c.image_h), static_cast<cuuint64_t>(batch)};
    const cuuint64_t strides[3] = {static_cast<cuuint64_t>(c.in_channels * 2),
                                   static_cast<cuuint64_t>(c.image_w * c.in_channels * 2),
                                   static_cast<cuuint64_t>(c.image_h * c.image_w * c.in_channels * 2)};
    const int lower[2] = {static_cast<int>(-c.padding), static_cast<int>(-c.padding)};
    const int upper[2] = {static_cast<int>(c.padding - (c.kernel_w - 1)), static_cast<int>(c.padding - (c.kernel_h - 1))};
    const cuuint32_t estr[4] = {1, static_cast<cuuint32_t>(c.stride), static_cast<cuuint32_t>(c.stride), 1};
    const CUresult r = encode_im2col(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void*>(x), dims, strides,
                                     lower, upper, dev::kBK, dev::kBM, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                     CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) throw CudaError("cuTensorMapEncodeIm2col failed (" + std::to_string(int(r)) + ")");
    // Driver <= 13.1 mis-encodes im2col maps of tensors under 128 KiB; clear
    // the offending bit exactly as CUTLASS does (copy_traits_sm90_im2col.hpp).
    const int64_t bytes = static_cast<int64_t>(batch) * c.image_h * c.image_w * c.in_channels * 2;
    if (driver_version <= 13010 && bytes < 131072) reinterpret_cast<uint64_t*>(map)[1] &= ~(1ull << 21);
  }

  int register_tenant(const gm_tenant_desc& t) {
    if (!t.layers || t.n_layers == 0) throw std::invalid_argument("register_tenant: tenant has no layers");
    std::vector<int> ops;
    std::vector<Operator> fresh;
    std::vector<dev::MemberDesc> descs;
    for (size_t i = 0; i < t.n_layers; ++i) {
      const gm_layer_desc& L = t.layers[i];
      Operator op;
      dev::MemberDesc md;
      std::memset(&md, 0, sizeof(md));
      op.kind = L.kind;
      op.x = L.x;
      if (!L.x || !L.w || !L.y) throw std::invalid_argument("register_tenant: null operand pointer");
      if (!aligned16(L.y)) throw std::invalid_argument("register_tenant: output must be 16-byte aligned");
      if (L.kind == GM_LAYER_CONV) {
        op.conv = to_conv(L.conv);
        op.batch = L.batch < 1 ? 1 : L.batch;
        op.shape = with_batch(lower_conv(op.conv), op.batch);
        const Conv& c = op.conv;
        const int64_t K = op.shape.k;
        const int64_t ldw = L.ldw > 0 ? L.ldw : K;
        if (ldw < K) throw std::invalid_argument("register_tenant: ldw < R*S*Cin");
        tiled_map(&md.b, L.w, op.shape.n, K, ldw, dev::kBN);
        const int64_t P = (c.image_h + 2 * c.padding - c.kernel_h) / c.stride + 1;
        const int64_t Q = (c.image_w + 2 * c.padding - c.kernel_w) / c.stride + 1;
        const bool pointwise = c.kernel_h == 1 && c.kernel_w == 1 && c.stride == 1 && c.padding == 0;
        if (pointwise && c.in_channels % 8 == 0) {
          md.a_mode = dev::kATiled;  // 1x1 stride-1 conv == GEMM over NHWC rows
          tiled_map(&md.a, L.x, op.shape.m, c.in_channels, c.in_channels, dev::kBM);
        } else if (c.in_channels % dev::kBK == 0 && c.kernel_h == c.kernel_w && c.stride <= 8 &&
                   c.padding <= 127 && c.kernel_h - 1 - c.padding <= 128) {
          md.a_mode = dev::kAIm2col;  // implicit GEMM through the TMA im2col unit
          im2col_map(&md.a, L.x, c, op.batch);
          md.pq = static_cast<int32_t>(P * Q);
          md.q = static_cast<int32_t>(Q);
          md.stride = static_cast<int32_t>(c.stride);
          md.pad = static_cast<int32_t>(c.padding);
          md.s_taps = static_cast<int32_t>(c.kernel_w);
          md.c_blocks = static_cast<int32_t>(c.in_channels / dev::kBK);
        } else {
          md.a_mode = dev::kATiled;  // explicit im2col pre-pass, then GEMM
          op.prepass = true;
          op.ldk = (K + 7) / 8 * 8;
          cuda_check(cudaMalloc(&op.scratch, static_cast<size_t>(op.shape.m * op.ldk * 2)), "cudaMalloc(im2col)");
          tiled_map(&md.a, op.scratch, op.shape.m, K, op.ldk, dev::kBM);
        }
      } else if (L.kind == GM_LAYER_GEMM) {
        op.shape = to_shape(L.gemm);
        if (!op.shape.valid()) throw std::invalid_argument("register_tenant: invalid GEMM shape");
        const int64_t ldx = L.ldx > 0 ? L.ldx : op.shape.k;
        const int64_t ldw = L.ldw > 0 ? L.ldw : op.shape.k;
        md.a_mode = dev::kATiled;
        tiled_map(&md.a, L.x, op.shape.m, op.shape.k, ldx, dev::kBM);
        tiled_map(&md.b, L.w, op.shape.n, op.shape.k, ldw, dev::kBN);
      } else {
        throw std::invalid_argument("register_tenant: unknown layer kind");
      }
      if (op.shape.n % 8 != 0) throw std::invalid_argument("register_tenant: output channels must be a multiple of 8");
      if (op.shape.m > int64_t(0xFFFF) * dev::kBM || op.shape.m > INT32_MAX)
        throw std::invalid_argument("register_tenant: M too large for the tile table");
      md.y = static_cast<__nv_bfloat16*>(L.y);
      md.ldy = op.shape.n;
      md.m = static_cast<int32_t>(op.shape.m);
      md.n = static_cast<int32_t>(op.shape.n);
      md.k_blocks = static_cast<int32_t>((op.shape.k + dev::kBK - 1) / dev::kBK);
      md.idesc = make_idesc(static_cast<int>(op.shape.n));
      md.relu = L.relu ? 1 : 0;
      op.slot = static_cast<int>(host_desc.size() + descs.size());
      if (op.slot > 0xFFFF) throw std::invalid_argument("register_tenant: too many registered operators");
      descs.push_back(md);
      fresh.push_back(op);
    }
    // Commit: grow the device descriptor array and upload.
    const size_t need_n = host_desc.size() + descs.size();
    if (need_n > d_cap) {
      size_t cap = std::max<size_t>(64, d_cap * 2);
      while (cap < need_n) cap *= 2;
      dev::MemberDesc* nd = nullptr;
      cuda_check(cudaMalloc(&nd, cap * sizeof(dev::MemberDesc)), "cudaMalloc(descriptors)");
      if (d_desc) {
        cuda_check(cudaDeviceSynchronize(), "cudaDeviceSynchronize");
        cudaFree(d_desc);
      }
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
    tenant_ops.push_back(std::move(ops));
    tenant_slo.push_back(t.slo_latency > 0 ? t.slo_latency : 0.1);
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
    for (int f : members) {
      const Operator& op = flat[f];
      const int64_t mt = (op.shape.m + dev::kBM - 1) / dev::kBM;
      const int64_t nt = (op.shape.n + dev::kBN - 1) / dev::kBN;
      for (int64_t a = 0; a < mt; ++a)
        for (int64_t b = 0; b < nt; ++b)
          table.push_back(dev::TileEntry{static_cast<uint16_t>(op.slot), 0, static_cast<uint16_t>(a),
                                         static_cast<uint16_t>(b)});
      if (op.prepass) p.prepass_ops.push_back(f);
    }
    p.n_tiles = static_cast<int>(table.size());
    cuda_check(cudaMalloc(&p.tiles, std::max<size_t>(1, table.size()) * sizeof(dev::TileEntry)), "cudaMalloc(tiles)");
    cuda_check(cudaMemcpy(p.tiles, table.data(), table.size() * sizeof(dev::TileEntry), cudaMemcpyHostToDevice),
               "upload tile table");
    return prepared.emplace(key, std::move(p)).first->second;
  }

  int launch(Prepared& p, cudaStream_t stream) {
    int launches = 0;
    for (int f : p.prepass_ops) {
      const Operator& op = flat[f];
      const Conv& c = op.conv;
      const int P = static_cast<int>((c.image_h + 2 * c.padding - c.kernel_h) / c.stride + 1);
      const int Q = static_cast<int>((c.image_w + 2 * c.padding - c.kernel_w) / c.stride + 1);
      const int64_t total = op.shape.m * op.ldk;
      const int grid = static_cast<int>(std::min<int64_t>((total + 255) / 256, int64_t(sms) * 16));
      dev::im2col_prepass<<<grid, 256, 0, stream>>>(
          static_cast<const __nv_bfloat16*>(op.x), static_cast<__nv_bfloat16*>(op.scratch), op.batch,
          static_cast<int>(c.image_h), static_cast<int>(c.image_w), static_cast<int>(c.in_channels),
          static_cast<int>(c.kernel_h), static_cast<int>(c.kernel_w), static_cast<int>(c.stride),
          static_cast<int>(c.padding), P, Q, static_cast<int>(op.ldk));
      cuda_check(cudaGetLastError(), "launch im2col_prepass");
      ++launches;
      ++n_prepasses;
    }
    const int grid = std::max(1, std::min(p.n_tiles, sms));
    dev::superkernel<<<grid, dev::kThreads, dev::kSmemBytes, stream>>>(d_desc, p.tiles, p.n_tiles);
    cuda_check(cudaGetLastError(), "launch superkernel");
    ++launches;
    ++n_superkernels;
    n_tiles += p.n_tiles;
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
    if (cuda_device >= 0) {
      ctx->rt = new Runtime();
      ctx->rt->init(cuda_device);
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
  GM_API_END
}

int gm_ctx_cache(gm_ctx* ctx, gm_cache** c) {
  GM_API_BEGIN
  if (!ctx || !c) throw std::invalid_argument("null argument");
  *c = &ctx->cache;
  GM_API_END
}

int gm_ctx_device_spec(const gm_ctx* ctx, gm_device_spec* out) {
  GM_API_BEGIN
  if (!ctx || !out) throw std::invalid_argument("null argument");
  *out = from_device(ctx->dev);
  GM_API_END
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
  GM_API_END
}

int gm_layer_shape(gm_ctx* ctx, int32_t tenant, int32_t layer, gm_gemm_shape* out) {
  GM_API_BEGIN
  if (!out) throw std::invalid_argument("null argument: out");
  *out = from_shape(runtime_of(ctx).op_of(tenant, layer).shape);
  GM_API_END
}

int gm_tenant_count(const gm_ctx* ctx, int32_t* n) {
  GM_API_BEGIN
  if (!ctx || !n) throw std::invalid_argument("null argument");
  *n = ctx->rt ? static_cast<int32_t>(ctx->rt->tenant_ops.size()) : 0;
  GM_API_END
}

int gm_prepare(gm_ctx* ctx, const gm_plans* p, size_t i) {
  GM_API_BEGIN
  if (!p || i >= p->plans.size()) throw std::invalid_argument("plan index out of range");
  Runtime& rt = runtime_of(ctx);
  cuda_check(cudaSetDevice(rt.device), "cudaSetDevice");
  rt.prepare(members_of(rt, p->plans[i]));
  GM_API_END
}

int gm_dispatch(gm_ctx* ctx, const gm_plans* p, size_t i, uint64_t stream, double* planned_s, int* cache_hit) {
  GM_API_BEGIN
  if (!p || i >= p->plans.size()) throw std::invalid_argument("plan index out of range");
  Runtime& rt = runtime_of(ctx);
  const Plan& plan = p->plans[i];
  Prepared& prep = rt.prepare(members_of(rt, plan));
  const int64_t misses = ctx->cache.c.misses;
  const double dur = charge(plan, ctx->cache.c, ctx->dev);
  rt.launch(prep, reinterpret_cast<cudaStream_t>(stream));
  if (planned_s) *planned_s = dur;
  if (cache_hit) *cache_hit = ctx->cache.c.misses == misses ? 1 : 0;
  GM_API_END
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
  GM_API_END
}

int gm_members_launch_count(gm_ctx* ctx, const int32_t* tenants, const int32_t* layers, size_t n, int32_t* launches) {
  GM_API_BEGIN
  if (n == 0 || !tenants || !layers || !launches) throw std::invalid_argument("empty dispatch");
  Runtime& rt = runtime_of(ctx);
  int l = 1;
  for (size_t j = 0; j < n; ++j) l += rt.op_of(tenants[j], layers[j]).prepass ? 1 : 0;
  *launches = l;
  GM_API_END
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
  GM_API_END
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
  GM_API_END
}

int gm_dispatch_plans(gm_ctx* ctx, const gm_plans* p, uint64_t stream, int32_t* launches) {
  GM_API_BEGIN
  if (!p) throw std::invalid_argument("null argument: plans");
  Runtime& rt = runtime_of(ctx);
  int l = 0;
  for (const Plan& plan : p->plans) l += rt.launch(rt.prepare(members_of(rt, plan)), reinterpret_cast<cudaStream_t>(stream));
  if (launches) *launches = l;
  GM_API_END
}

int gm_ctx_launch_stats(const gm_ctx* ctx, int64_t* superkernels, int64_t* prepasses, int64_t* tiles) {
  GM_API_BEGIN
  if (!ctx) throw std::invalid_argument("null context");
  const Runtime* rt = ctx->rt;
  if (superkernels) *superkernels = rt ? rt->n_superkernels : 0;
  if (prepasses) *prepasses = rt ? rt->n_prepasses : 0;
  if (tiles) *tiles = rt ? rt->n_tiles : 0;
  GM_API_END
}

}  // extern "C"
