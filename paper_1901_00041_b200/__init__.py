"""B200-native space-time multiplexing path of arXiv:1901.00041 ("gpumux").

Host planner + C-ABI + sm_100a tcgen05 super-kernel.  See DESIGN.md.
"""
from .scheduler import (BatchPolicy, ConvSpec, DeviceSpec, GemmShape, KernelCost, KernelGroup, KernelRequest,
                        RequestQueue, SuperKernel, SuperKernelCache, TenantHealth, b200_profile, batch_inputs,
                        detect_stragglers, dispatch_cost, dispatch_duration, evict, form_batches, gemm_bytes,
                        gemm_flops, geomean, im2col_gemm_dims, percentile_nearest_rank, plan_super_kernel,
                        record_latency, shape_key, slo_headroom, thread_blocks, to_ns, to_seconds, v100_profile)

__all__ = [n for n in dir() if not n.startswith("_")]
