"""Tenant workloads: the reference presets and real-layer model graphs.

* ``reference_presets()`` restates the reference's shipped presets
  (proj/src/workload.cpp:15-95): ``rnn-matvec``, ``resnet18-conv2_2``,
  ``square-256`` and the stylised ``resnet50`` / ``mobilenetv2`` GEMM lists.
  They are plan-parity inputs (GemmShape lists), not executable graphs.
* The model builders return executable operator lists with real
  ConvSpecs (torchvision layer definitions), which the reference lacks
  (SURVEY §8(d)): ResNet-18/50, VGG-16, MobileNet-v2 (depthwise layers are
  tagged ``dwconv``: the super-kernel's CUDA-core depthwise tile type), BERT-base
  projection/FFN GEMMs.  Convs are listed in forward order; a bottleneck's
  downsample follows its conv3, a basic block's follows its conv2.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import List, Optional

from .scheduler import ConvSpec, GemmShape, batch_inputs, im2col_gemm_dims


@dataclass(frozen=True)
class WorkloadPreset:
    """workload.hpp:24-29."""
    name: str
    layers: tuple
    weights_bytes: float
    slo_latency: float


def reference_presets() -> List[WorkloadPreset]:
    """The reference's preset table (workload.cpp:15-95), restated."""
    out = [
        WorkloadPreset("rnn-matvec", (GemmShape(512, 1, 512),), 512.0 * 512 * 4, 0.05),
        WorkloadPreset("resnet18-conv2_2", (GemmShape(256, 128, 1152),), 1152.0 * 128 * 4, 0.05),
        WorkloadPreset("square-256", (GemmShape(256, 256, 256),), 256.0 * 256 * 4, 0.05),
    ]
    l = [GemmShape(1024, 64, 147)]
    for _ in range(3):
        l += [GemmShape(256, 64, 64), GemmShape(256, 64, 576), GemmShape(256, 256, 64)]
    l.append(GemmShape(256, 256, 64))
    for _ in range(4):
        l += [GemmShape(64, 128, 256), GemmShape(64, 128, 1152), GemmShape(64, 512, 128)]
    l.append(GemmShape(64, 512, 256))
    for _ in range(6):
        l += [GemmShape(16, 256, 512), GemmShape(16, 256, 2304), GemmShape(16, 1024, 256)]
    l.append(GemmShape(16, 1024, 512))
    for _ in range(3):
        l += [GemmShape(4, 512, 1024), GemmShape(4, 512, 4608), GemmShape(4, 2048, 512)]
    l += [GemmShape(4, 2048, 1024), GemmShape(1, 1000, 2048)]
    out.append(WorkloadPreset("resnet50", tuple(l), 102.4e6, 0.040))
    m = [GemmShape(1024, 32, 27), GemmShape(256, 96, 16), GemmShape(256, 96, 9), GemmShape(256, 24, 96)]
    for _ in range(2):
        m += [GemmShape(64, 144, 24), GemmShape(64, 144, 9), GemmShape(64, 32, 144)]
    for _ in range(3):
        m += [GemmShape(16, 192, 32), GemmShape(16, 192, 9), GemmShape(16, 64, 192)]
    for _ in range(2):
        m += [GemmShape(4, 384, 64), GemmShape(4, 384, 9), GemmShape(4, 96, 384)]
    for _ in range(2):
        m += [GemmShape(4, 576, 96), GemmShape(4, 576, 9), GemmShape(4, 160, 576)]
    m += [GemmShape(4, 960, 160), GemmShape(4, 960, 9), GemmShape(4, 320, 960), GemmShape(4, 1280, 320),
          GemmShape(1, 1000, 1280)]
    out.append(WorkloadPreset("mobilenetv2", tuple(m), 13.6e6, 0.020))
    return out


def find_preset(name: str) -> Optional[WorkloadPreset]:
    for p in reference_presets():
        if p.name == name:
            return p
    return None


# ---------------------------------------------------------------- real graphs

ACT_NONE, ACT_RELU, ACT_RELU6, ACT_GELU = 0, 1, 2, 3  # gm_activation
POOLS = ("maxpool", "avgpool")
WINDOWED = ("conv", "dwconv") + POOLS


@dataclass(frozen=True)
class Layer:
    """One operator of a tenant graph.

    conv/dwconv/maxpool/avgpool: ``conv`` holds the ConvSpec (per image; a
          pool's kernel is its window, in == out channels).
    gemm: ``rows`` rows per query (1 for a classifier, seq_len for BERT),
          ``n`` outputs, ``k`` inner dimension.

    Dataflow: ``src`` names the earlier layer whose output this layer reads
    (None = its own input buffer, e.g. the tenant's query batch), starting at
    column ``src_col`` of that output viewed as [rows, -1] (BERT's attention
    output projection reads the V third of the qkv projection); ``res`` names
    the earlier layer added before the activation ``act`` (residual blocks).
    """
    name: str
    kind: str
    conv: Optional[ConvSpec] = None
    rows: int = 0
    n: int = 0
    k: int = 0
    act: int = ACT_NONE
    src: Optional[int] = None
    res: Optional[int] = None
    src_col: int = 0

    def gemm_shape(self, batch: int = 1) -> GemmShape:
        if self.kind == "dwconv" or self.kind in POOLS:
            # the reference's model of a per-channel op: K = R*S (workload.cpp:66)
            s = batch_inputs(im2col_gemm_dims(self.conv), batch)
            return GemmShape(s.m, s.n, self.conv.kernel_h * self.conv.kernel_w)
        if self.kind == "conv":
            return batch_inputs(im2col_gemm_dims(self.conv), batch)
        return GemmShape(self.rows * batch, self.n, self.k)

    def flops(self, batch: int = 1) -> int:
        """Multiply-add FLOPs (2mnk); pools do no multiply-adds and count 0."""
        if self.kind in POOLS:
            return 0
        s = self.gemm_shape(batch)  # dwconv: per-channel filter, K = R*S
        return 2 * s.m * s.n * s.k

    def compulsory_bytes(self, batch: int = 1, elem: int = 2) -> int:
        """Implicit-GEMM bf16 traffic: input + weights + output;
        plus the residual read when one is fused."""
        s = self.gemm_shape(batch)
        extra = s.m * s.n if self.res is not None else 0
        if self.kind in WINDOWED:
            c = self.conv
            if self.kind in POOLS:
                w = 0
            else:
                w = c.out_channels * c.kernel_h * c.kernel_w * (1 if self.kind == "dwconv" else c.in_channels)
            return elem * (batch * c.image_h * c.image_w * c.in_channels + w + s.m * s.n + extra)
        return elem * (s.m * s.k + s.n * s.k + s.m * s.n + extra)


def _conv(name, hw, cin, cout, r, stride, pad, act=ACT_NONE, src=None, res=None):
    return Layer(name, "conv", ConvSpec(hw, hw, r, r, cin, cout, stride, pad), act=act, src=src, res=res)


def _pool(name, kind, hw, c, r, stride, pad, src):
    return Layer(name, kind, ConvSpec(hw, hw, r, r, c, c, stride, pad), src=src)


def resnet50(image: int = 224, classifier: bool = True) -> List[Layer]:
    """torchvision resnet50 (v1.5: stride on the 3x3) as a dataflow graph:
    stem conv + relu, maxpool 3x3/2, 16 bottlenecks (conv1/conv2 + relu;
    relu(conv3 + identity), or relu(downsample + conv3) with the add fused into
    the downsample, which is listed after conv3), global avgpool, fc.
    BatchNorm is folded into the (synthetic) weights."""
    L = [_conv("conv1", image, 3, 64, 7, 2, 3, act=ACT_RELU)]
    hw = (image + 6 - 7) // 2 + 1
    L.append(_pool("maxpool", "maxpool", hw, 64, 3, 2, 1, src=0))
    hw = (hw + 2 - 3) // 2 + 1
    cin, block_in = 64, 1
    for stage, (width, blocks, stride) in enumerate([(64, 3, 1), (128, 4, 2), (256, 6, 2), (512, 3, 2)], start=1):
        out = width * 4
        for b in range(blocks):
            s = stride if b == 0 else 1
            p = f"layer{stage}.{b}"
            L.append(_conv(p + ".conv1", hw, cin, width, 1, 1, 0, act=ACT_RELU, src=block_in))
            L.append(_conv(p + ".conv2", hw, width, width, 3, s, 1, act=ACT_RELU, src=len(L) - 1))
            ohw = (hw + 2 - 3) // s + 1
            if b == 0:
                L.append(_conv(p + ".conv3", ohw, width, out, 1, 1, 0, src=len(L) - 1))
                L.append(_conv(p + ".downsample", hw, cin, out, 1, s, 0, act=ACT_RELU, src=block_in, res=len(L) - 1))
            else:
                L.append(_conv(p + ".conv3", ohw, width, out, 1, 1, 0, act=ACT_RELU, src=len(L) - 1, res=block_in))
            block_in = len(L) - 1
            hw, cin = ohw, out
    if classifier:
        L.append(_pool("avgpool", "avgpool", hw, cin, hw, 1, 0, src=block_in))
        L.append(Layer("fc", "gemm", rows=1, n=1000, k=2048, src=len(L) - 1))
    return L


def resnet18(image: int = 224, classifier: bool = True) -> List[Layer]:
    """torchvision resnet18 as a dataflow graph (basic blocks: relu(conv2 +
    identity), or relu(downsample + conv2) fused into the downsample); at
    image=128 layer2.* is the paper's conv2_2 (256,128,1152)."""
    L = [_conv("conv1", image, 3, 64, 7, 2, 3, act=ACT_RELU)]
    hw = (image + 6 - 7) // 2 + 1
    L.append(_pool("maxpool", "maxpool", hw, 64, 3, 2, 1, src=0))
    hw = (hw + 2 - 3) // 2 + 1
    cin, block_in = 64, 1
    for stage, (width, stride) in enumerate([(64, 1), (128, 2), (256, 2), (512, 2)], start=1):
        for b in range(2):
            s = stride if b == 0 else 1
            p = f"layer{stage}.{b}"
            L.append(_conv(p + ".conv1", hw, cin, width, 3, s, 1, act=ACT_RELU, src=block_in))
            ohw = (hw + 2 - 3) // s + 1
            if b == 0 and (s != 1 or cin != width):
                L.append(_conv(p + ".conv2", ohw, width, width, 3, 1, 1, src=len(L) - 1))
                L.append(_conv(p + ".downsample", hw, cin, width, 1, s, 0, act=ACT_RELU, src=block_in,
                               res=len(L) - 1))
            else:
                L.append(_conv(p + ".conv2", ohw, width, width, 3, 1, 1, act=ACT_RELU, src=len(L) - 1,
                               res=block_in))
            block_in = len(L) - 1
            hw, cin = ohw, width
    if classifier:
        L.append(_pool("avgpool", "avgpool", hw, cin, hw, 1, 0, src=block_in))
        L.append(Layer("fc", "gemm", rows=1, n=1000, k=512, src=len(L) - 1))
    return L


def vgg16(image: int = 224, classifier: bool = True) -> List[Layer]:
    """torchvision vgg16: 13 convs 3x3 p1 + relu, 2x2 max pools, 3 fc (relu on
    the first two; the flatten reads pool5's NHWC output, adaptive avgpool is
    the identity at 224)."""
    cfg = [64, 64, "M", 128, 128, "M", 256, 256, 256, "M", 512, 512, 512, "M", 512, 512, 512, "M"]
    L, hw, cin, i = [], image, 3, 0
    for v in cfg:
        src = len(L) - 1 if L else None
        if v == "M":
            L.append(_pool(f"pool{len([x for x in L if x.kind == 'maxpool']) + 1}", "maxpool", hw, cin, 2, 2, 0, src))
            hw //= 2
            continue
        L.append(_conv(f"features.{i}", hw, cin, v, 3, 1, 1, act=ACT_RELU, src=src))
        cin, i = v, i + 1
    if classifier:
        L += [Layer("classifier.0", "gemm", rows=1, n=4096, k=512 * hw * hw, act=ACT_RELU, src=len(L) - 1),
              Layer("classifier.3", "gemm", rows=1, n=4096, k=4096, act=ACT_RELU, src=len(L)),
              Layer("classifier.6", "gemm", rows=1, n=1000, k=4096, src=len(L) + 1)]
    return L


def mobilenet_v2(image: int = 224, classifier: bool = True) -> List[Layer]:
    """torchvision mobilenet_v2 (width 1.0) as a dataflow graph: inverted
    residuals (expand 1x1 + relu6, depthwise 3x3 ``dwconv`` + relu6, linear
    project 1x1, + input when stride 1 and in == out channels), features.18
    1x1 + relu6, global avgpool, classifier."""
    L = [_conv("features.0", image, 3, 32, 3, 2, 1, act=ACT_RELU6)]
    hw = (image + 2 - 3) // 2 + 1
    cin, block_in = 32, 0
    settings = [(1, 16, 1, 1), (6, 24, 2, 2), (6, 32, 3, 2), (6, 64, 4, 2), (6, 96, 3, 1), (6, 160, 3, 2),
                (6, 320, 1, 1)]
    idx = 1
    for t, c, n, s in settings:
        for b in range(n):
            stride = s if b == 0 else 1
            hidden = cin * t
            p = f"features.{idx}"
            src = block_in
            if t != 1:
                L.append(_conv(p + ".expand", hw, cin, hidden, 1, 1, 0, act=ACT_RELU6, src=src))
                src = len(L) - 1
            L.append(Layer(p + ".dw", "dwconv", ConvSpec(hw, hw, 3, 3, hidden, hidden, stride, 1), act=ACT_RELU6,
                           src=src))
            ohw = (hw + 2 - 3) // stride + 1
            residual = block_in if stride == 1 and cin == c else None
            L.append(_conv(p + ".project", ohw, hidden, c, 1, 1, 0, src=len(L) - 1, res=residual))
            block_in = len(L) - 1
            hw, cin, idx = ohw, c, idx + 1
    L.append(_conv("features.18", hw, cin, 1280, 1, 1, 0, act=ACT_RELU6, src=block_in))
    if classifier:
        L.append(_pool("avgpool", "avgpool", hw, 1280, hw, 1, 0, src=len(L) - 1))
        L.append(Layer("classifier.1", "gemm", rows=1, n=1000, k=1280, src=len(L) - 1))
    return L


def bert_base_gemms(seq_len: int = 128, layers: int = 1) -> List[Layer]:
    """BERT-base projection/FFN GEMMs per encoder layer (hidden 768, FFN 3072)
    as a chain: qkv; attn_out reads the V third of qkv's output (the attention
    core softmax(QK^T)V and LayerNorm are not GEMM-shaped tenant operators and
    are out of scope) and adds the layer input; ffn1 + GELU; ffn2 adds
    attn_out's output; the next layer reads ffn2."""
    out = []
    layer_in = None
    for i in range(layers):
        p = f"encoder.{i}"
        base = len(out)
        out += [Layer(p + ".qkv", "gemm", rows=seq_len, n=2304, k=768, src=layer_in),
                Layer(p + ".attn_out", "gemm", rows=seq_len, n=768, k=768, src=base, src_col=1536,
                      res=layer_in),
                Layer(p + ".ffn1", "gemm", rows=seq_len, n=3072, k=768, act=ACT_GELU, src=base + 1),
                Layer(p + ".ffn2", "gemm", rows=seq_len, n=768, k=3072, src=base + 2, res=base + 1)]
        layer_in = base + 3
    return out


def conv2_2() -> List[Layer]:
    """The paper's microbenchmark layer: ResNet-18 conv2_2 at 16x16."""
    return [_conv("conv2_2", 16, 128, 128, 3, 1, 1)]


def table1_layers(preset: str) -> List[Layer]:
    """One tenant's operator for the paper's Table-1 microbenchmarks
    (reference presets, workload.cpp:18-20): ``resnet18-conv2_2`` as the real
    3x3 conv (implicit GEMM through TMA im2col), ``square-256`` and
    ``rnn-matvec`` as GEMMs.  The matvec's N = 1 is computed as N = 8 (output
    rows must be 16-byte aligned for the TMA store); its FLOPs are counted at
    the reference shape (``table1_flops``)."""
    if preset == "resnet18-conv2_2":
        return conv2_2()
    p = find_preset(preset)
    if p is None:
        raise KeyError(preset)
    s = p.layers[0]
    return [Layer(preset, "gemm", rows=s.m, n=max(s.n, 8), k=s.k)]


def table1_flops(preset: str) -> int:
    """Reference FLOPs of one Table-1 member (2mnk at the preset's shape)."""
    if preset == "resnet18-conv2_2":
        return conv2_2()[0].flops(1)
    s = find_preset(preset).layers[0]
    return 2 * s.m * s.n * s.k


def graph_json(layers: List[Layer]) -> List[dict]:
    """The layer graph as plain data (oracle/graphs/*.json: the form the CPU
    baseline and the reference arm read without importing this package)."""
    out = []
    for L in layers:
        c = L.conv
        out.append({"name": L.name, "kind": L.kind,
                    "conv": None if c is None else [c.image_h, c.image_w, c.kernel_h, c.kernel_w, c.in_channels,
                                                    c.out_channels, c.stride, c.padding],
                    "rows": L.rows, "n": L.n, "k": L.k, "act": L.act, "src": L.src, "res": L.res,
                    "src_col": L.src_col})
    return out


# graphs exported to oracle/graphs (tools/export_graphs.py; pinned by tests/test_workload.py)
EXPORTED_GRAPHS = {
    "resnet50_224": lambda: resnet50(224),
    "vgg16_224": lambda: vgg16(224),
    "mobilenet_v2_224": lambda: mobilenet_v2(224),
    "bert_base_12": lambda: bert_base_gemms(128, layers=12),
    "resnet18_128": lambda: resnet18(128, classifier=False),
    "conv2_2": lambda: conv2_2(),
}


MODELS = {
    "resnet50": resnet50,
    "resnet18": resnet18,
    "vgg16": vgg16,
    "mobilenet_v2": mobilenet_v2,
    "bert_base": bert_base_gemms,
    "conv2_2": conv2_2,
}
