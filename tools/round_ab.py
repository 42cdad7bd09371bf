"""Round-program A/B over runtime options on one box (debug aid).

  python tools/round_ab.py --config headline|mix|bert4 --opts "-" "greedy_schedule=1" ...
Prints the mean round time (CUDA events, 10 replays after 3 warmups) per option set.
"""
import argparse
import sys

import torch

sys.path.insert(0, ".")
from paper_1901_00041_b200 import workload as W  # noqa: E402
from paper_1901_00041_b200.engine import SpaceTimeEngine  # noqa: E402


def build(config, opts):
    if config == "headline":
        return SpaceTimeEngine([W.resnet50(224)] * 4, [8] * 4, options=opts)
    if config.startswith("r50x"):  # r50x<T>b<B>: T tenants x ResNet-50 batch B
        t, b = config[4:].split("b")
        return SpaceTimeEngine([W.resnet50(224)] * int(t), [int(b)] * int(t), options=opts)
    if config == "mix":
        ms = [W.resnet50(224), W.vgg16(224), W.mobilenet_v2(224)] * 2
        return SpaceTimeEngine(ms, [4] * 6, options=opts)
    if config.startswith("t1r"):  # Table-1 microbench: R tenants x conv2_2 b1
        r = int(config[3:])
        return SpaceTimeEngine([W.conv2_2()] * r, [1] * r, options=opts)
    if config.startswith("solo_"):  # solo_<model>b<B>: one tenant alone (chain latency)
        name, b = config[5:].rsplit("b", 1)
        layers = {"vgg16": W.vgg16(224), "resnet50": W.resnet50(224), "mobilenet": W.mobilenet_v2(224)}[name]
        return SpaceTimeEngine([layers], [int(b)], options=opts)
    if config.startswith("bert"):  # bert<B>: 16 tenants x BERT-base (12 layers), batch B
        return SpaceTimeEngine([W.bert_base_gemms(128, 12)] * 16, [int(config[4:])] * 16, options=opts)
    raise SystemExit(config)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="headline")
    ap.add_argument("--opts", nargs="+", default=["-"])
    ap.add_argument("--reps", type=int, default=2)
    a = ap.parse_args()
    s = torch.cuda.Stream()
    for rep in range(a.reps):
        for o in a.opts:
            opts = {} if o == "-" else {kv.split("=")[0]: int(kv.split("=")[1]) for kv in o.split(",")}
            eng = build(a.config, opts)
            g = eng.capture_round(eng.plan_round())
            for _ in range(3):
                g.launch(s.cuda_stream)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            e0.record(s)
            for _ in range(10):
                g.launch(s.cuda_stream)
            e1.record(s)
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / 10
            print(f"{a.config:9s} {o:40s} {ms * 1e3:8.1f} us  {eng.flops_per_round() / ms / 1e9:7.1f} TF/s", flush=True)
            del g, eng


if __name__ == "__main__":
    main()
