"""Small driver for ncu: builds a bench workload and launches rounds eagerly
(no graph) so each launch is a separate, profilable kernel.
--round: one persistent round-program launch per round (the headline path);
otherwise one launch per formed super-kernel.  Never used for bench numbers.
--config: headline (4 x ResNet-50@224 b8), bert4 (16 x BERT-base b4),
mix4 (2 x {ResNet-50, VGG-16, MobileNet-v2}@224 b4), table1 (R x conv2_2 b1)."""
import argparse
import sys

import torch

sys.path.insert(0, ".")
from paper_1901_00041_b200 import workload as W  # noqa: E402
from paper_1901_00041_b200.engine import SpaceTimeEngine  # noqa: E402


def build(config, tenants, batch, model, r):
    if config == "bert4":
        return SpaceTimeEngine([W.bert_base_gemms(128, layers=12)] * 16, [4] * 16)
    if config == "mix4":
        models = [W.resnet50(224), W.vgg16(224), W.mobilenet_v2(224)] * 2
        return SpaceTimeEngine(models, [4] * len(models))
    if config == "table1":
        return SpaceTimeEngine([W.table1_layers("resnet18-conv2_2")] * r, [1] * r)
    layers = W.resnet50(224) if model == "resnet50" else W.MODELS[model]()
    return SpaceTimeEngine([layers] * tenants, [batch] * tenants)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="headline", choices=["headline", "bert4", "mix4", "table1"])
    ap.add_argument("--model", default="resnet50")
    ap.add_argument("--tenants", type=int, default=4)
    ap.add_argument("--batch", type=int, default=8)
    ap.add_argument("--r", type=int, default=120, help="table1: tenants")
    ap.add_argument("--rounds", type=int, default=2)
    ap.add_argument("--round", action="store_true")
    a = ap.parse_args()
    eng = build(a.config, a.tenants, a.batch, a.model, a.r)
    rnd = eng.plan_round()
    s = torch.cuda.Stream()
    for _ in range(a.rounds):
        (rnd.launch_round if a.round else rnd.launch)(s.cuda_stream)
    torch.cuda.synchronize()
    print("plans per round:", len(rnd.kernels))


if __name__ == "__main__":
    main()
