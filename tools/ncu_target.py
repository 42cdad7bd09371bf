"""Small driver for ncu: builds the bench workload and replays the packed
round eagerly (no graph) `--rounds` times so every super-kernel launch is a
separate, profilable kernel.  Never used for bench numbers."""
import argparse
import sys

import torch

sys.path.insert(0, ".")
from paper_1901_00041_b200 import workload as W  # noqa: E402
from paper_1901_00041_b200.engine import SpaceTimeEngine  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--model", default="resnet50")
    ap.add_argument("--tenants", type=int, default=4)
    ap.add_argument("--batch", type=int, default=8)
    ap.add_argument("--rounds", type=int, default=2)
    a = ap.parse_args()
    layers = W.resnet50(224) if a.model == "resnet50" else W.MODELS[a.model]()
    eng = SpaceTimeEngine([layers] * a.tenants, [a.batch] * a.tenants)
    rnd = eng.plan_round()
    s = torch.cuda.Stream()
    for _ in range(a.rounds):
        rnd.launch(s.cuda_stream)
    torch.cuda.synchronize()
    print("launches per round:", len(rnd.kernels))


if __name__ == "__main__":
    main()
