"""Small driver for ncu: builds the bench workload and launches rounds
eagerly (no graph) so each launch is a separate, profilable kernel.
--round: one persistent round-program launch per round (the headline path);
otherwise one launch per formed super-kernel.  Never used for bench numbers."""
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
    ap.add_argument("--round", action="store_true")
    a = ap.parse_args()
    layers = W.resnet50(224) if a.model == "resnet50" else W.MODELS[a.model]()
    eng = SpaceTimeEngine([layers] * a.tenants, [a.batch] * a.tenants)
    rnd = eng.plan_round()
    s = torch.cuda.Stream()
    for _ in range(a.rounds):
        (rnd.launch_round if a.round else rnd.launch)(s.cuda_stream)
    torch.cuda.synchronize()
    print("plans per round:", len(rnd.kernels))


if __name__ == "__main__":
    main()
