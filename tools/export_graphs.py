"""Export the product's model graphs (workload.py) to oracle/graphs/*.json,
the package-free form bench.py's reference arm and CPU baseline read."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1901_00041_b200 import workload as W  # noqa: E402

for name, build in W.EXPORTED_GRAPHS.items():
    with open(os.path.join(ROOT, "oracle", "graphs", name + ".json"), "w") as f:
        json.dump(W.graph_json(build()), f, indent=0)
        f.write("\n")
    print(name)
