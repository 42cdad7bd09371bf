"""Summarise a tools/trace_round.py --out JSON by ResNet stage (debug aid)."""
import json
import sys
from collections import OrderedDict

for path in sys.argv[1:]:
    d = json.load(open(path))
    seg = OrderedDict()
    for r in d["rows"]:
        m = int(r["sig"].split("x")[0])
        k = int(r["sig"].split("x")[2].split("*")[0])
        seg.setdefault((m, "stem" if k == 147 else ""), []).append(r)
    print(f"{path}: span {d['span_us']:.1f}us roof {d['roof_us']:.1f}us")
    for key, rs in seg.items():
        st = min(r["start_us"] for r in rs)
        en = max(r["start_us"] + r["span_us"] for r in rs)
        means = tuple(sum(r[f] for r in rs) / len(rs) for f in ("gate", "load", "mma", "drain", "epi"))
        print(f"  {str(key):16s} [{st:6.1f},{en:6.1f}] wall {en - st:6.1f}us roof {sum(r['roof_us'] for r in rs):6.1f}"
              f" | gate {means[0]:6.2f} load {means[1]:5.2f} mma {means[2]:5.2f} drain {means[3]:5.2f} epi {means[4]:5.2f}")
