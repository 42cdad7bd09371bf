"""Instruction count per kernel of the product library (cuobjdump -sass)."""
import re
import subprocess
import sys

lib = sys.argv[1] if len(sys.argv) > 1 else "paper_1901_00041_b200/_lib/libgpumux_b200.so"
out = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
fn, last = None, {}
for line in out.splitlines():
    m = re.search(r"Function : (\S+)", line)
    if m:
        fn = m.group(1)
        continue
    m = re.search(r"/\*([0-9a-f]{4,})\*/", line)
    if m and fn:
        last[fn] = int(m.group(1), 16)
for f, off in sorted(last.items(), key=lambda x: x[1]):
    print(off // 16 + 1, f)
