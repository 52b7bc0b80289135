"""Build experimental library variants in parallel: name:DEF=V,DEF2=V2 ... -> build/libclipseg_<name>.so
and print registers / spills of the compacting kernels.
  python scripts/build_variants.py e0: f64a:CLIPSEG_SHAPE_F64_2D=12,12,3 ..."""
import os
import re
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import build_all  # noqa: E402


def one(spec):
    name, _, defs = spec.partition(":")
    # a shape macro value contains commas: split definitions on ';'
    d = [x for x in defs.split(";") if x]
    _, log = build_all.build_variant(name, d, verbose=True)
    rows, cur, stack = [], None, None
    for line in log.splitlines():
        m = re.search(r"Compiling entry function '(\S+)'", line)
        if m:
            cur = m.group(1)
        m = re.search(r"(\d+) bytes spill stores", line)
        if m:
            stack = m.group(1)
        m = re.search(r"Used (\d+) registers", line)
        if m and cur and "compact" in cur and "ELb1ELb0" in cur:
            dem = subprocess.run(["c++filt", cur], capture_output=True, text=True).stdout.split("(")[0]
            rows.append(f"   {m.group(1):>4} regs {stack:>4} B spill  {dem[-60:]}")
            cur = None
    return name, rows


with ThreadPoolExecutor(8) as ex:
    for name, rows in ex.map(one, sys.argv[1:]):
        print(name)
        print("\n".join(rows))
