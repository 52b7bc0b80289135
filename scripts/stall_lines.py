"""Warp-stall samples per CUDA source line: python scripts/stall_lines.py src.csv cubin mangled [top]"""
import collections
import csv
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from sass_lines import cubin_lines  # noqa: E402

src, cubin, mangled = sys.argv[1:4]
top = int(sys.argv[4]) if len(sys.argv) > 4 else 30
rows = list(csv.reader(open(src)))
hdr, body, kern = None, [], None
for r in rows:
    if r and r[0] == "Kernel Name":
        if body:
            break
        kern = r[1]
    elif r and r[0] == "Address":
        hdr = r
    elif hdr and r:
        body.append(dict(zip(hdr, r)))
lines = cubin_lines(cubin, mangled)
assert len(lines) == len(body), (len(lines), len(body))
st, tot = collections.Counter(), 0
reasons = collections.defaultdict(collections.Counter)
rk = [k for k in hdr if k.startswith("stall_") and "Not Issued" not in k]
for (ln, _), d in zip(lines, body):
    s = int(d.get("Warp Stall Sampling (All Samples)") or 0)
    st[ln] += s
    tot += s
    for k in rk:
        v = int(d.get(k) or 0)
        if v:
            reasons[ln][k] += v
for ln, s in st.most_common(top):
    print(f"{100 * s / tot:5.1f}% {ln:30s}", ", ".join(f"{k[6:]} {v}" for k, v in reasons[ln].most_common(3)))
