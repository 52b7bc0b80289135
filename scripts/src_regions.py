"""Stall samples and executed instructions per source line of an ncu source page (SASS rows),
joined to a cubin's line table (as sass_lines.py): where warps spend their samples.
  python scripts/src_regions.py src.csv cubin mangled n_segments [top]"""
import collections
import sys

sys.path.insert(0, __file__.rsplit("/", 1)[0])
from sass_lines import cubin_lines  # noqa: E402
import csv  # noqa: E402


def main():
    src, cubin, mangled, n = sys.argv[1:5]
    top = int(sys.argv[5]) if len(sys.argv) > 5 else 40
    rows = list(csv.reader(open(src)))
    hdr, items = None, []
    for r in rows:
        if r and r[0] == "Address":
            hdr = r
            continue
        if hdr and r and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            items.append((int(d["Warp Stall Sampling (All Samples)"] or 0), int(d["Instructions Executed"] or 0)))
    lines = cubin_lines(cubin, mangled)
    assert len(lines) == len(items), (len(lines), len(items))
    agg = collections.defaultdict(lambda: [0, 0])
    for (smp, ie), (ln, _op) in zip(items, lines):
        agg[ln][0] += smp
        agg[ln][1] += ie
    tot = sum(v[0] for v in agg.values())
    print(f"samples {tot}")
    for ln, (smp, ie) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
        print(f"{100 * smp / tot:6.2f}% samples {32 * ie / float(n):8.2f} inst/seg  {ln}")


if __name__ == "__main__":
    main()
