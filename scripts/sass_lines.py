"""Dynamic instruction counts per CUDA source line: joins an ncu source page (SASS rows in
address order, with 'Instructions Executed') to the local cubin's line table.
  ncu -i rep --page source --csv --print-source sass > src.csv
  python scripts/sass_lines.py src.csv <cubin> <mangled-kernel-substring> [n_segments] [top]
The cubin must be the one the capture ran (same source, same flags)."""
import collections
import csv
import re
import subprocess
import sys


def ncu_counts(path, pat):
    rows = list(csv.reader(open(path)))
    cur, hdr, out = None, None, []
    for r in rows:
        if r and r[0] == "Kernel Name":
            if out:
                break
            cur, hdr = r[1], None
        elif r and r[0] == "Address":
            hdr = r
        elif hdr and r and pat in (cur or ""):
            d = dict(zip(hdr, r))
            out.append((d["Source"].strip(), int(d.get("Instructions Executed") or 0)))
    return out


def cubin_lines(cubin, mangled):
    txt = subprocess.run(["nvdisasm", "-g", "-c", cubin], capture_output=True, text=True).stdout
    sec = None
    line = "?"
    res = []
    for ln in txt.splitlines():
        m = re.match(r"\s*\.section\s+\.text\.([^,\s]+)", ln)
        if m:
            sec = m.group(1).rstrip(",")
            continue
        if sec != mangled:
            continue
        m = re.search(r"//## File \"([^\"]+)\", line (\d+)", ln)
        if m:
            line = f"{m.group(1).split('/')[-1]}:{m.group(2)}"
            continue
        m = re.match(r"\s*/\*([0-9a-f]{4,})\*/\s+(.*?);", ln)
        if m:
            res.append((line, m.group(2).strip()))
    return res


def main():
    src, cubin, mangled = sys.argv[1:4]
    nseg = float(sys.argv[4]) if len(sys.argv) > 4 else 1.0
    top = int(sys.argv[5]) if len(sys.argv) > 5 else 60
    counts = ncu_counts(src, sys.argv[6] if len(sys.argv) > 6 else "clip_compact")
    lines = cubin_lines(cubin, mangled)
    if len(counts) != len(lines):
        sys.exit(f"instruction count mismatch: ncu {len(counts)} vs cubin {len(lines)}")
    per = collections.Counter()
    ops = collections.defaultdict(collections.Counter)
    for (ln, sass), (_, ex) in zip(lines, counts):
        per[ln] += ex
        op = [o for o in sass.split() if not o.startswith("@")][0]
        ops[ln][op] += ex
    tot = sum(per.values())
    print(f"total thread-inst/seg {32 * tot / nseg:.1f}")
    for ln, ex in per.most_common(top):
        mix = ", ".join(f"{o} {32 * c / nseg:.2f}" for o, c in ops[ln].most_common(4))
        print(f"{32 * ex / nseg:7.2f}  {ln:28s} {mix}")


if __name__ == "__main__":
    main()
