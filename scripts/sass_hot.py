"""Per-SASS-instruction execution counts and stall samples from an ncu source page.
  ncu -i rep --page source --csv --print-source sass > src.csv
  python scripts/sass_hot.py src.csv [kernel-substring] [n_segments]
Prints instruction-count totals by opcode (dynamic) and the hottest stall lines."""
import collections
import csv
import sys


def blocks(path):
    rows = list(csv.reader(open(path)))
    cur, hdr, body = None, None, []
    for r in rows:
        if r and r[0] == "Kernel Name":
            if cur:
                yield cur, hdr, body
            cur, hdr, body = r[1], None, []
        elif r and r[0] == "Address":
            hdr = r
        elif hdr and r:
            body.append(dict(zip(hdr, r)))
    if cur:
        yield cur, hdr, body


def main():
    path = sys.argv[1]
    pat = sys.argv[2] if len(sys.argv) > 2 else ""
    nseg = float(sys.argv[3]) if len(sys.argv) > 3 else None
    seen = set()
    for name, hdr, body in blocks(path):
        if pat not in name or name in seen:
            continue
        seen.add(name)
        ops = collections.Counter()
        total = 0
        for d in body:
            ex = int(d.get("Instructions Executed") or 0)
            op = d["Source"].strip().split()
            op = [o for o in op if not o.startswith("@")]
            ops[op[0] if op else "?"] += ex
            total += ex
        print("==", name[:100])
        print(f"   dynamic warp-instructions {total}" + (f"  thread-inst/seg {32 * total / nseg:.1f}" if nseg else ""))
        for k, v in ops.most_common(30):
            print(f"   {k:28s} {v:12d}" + (f"  {32 * v / nseg:7.2f}/seg" if nseg else ""))
        hot = sorted(body, key=lambda d: -int(d.get("Warp Stall Sampling (All Samples)") or 0))[:25]
        print("   hottest stall lines:")
        for d in hot:
            print(f"     {d['Address'][-5:]} {int(d.get('Warp Stall Sampling (All Samples)') or 0):7d}  {d['Source'].strip()[:80]}")


if __name__ == "__main__":
    main()
