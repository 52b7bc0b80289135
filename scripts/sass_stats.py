"""Per-kernel SASS statistics of a built .so (run here, no GPU needed).

  python scripts/sass_stats.py paper_1110_5450_b200/lib/libclipseg.so [name-substring]

For each kernel: total instructions, opcode histogram, and the instructions of the
hottest loop body (the largest backward-branch range), which is what the per-segment
issue budget of DESIGN.md §5 is checked against.
"""
import collections
import re
import subprocess
import sys


def functions(so):
    out = subprocess.run(["cuobjdump", "-sass", so], capture_output=True, text=True).stdout
    cur, body = None, []
    for line in out.splitlines():
        m = re.match(r"\s+Function : (\S+)", line)
        if m:
            if cur:
                yield cur, body
            cur, body = m.group(1), []
            continue
        m = re.match(r"\s+/\*([0-9a-f]{4,})\*/\s+(.*?);", line)
        if m and cur:
            body.append((int(m.group(1), 16), m.group(2).strip()))
    if cur:
        yield cur, body


def opcode(ins):
    ins = re.sub(r"^@!?U?P\w+\s+", "", ins)
    return ins.split()[0] if ins else ""


def main():
    so = sys.argv[1]
    pat = sys.argv[2] if len(sys.argv) > 2 else ""
    for name, body in functions(so):
        if pat not in name:
            continue
        ops = collections.Counter(opcode(i) for _, i in body)
        print(f"== {name}: {len(body)} instructions")
        print("   " + ", ".join(f"{k}:{v}" for k, v in ops.most_common(24)))
        # largest loop: backward BRA target..source
        best = None
        for addr, ins in body:
            m = re.search(r"BRA\s+(?:`\(\.L_x_\d+\)\s*)?0x([0-9a-f]+)", ins)
            if m:
                tgt = int(m.group(1), 16)
                if tgt < addr and (best is None or addr - tgt > best[1] - best[0]):
                    best = (tgt, addr)
        if best:
            loop = [i for a, i in body if best[0] <= a <= best[1]]
            lops = collections.Counter(opcode(i) for i in loop)
            print(f"   hottest loop [{best[0]:#x},{best[1]:#x}]: {len(loop)} instructions")
            print("   " + ", ".join(f"{k}:{v}" for k, v in lops.most_common(24)))


if __name__ == "__main__":
    main()
