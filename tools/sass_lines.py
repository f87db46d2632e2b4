"""Per-source-line executed-instruction attribution of one kernel.

  python tools/sass_lines.py <ncu-rep> <kernel regex[@skip]> <cubin> <mangled name> [units] [top]

Joins ncu's per-SASS "Instructions Executed" (source page) with the line
table nvdisasm -g prints for the same function (build with -lineinfo).
`units` divides the counts (e.g. 32-point warp rows of the launch).  A
kernel regex of the form re@skip#column attributes another source-page
column (e.g. stall_wait, stall_short_sb)."""
import collections
import csv
import io
import re
import subprocess
import sys


def main():
    rep, kre, cubin, fn = sys.argv[1:5]
    units = float(sys.argv[5]) if len(sys.argv) > 5 else 1.0
    top = int(sys.argv[6]) if len(sys.argv) > 6 else 40
    skip = "0"
    col = "Instructions Executed"
    if "#" in kre:  # kernel regex#column: attribute another source-page column (e.g. stall_wait)
        kre, col = kre.split("#")
    if "@" in kre:
        kre, skip = kre.split("@")
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass", "-k",
                          "regex:" + kre, "--launch-skip", skip, "--launch-count", "1"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h = rows[1]
    ai, ei, si = h.index("Address"), h.index(col), h.index("Source")
    counts = []
    for r in rows[2:]:
        if len(r) > ei:
            try:
                counts.append((int(r[ai], 16), int(r[ei]), r[si].strip()))
            except ValueError:
                pass
    base = counts[0][0]
    dis = subprocess.run(["nvdisasm", "-g", "-c", cubin], capture_output=True, text=True).stdout
    sec = dis[dis.index(".text." + fn + ":"):]
    nxt = sec.find("//---------------------", 10)
    sec = sec[:nxt] if nxt > 0 else sec
    line_of = {}
    cur = None
    for ln in sec.splitlines():
        m = re.search(r'//## File "([^"]+)", line (\d+)', ln)
        if m:
            cur = m.group(1).split("/")[-1] + ":" + m.group(2)
            continue
        m = re.match(r"\s+/\*([0-9a-f]{4,})\*/", ln)
        if m:
            line_of[int(m.group(1), 16)] = cur
    agg = collections.Counter()
    ops = collections.defaultdict(collections.Counter)
    for a, n, s in counts:
        key = line_of.get(a - base, "?")
        agg[key] += n
        op = re.match(r"(@!?U?P\w+\s+)?([A-Z0-9_]+)", s)
        ops[key][op.group(2) if op else s] += n
    tot = sum(agg.values())
    print(f"total {tot / units:.1f} per unit")
    for k, n in agg.most_common(top):
        print(f"{n / units:8.1f} {k:24s} " + " ".join(f"{o}={c / units:.0f}" for o, c in ops[k].most_common(5)))


if __name__ == "__main__":
    main()
