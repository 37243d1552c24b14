"""Summarise an ncu --metrics gpu__time_duration.sum launch list (library kernels only)."""
import collections
import csv
import re
import sys


def main(path, out=None, title=""):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
    h = rows[hi]
    data = rows[hi + 1:]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    tot, cnt = collections.defaultdict(float), collections.Counter()
    for r in data:
        if len(r) <= vi:
            continue
        name = re.sub(r"\(.*", "", r[ki])
        for pre in ("fsa::<unnamed>::", "fsa::", "void ", "unnamed>::"):
            name = name.replace(pre, "")
        v = float(r[vi].replace(",", "")) * {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3}[r[ui]]
        tot[name] += v
        cnt[name] += 1
    T = sum(tot.values())
    lines = [f"# {title}", "# ncu --metrics gpu__time_duration.sum --clock-control none (cold-cache, serialised: compare shares)",
             f"# library kernels: {sum(cnt.values())} launches, {T/1e3:.2f} ms total", "# share  launches  avg_us  kernel"]
    for k, v in sorted(tot.items(), key=lambda x: -x[1]):
        lines.append(f"{100*v/T:6.2f}% {cnt[k]:6d} {v/cnt[k]:9.1f}  {k[:110]}")
    txt = "\n".join(lines) + "\n"
    if out:
        open(out, "w").write(txt)
    print(txt)


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else None, sys.argv[3] if len(sys.argv) > 3 else "")
