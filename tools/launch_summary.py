"""Aggregate an `ncu --metrics gpu__time_duration.sum --csv` launch list per kernel.

    python tools/launch_summary.py gpurun_out/launches_TAG.csv > profiles/rN/launch_list_summary_TAG.txt

Shares are of the FDK step's kernels (filter + back-projection); ncu's launches are cold-cache
and serialised, so compare shares, not absolute times."""
import collections
import csv
import sys

FDK = ("bp_quad2_kernel", "bp_tmem2_kernel", "bp_tmem_kernel", "bp_raw_kernel", "bp_kernel", "filter_f4k_kernel",
       "filter_fft_kernel")


def main(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    head = rows[0]
    ki, mi, vi = head.index("Kernel Name"), head.index("Metric Name"), head.index("Metric Value")
    t = collections.defaultdict(float)
    n = collections.Counter()
    for r in rows[1:]:
        if r[mi] != "gpu__time_duration.sum":
            continue
        unit = r[head.index("Metric Unit")] if "Metric Unit" in head else "ns"
        scale = {"ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "nsecond": 1e-6, "ms": 1.0,
                 "msecond": 1.0}.get(unit, 1e-6)
        t[r[ki]] += float(r[vi].replace(",", "")) * scale
        n[r[ki]] += 1
    fdk = sum(v for k, v in t.items() if any(f in k for f in FDK))
    print(f"ncu launch list {path}\n(cold-cache, serialised launches; compare shares, not absolutes)\n")
    for k, v in sorted(t.items(), key=lambda kv: -kv[1]):
        share = f"{v / fdk:.3f}" if any(f in k for f in FDK) else "  n/a (not in the FDK step)"
        print(f"{n[k]:4d} launches {v:11.2f} ms total {v / n[k]:10.2f} ms/launch  share {share}  "
              f"{k[:110]}")


if __name__ == "__main__":
    main(sys.argv[1])
