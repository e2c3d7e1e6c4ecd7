"""Read ncu --page raw/details CSV exports (tools/prof_r02.sh) here on the CPU box.

    python tools/ncu_csv.py raw  X_raw.csv [metric ...]     # one line per launch, chosen metrics
    python tools/ncu_csv.py det  X_details.csv [section]    # details page rows (optionally one section)
    python tools/ncu_csv.py sass X_sass.csv [top]            # hottest SASS lines by stall samples"""
import csv
import sys

DEF = ["gpu__time_duration.sum", "dram__bytes_read.sum", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
       "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
       "lts__t_sector_hit_rate.pct", "smsp__inst_executed.sum"]


def raw(path, metrics):
    r = list(csv.reader(open(path)))
    h = r[0]
    cols = [h.index("Kernel Name")] + [h.index(m) for m in metrics if m in h]
    print("kernel".ljust(58), *[m.split(".")[0][-22:] for m in metrics if m in h])
    for row in r[2:]:
        print(row[cols[0]].split("(")[0].replace("void ", "")[-58:].ljust(58), *[row[c] for c in cols[1:]])


def det(path, section=None):
    for row in csv.DictReader(open(path)):
        if section and section.lower() not in row.get("Section Name", "").lower():
            continue
        print(row.get("ID"), row.get("Kernel Name", "")[:40], "|", row.get("Section Name"), "|",
              row.get("Metric Name"), "=", row.get("Metric Value"), row.get("Metric Unit"))


def sass(path, top=40):
    rows = list(csv.reader(open(path)))
    h = next(i for i, r in enumerate(rows) if r and ("Source" in r or "# Address" in r or "Address" in r))
    hdr = rows[h]
    src = hdr.index("Source")
    cand = [i for i, c in enumerate(hdr) if "Warp Stall Sampling (All" in c]
    si = cand[0] if cand else None
    body = [r for r in rows[h + 1:] if len(r) > max(src, si or 0)]
    tot = sum(float(r[si] or 0) for r in body) if si is not None else 0
    body.sort(key=lambda r: -float(r[si] or 0))
    print("samples total", tot, "column", hdr[si])
    for r in body[:top]:
        print(f"{float(r[si] or 0):8.0f} {100 * float(r[si] or 0) / max(tot, 1):5.1f}%  {r[src][:110]}")


if __name__ == "__main__":
    mode, path = sys.argv[1], sys.argv[2]
    if mode == "raw":
        raw(path, sys.argv[3:] or DEF)
    elif mode == "det":
        det(path, sys.argv[3] if len(sys.argv) > 3 else None)
    else:
        sass(path, int(sys.argv[3]) if len(sys.argv) > 3 else 40)
