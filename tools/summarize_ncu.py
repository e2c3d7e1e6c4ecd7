"""Summarise ncu output for profiles/ (run here, on the CPU box).

  python tools/summarize_ncu.py launches gpurun_out/launches.csv   # per-kernel share of a launch list
  python tools/summarize_ncu.py full gpurun_out/prof.ncu-rep        # key counters per profiled launch
  python tools/summarize_ncu.py sass gpurun_out/prof.ncu-rep [k]    # opcode mix + stall reasons of launch k
  python tools/summarize_ncu.py traffic gpurun_out/prof.ncu-rep out.json  # DRAM bytes per launch
"""
import csv
import io
import subprocess
import sys
from collections import Counter, defaultdict


def launches(path):
    rows = list(csv.reader(open(path)))
    h = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    hdr = rows[h]
    ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    agg = defaultdict(lambda: [0, 0.0])
    for r in rows[h + 1:]:
        if len(r) <= vi:
            continue
        scale = {"ns": 1e-3, "us": 1.0, "usecond": 1.0, "nsecond": 1e-3, "ms": 1e3}.get(r[ui], 1e-3)
        name = r[ki].split("(")[0].replace("void ", "").replace("(anonymous namespace)::", "")
        agg[name][0] += 1
        agg[name][1] += float(r[vi].replace(",", "")) * scale
    tot = sum(v[1] for v in agg.values())
    print(f"{'launches':>8} {'total_us':>12} {'avg_us':>10} {'share':>7}  kernel")
    for k, (n, us) in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"{n:8d} {us:12.1f} {us / n:10.1f} {100 * us / tot:6.1f}%  {k}")
    print(f"{'':8} {tot:12.1f} us total (ncu, cold-cache, serialised)")


KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "lts__t_sector_hit_rate.pct", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__grid_size", "launch__block_size", "launch__shared_mem_per_block_dynamic",
        "smsp__inst_executed.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum"]


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    return rows[0], rows[1], rows[2:]


def full(rep):
    hdr, units, data = raw(rep)
    for r in data:
        print("----", r[hdr.index("Kernel Name")][:110])
        for k in KEYS:
            if k in hdr:
                i = hdr.index(k)
                print(f"  {k:60s} {r[i]:>18s} {units[i]}")


def traffic(rep, out_json):
    """DRAM bytes per profiled launch (dram__bytes_read.sum + _write.sum) ->
    JSON consumed by bench.py's roofline.traffic."""
    import json
    hdr, units, data = raw(rep)
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}
    tscale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}
    launches = []
    for r in data:
        def val(k):
            i = hdr.index(k)
            return float(r[i].replace(",", "")) * scale.get(units[i], 1)
        ti = hdr.index("gpu__time_duration.sum")
        launches.append({"kernel": r[hdr.index("Kernel Name")].split("(")[0].replace("void ", ""),
                         "dram_read": val("dram__bytes_read.sum"),
                         "dram_write": val("dram__bytes_write.sum"),
                         "us": float(r[ti].replace(",", "")) * tscale.get(units[ti], 1e-3),
                         "l2_hit_pct": float(r[hdr.index("lts__t_sector_hit_rate.pct")])})
    # one suite pass in query order: flight 1 = one launch, a fused join pass
    # = one launch, a split plan = scan + gather
    names = ["q11", "q12", "q13", "q21", "q22", "q23", "q31", "q32", "q33", "q34", "q41", "q42", "q43"]
    per_query, i = {}, 0
    for q in names:
        if i >= len(launches):
            break
        parts = [launches[i]]
        i += 1
        if "scan_emit" in parts[0]["kernel"] and i < len(launches) and "gather" in launches[i]["kernel"]:
            parts.append(launches[i])
            i += 1
        per_query[q] = {"kernels": [x["kernel"] for x in parts],
                        "dram_bytes": sum(x["dram_read"] + x["dram_write"] for x in parts),
                        "us": sum(x["us"] for x in parts)}
    doc = {"source": rep, "launches": launches}
    if len(per_query) == 13 and i == len(launches):
        doc["per_query"] = per_query
    json.dump(doc, open(out_json, "w"), indent=1)
    for L in launches:
        print(f"{L['us']:9.1f} us  {(L['dram_read'] + L['dram_write']) / 1e9:7.3f} GB  "
              f"L2 hit {L['l2_hit_pct']:5.1f}%  {L['kernel'][:80]}")


def sass(rep, which=0):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True, check=True).stdout
    kern, cur, hdr = [], None, None
    for r in csv.reader(io.StringIO(out)):
        if r and r[0] == "Kernel Name":
            cur = [r[1], []]
            kern.append(cur)
        elif r and r[0] == "Address":
            hdr = r
        elif cur is not None and len(r) > 5:
            cur[1].append(r)
    name, ins = kern[which]
    ie = hdr.index("Instructions Executed")
    smp = hdr.index("Warp Stall Sampling (All Samples)")
    tot = sum(int(x[ie]) for x in ins)
    ts = sum(int(x[smp]) for x in ins) or 1
    print(name[:120])
    print(f"warp instructions executed {tot}, stall samples {ts}")
    op = Counter()
    for x in ins:
        t = x[1].split()
        o = t[1] if t[0].startswith("@") else t[0]
        op[o.split(".")[0]] += int(x[ie])
    for o, c in op.most_common(16):
        print(f"  {o:10s} {c:12d} {100 * c / tot:5.1f}%")
    print("stall reasons (share of samples):")
    for col in hdr:
        if col.startswith("stall_") and "(Not" not in col:
            i = hdr.index(col)
            s = sum(int(x[i]) for x in ins)
            if s * 100 >= ts:
                print(f"  {col:28s} {100 * s / ts:5.1f}%")


if __name__ == "__main__":
    mode, path = sys.argv[1], sys.argv[2]
    if mode == "launches":
        launches(path)
    elif mode == "full":
        full(path)
    elif mode == "traffic":
        traffic(path, sys.argv[3])
    else:
        sass(path, int(sys.argv[3]) if len(sys.argv) > 3 else 0)


def hot(rep, which=0, top=40):
    """Top SASS instructions of launch `which` by warp-stall samples."""
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True, check=True).stdout
    kern, cur, hdr = [], None, None
    for r in csv.reader(io.StringIO(out)):
        if r and r[0] == "Kernel Name":
            cur = [r[1], []]
            kern.append(cur)
        elif r and r[0] == "Address":
            hdr = r
        elif cur is not None and len(r) > 5:
            cur[1].append(r)
    name, ins = kern[which]
    smp = hdr.index("Warp Stall Sampling (All Samples)")
    ts = sum(int(x[smp]) for x in ins) or 1
    print(name[:120])
    idx = sorted(range(len(ins)), key=lambda i: -int(ins[i][smp]))[:top]
    for i in sorted(idx):
        print(f"{i:5d} {100 * int(ins[i][smp]) / ts:5.1f}%  {ins[i][1][:90]}")


if __name__ == "__main__" and sys.argv[1] == "hot":
    hot(sys.argv[2], int(sys.argv[3]) if len(sys.argv) > 3 else 0)
