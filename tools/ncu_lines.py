"""Per-source-line instruction and stall-sample shares of one profiled kernel
(ncu --page source --print-source cuda,sass), run here on the CPU box.

    python tools/ncu_lines.py gpurun_out/prof.ncu-rep "ssb_pipeline_kernel<(int)3" [top]"""
import csv
import io
import subprocess
import sys

rep, pat = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True, check=True).stdout
agg, path, fn, hdr, seen = {}, None, None, None, None
for r in csv.reader(io.StringIO(out)):
    if not r:
        continue
    if r[0] == "File Path":
        path = r[1].split("/")[-1]
    elif r[0] == "Function Name":
        fn = r[1]
        if pat in fn and seen is None:
            seen = fn
    elif r[0] == "Line No":
        hdr = r
    elif fn == seen and seen is not None and r[0] not in ("",) and hdr:
        ie, smp = hdr.index("Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)")
        try:
            agg[(path, int(r[0]))] = (int(r[ie]), int(r[smp]), r[1].strip())
        except ValueError:
            pass
print(seen)
ti = sum(v[0] for v in agg.values()) or 1
ts = sum(v[1] for v in agg.values()) or 1
print(f"instructions {ti}  stall samples {ts}")
for (p, ln), (i, s, src) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
    print(f"{100 * i / ti:5.1f}% inst {100 * s / ts:5.1f}% smp  {p}:{ln}  {src[:100]}")
