"""Print gpurun_out/sweep/<op>.jsonl (tools/op_sweep.sh) as a variant x config table of kernel ms."""
import json
import sys

f = sys.argv[1]
rows = {}
for line in open(f):
    d = json.loads(line)
    key = (d.get("variant"), d.get("sigma")) if d.get("bench") == "select" else (
        d.get("ht_bytes", 0) >> 10 if d.get("bench") == "join_probe" else (d.get("variant"), d.get("n")))
    rows.setdefault(d["env"], {})[key] = f"{d['kernel_ms']}{'' if d.get('golden_ok', True) in (True, None) else '!'}"
envs = list(rows)
print("config".ljust(24), *[e[-20:].rjust(20) for e in envs])
for k in rows[envs[0]]:
    print(str(k).ljust(24), *[str(rows[e].get(k)).rjust(20) for e in envs])
