"""Print variant / kernel_ms / sorted from bench_ops sort JSON lines on stdin."""
import json
import sys

for line in sys.stdin:
    if line.startswith("{"):
        r = json.loads(line)
        print(r.get("variant"), r.get("kernel_ms"), r.get("sorted"), r.get("golden_ok", ""))
