"""Print ms/step and per-stage ms from the last JSON line of a bench.py log."""
import json
import sys

line = [l for l in open(sys.argv[1]) if l.startswith("{")][-1]
d = json.loads(line)
print(d["ms_per_step"], {k: v["ms"] for k, v in d["stages"].items()})
