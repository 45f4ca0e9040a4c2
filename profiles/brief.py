"""one-line summary of a bench.py JSON line read from stdin (for quick A/B runs)"""
import json
import sys

tag = " ".join(sys.argv[1:])
for line in sys.stdin:
    line = line.strip()
    if not line.startswith("{"):
        continue
    d = json.loads(line)
    k = {n: round(v["ms"] * 1000, 1) for n, v in d["roofline"]["kernels"].items()}
    print(tag, "T", d["config"]["frames_in_flight"], "fps", round(d["value"], 1), "p50", round(d["p50_latency_ms"], 2),
          "e2e", round((d.get("e2e") or {}).get("value", 0.0), 1), "apply_us", round(d["roofline"]["apply"]["ms"] * 1000, 1),
          k, "clk", (d.get("clocks") or {}).get("sm_mhz"), flush=True)
