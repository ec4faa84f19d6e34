"""one line per bench JSON (gpurun_out/*.json): step, split, index, e2e, roofline"""
import json
import sys

for f in sys.argv[1:]:
    for ln in open(f):
        ln = ln.strip()
        if not ln.startswith("{"):
            continue
        d = json.loads(ln)
        if "unavailable" in d or "config" not in d:
            print(f, ln[:200])
            continue
        c = d["config"]
        ix = c.get("index", {})
        ps = d.get("paper_split_ms", {})
        print(f"{f}: {c['workload']} | step {d['ms_per_step']:.2f} ms | X {ps.get('X_extract_kernel', 0):.2f} "
              f"ingest {ps.get('ingest_sort', 0):.2f} | {ix.get('lookup')} {ix.get('key_bits')}b "
              f"probe {ix.get('max_probe')} | e2e {(d.get('e2e') or {}).get('ms_per_step')} | "
              f"frac {d['roofline']['frac']:.4f} | value {d['value']:.3e} | clk {d['clocks'].get('sm_mhz')}")
