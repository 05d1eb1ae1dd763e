#!/usr/bin/env python
"""One line per bench JSON: workload, kernel ms, value, e2e, roofline frac, clocks, cpu."""
import json, sys
for f in sys.argv[1:]:
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
    except Exception as e:  # noqa: BLE001
        print(f, "unreadable", e); continue
    r = d.get("roofline") or {}; e = d.get("e2e") or {}; c = d.get("cpu_baseline") or {}
    print(f"{f.split('/')[-1]:22s} {d.get('config',{}).get('workload','?'):28s} ms={d.get('ms_per_step',0):9.3f} "
          f"val={d.get('value',0):.3e} e2e={e.get('value',0):.3e} ({e.get('ms_per_step')}) frac={r.get('frac')} "
          f"clk={d.get('clocks',{}).get('sm_mhz')} {d.get('clocks',{}).get('reasons')} cpu={c.get('value')}")
