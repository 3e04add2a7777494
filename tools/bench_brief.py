#!/usr/bin/env python
"""One-line digest of a bench.py JSON log (last JSON line of the file)."""
import json
import sys

for line in reversed(open(sys.argv[1]).read().splitlines()):
    if line.startswith("{"):
        d = json.loads(line)
        r = d.get("roofline") or {}
        e = d.get("e2e") or {}
        print(f"value {d['value']:.4g} {d['unit']}  ms/step {d.get('ms_per_step', 0):.3f}  "
              f"d1-field {r.get('launch_ms', 0):.3f} ms {r.get('gcones_per_s', 0):.2f} Gcones/s "
              f"frac {r.get('frac', 0):.3f} share {r.get('field_share_of_step', 0):.2f}  "
              f"e2e {e.get('value', 0):.4g}  clocks {d.get('clocks')}  "
              f"cpu {(d.get('cpu_baseline') or {}).get('value')}")
        break
