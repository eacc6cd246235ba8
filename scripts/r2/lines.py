"""Print the key fields of bench JSON lines: python scripts/r2/lines.py FILE..."""
import json, sys
for f in sys.argv[1:]:
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
    except Exception as e:
        print(f, "unreadable", e); continue
    r = d.get("roofline", {})
    e = d.get("e2e", {})
    print(f"{f}: {d.get('config',{}).get('workload')} value={d.get('value'):.1f} ms={d.get('ms_per_step'):.4f} "
          f"frac={r.get('frac', 0):.3f} e2e={e.get('value', 0):.2f} clocks={d.get('clocks',{}).get('sm_mhz')} {d.get('clocks',{}).get('reasons')}")
