"""one-line summary of bench JSON lines in the given logs"""
import json, sys
for f in sys.argv[1:]:
    for l in open(f):
        if l.startswith('{'):
            d = json.loads(l); r = d.get('roofline', {}); ph = r.get('phase_ms_last_step', {})
            print(f"{f}: {d['ms_per_step']:.3f} ms/step {d['value']/1e9:.3f} Gev/s frac {r.get('frac', 0):.3f} ev {r.get('avg_launch_ms', 0):.4f} ms "
                  f"ct {d.get('counter_pass', {}).get('avg_launch_ms', 0) if isinstance(d.get('counter_pass'), dict) else r.get('counter_pass', {}).get('avg_launch_ms', 0)} syncs {d.get('host_syncs_per_step')} launches {d.get('launches_per_step')}")
            print("   ", " ".join(f"{k} {v:.3f}" for k, v in ph.items() if v is not None))
