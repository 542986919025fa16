"""Print the key fields of a bench.py JSON line (stdin or file)."""
import json
import sys

src = open(sys.argv[1]) if len(sys.argv) > 1 else sys.stdin
line = [l for l in src.read().strip().splitlines() if l.startswith("{")][-1]
d = json.loads(line)
e = d.get("e2e", {})
r = d.get("roofline", {})
print(f"value={d['value']:.4g} ms/step={d.get('ms_per_step', 0):.4f} kernel_ms={r.get('kernel_ms', 0):.4f} "
      f"frac={r.get('frac', 0):.3f} smem_frac={r.get('frac_smem_loaded', 0):.3f}")
print(f"e2e={e.get('value', 0):.4g} ms/img={e.get('ms_per_image', 0):.4f} "
      f"detect_ms={e.get('detect_latency_ms', 0):.4f} "
      f"phases={ {k: round(v, 4) for k, v in e.get('latency_phases_ms_median', {}).items()} }")
print(f"launches={d.get('gpu_launches')} clocks={d.get('clocks')} cand={d.get('search', {}).get('candidates')}")
if "cpu_baseline" in d:
    print(f"cpu_baseline={d['cpu_baseline']}")
