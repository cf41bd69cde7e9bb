import json, sys
d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
print(f"{d['config']['workload'][:40]}: {d['ms_per_step']*1e3:.1f} us/step, value {d['value']:.3e} {d['unit']}, "
      f"vs cuBLAS {d.get('speedup_vs_cublas', float('nan')):.3f} (cuBLAS {d.get('cublas_dense_bf16', {}).get('ms_per_step', float('nan'))*1e3:.1f} us)")
r = d['roofline']
print(f"  roofline: {r['kernel']} {r['bound']} {r['achieved']:.0f} {r['unit']} frac {r['frac']:.3f}; clocks {d['clocks']}")
for l in d["per_layer"]:
    print(f"  {l['layer']:36s} {l['ms']*1e3:7.1f} us  frac {l['roofline_frac']:.3f}  " +
          " ".join(f"{k}={v*1e3:.1f}" for k, v in l["launch_ms"].items()))
if "e2e" in d: print("  e2e", {k: (round(v, 3) if isinstance(v, float) else v) for k, v in d["e2e"].items()})
if "cpu_baseline" in d: print("  cpu", d["cpu_baseline"])
