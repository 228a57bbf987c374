"""Summarise bench JSON lines under gpurun_out/ (one line per file)."""
import glob
import json
import sys

files = sys.argv[1:] or sorted(glob.glob("gpurun_out/b*.json"))
for f in files:
    try:
        j = json.loads(open(f).read().strip().splitlines()[-1])
    except Exception as e:  # noqa: BLE001
        print(f, "ERR", e)
        continue
    r = j["roofline"]
    cls = {k: round(v * 1e3, 1) for k, v in r["class_ms_per_step"].items() if v > 0}
    e2e = j["e2e"]["value"] if j.get("e2e") else None
    cpu = j["cpu_baseline"]["value"] if j.get("cpu_baseline") else None
    print(f"{f}: {j['config']['workload']} {j['config']['strategy']} ms/step {j['ms_per_step']:.4f} "
          f"value {j['value']:.1f} e2e {e2e and round(e2e, 1)} cpu {cpu and round(cpu, 2)} "
          f"dom {r['kernel']} frac {r['frac']:.3f} ({r['achieved']:.1f} {r['unit']}) "
          f"launches {j['gpu_launches']} clocks {j['clocks'].get('sm_mhz')} {j['clocks'].get('reasons')}")
    print("    class us/step:", cls)
    ws = j.get("window_stats", {})
    print("    window:", {k: v for k, v in ws.items() if any(v)})
