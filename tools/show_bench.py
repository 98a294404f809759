import json, sys
for line in sys.stdin:
    line = line.strip()
    if not line.startswith("{"):
        print(line[:300]); continue
    d = json.loads(line)
    print("ms/step", d.get("ms_per_step"), "value", d.get("value"), "e2e", d.get("e2e", {}).get("value"))
    for k in ("phases_ms", "subband_iterations", "roofline", "clocks", "cpu_baseline", "gpu_launches_per_step"):
        if k in d: print(k, d[k])
