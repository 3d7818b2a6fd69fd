"""One-screen summary of a bench.py JSON line (the last line of the file)."""
import json
import sys

d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
print("kernel", d["value"], d["unit"], "frac", d["roofline"]["frac"], "clocks", d["clocks"])
print("e2e", d["e2e"]["value"], "roundtrip", d["e2e"]["host_params_roundtrip"]["value"], "cpu", d.get("cpu_baseline", {}).get("value"))
p = d.get("pipeline") or {}
if "error" in p:
    print("pipeline error", p["error"])
else:
    print("config1", p["pred_off"]["samples_per_s"], p["pred_on"]["samples_per_s"], "ovh", p["prediction_overhead"],
          "serial", p["serial_streams"]["pred_off"]["samples_per_s"], p["serial_streams"]["pred_on"]["samples_per_s"],
          p["serial_streams"]["prediction_overhead"])
    print("tf32", p["tf32"]["pred_off"]["samples_per_s"], p["tf32"]["pred_on"]["samples_per_s"], p["tf32"]["prediction_overhead"])
    print("proj8", p["projected_8gpu"]["prediction_overhead"], p["projected_8gpu"]["pred_off"]["multi_gpu_samples_per_s"],
          p["projected_8gpu"]["pred_on"]["multi_gpu_samples_per_s"], "simt", p["projected_8gpu"].get("simt_fp32_gemms"),
          "multi-gpu roof ovh", p.get("multi_gpu_roofline_prediction_overhead"))
    print("cpu pipeline", p.get("cpu_baseline", {}).get("value"))
    for c, v in p.get("configs", {}).items():
        print(c, v.get("pred_off", {}).get("samples_per_s"), v.get("pred_on", {}).get("samples_per_s"),
              v.get("prediction_overhead"), v.get("multi_gpu_roofline_prediction_overhead"), v.get("error"))
    if "depth_sweep_1gpu" in p:
        print("depth sweep (1 GPU)", {k: (v["pred_off"], v["pred_on"], v["prediction_overhead"])
                                       for k, v in p["depth_sweep_1gpu"].items()})
