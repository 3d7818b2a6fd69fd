"""One-screen summary of a bench.py JSON line (the last line of the file)."""
import json
import sys

d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
print("kernel", d["value"], d["unit"], "frac", d["roofline"]["frac"], "clocks", d["clocks"])
e = d["e2e"]
print("e2e roundtrip", e["value"], "grad-in", e.get("grad_in_state_resident", {}).get("value"), "list api",
      e.get("list_api", {}).get("value"), "cpu", d.get("cpu_baseline", {}).get("value"))
print("kernels 1e9", {k: v["gbs"] for k, v in (d.get("kernels_1e9") or {}).items()})
p = d.get("pipeline") or {}
if "error" in p:
    print("pipeline error", p["error"])
else:
    print("config1", p["pred_off"]["samples_per_s"], p["pred_on"]["samples_per_s"], "ovh", p["prediction_overhead"],
          "frac", p["pred_on"].get("frac_of_roofline"), "bound", p["pred_on"].get("roofline", {}).get("single_gpu"),
          "serial", p["serial_streams"]["pred_off"]["samples_per_s"], p["serial_streams"]["pred_on"]["samples_per_s"],
          p["serial_streams"]["prediction_overhead"])
    print("tf32", p["tf32"]["pred_off"]["samples_per_s"], p["tf32"]["pred_on"]["samples_per_s"], p["tf32"]["prediction_overhead"])
    pj = p["projected_8gpu"]
    print("proj8", pj["prediction_overhead"], pj["pred_off"]["projection"]["one_stage_per_gpu_samples_per_s"],
          pj["pred_on"]["projection"]["one_stage_per_gpu_samples_per_s"], "frac", pj["pred_on"]["frac_of_roofline"],
          "simt", pj.get("simt_fp32_gemms"), "proj 1-stage/GPU ovh (D4)",
          p.get("projected_one_stage_per_gpu_prediction_overhead"))
    print("cpu pipeline", p.get("cpu_baseline", {}).get("value"))
    for c, v in p.get("configs", {}).items():
        print(c, v.get("pred_off", {}).get("samples_per_s"), v.get("pred_on", {}).get("samples_per_s"),
              v.get("prediction_overhead"), v.get("projected_one_stage_per_gpu_prediction_overhead"),
              "frac", v.get("pred_on", {}).get("frac_of_roofline"), v.get("error"))
    if "depth_sweep_1gpu" in p:
        print("depth sweep (1 GPU)", {k: (v["pred_off"], v["pred_on"], v["prediction_overhead"])
                                       for k, v in p["depth_sweep_1gpu"].items()})
