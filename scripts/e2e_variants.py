"""Host-buffer (e2e) K3 path: PCIe throughput under different chunk sizes /
slot counts, plus the device-resident-params variant (G in, flag out)."""
import json
import sys
import time
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2312_00839_b200.optim import HostStreamer, OptimizerConfig, OptimizerState  # noqa: E402

dev = torch.device("cuda", 0)
n = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000_000
pin = lambda: torch.empty(n, dtype=torch.float32).pin_memory()  # noqa: E731
t0 = time.time()
w, g, wo, wh = pin(), pin(), pin(), pin()
print(json.dumps({"pin_s": round(time.time() - t0, 2)}), flush=True)
w.normal_(0, 0.02)
g.normal_(0, 1e-2)
for chunk_log2, slots in ((25, 3), (24, 4), (26, 3), (26, 4), (27, 2), (23, 6)):
    opt = OptimizerState(OptimizerConfig("adam"), ["flat"], device=dev, eager_checks=False)
    st = HostStreamer(dev, chunk_elems=1 << chunk_log2, slots=slots)
    st.step_predict(opt, w, g, 1e-3, 1e-3, 3, wo, wh)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(3):
        st.step_predict(opt, w, g, 1e-3, 1e-3, 3, wo, wh)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 3
    print(json.dumps({"chunk_log2": chunk_log2, "slots": slots, "ms": round(ms, 2),
                      "pcie_gbs_per_dir": round(8 * n / (ms * 1e-3) / 1e9, 1),
                      "algorithmic_gbs": round(32 * n / (ms * 1e-3) / 1e9, 1)}), flush=True)
    del st, opt
    torch.cuda.empty_cache()
# raw PCIe copies for reference
d = torch.empty(n, device=dev)
for name, fn in (("h2d", lambda: d.copy_(w, non_blocking=True)), ("d2h", lambda: wo.copy_(d, non_blocking=True))):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    fn()
    e1.record()
    torch.cuda.synchronize()
    print(json.dumps({name: round(4 * n / (e0.elapsed_time(e1) * 1e-3) / 1e9, 1)}), flush=True)
# both directions at once (the e2e step's bound: 8 B/param each way)
d2 = torch.empty(n, device=dev)
s_in, s_out = torch.cuda.Stream(), torch.cuda.Stream()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
s_in.wait_stream(torch.cuda.current_stream())
s_out.wait_stream(torch.cuda.current_stream())
with torch.cuda.stream(s_in):
    d.copy_(w, non_blocking=True)
    d2.copy_(g, non_blocking=True)
with torch.cuda.stream(s_out):
    wo.copy_(d2, non_blocking=True)
    wh.copy_(d, non_blocking=True)
torch.cuda.current_stream().wait_stream(s_in)
torch.cuda.current_stream().wait_stream(s_out)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1)
print(json.dumps({"bidirectional_8B_each_way_ms": round(ms, 1),
                  "bidirectional_gbs_per_dir": round(8 * n / (ms * 1e-3) / 1e9, 1)}), flush=True)
