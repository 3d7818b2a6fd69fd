import faulthandler, sys, time, json
sys.path.insert(0, '.')
import torch
from paper_2312_00839_b200 import bench_pipeline as bp
faulthandler.dump_traceback_later(100, repeat=True)
dev = torch.device('cuda', 0)
for i in range(int(sys.argv[1])):
    t = time.time()
    r = bp.single_gpu_module_pipeline(torch, dev, 'config3_resnet101', n_batches=16)
    print(i, round(time.time() - t, 1), r['pred_off']['samples_per_s'], r['pred_on']['samples_per_s'], torch.cuda.max_memory_allocated() / 1e9, file=sys.stderr, flush=True)
