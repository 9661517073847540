"""Device time of one full mine call (all 14 columns, device output), CUDA events on the launch
stream (GPU box): python tools/time_mine.py LIB [config]"""
import os, sys
sys.path.insert(0, ".")
os.environ["TM_LIB"] = os.path.abspath(sys.argv[1])
import torch
import paper_2604_12241_b200 as tmb
from paper_2604_12241_b200 import synth
g0 = synth.time_ordered(synth.generate(synth.CONFIGS[sys.argv[2] if len(sys.argv) > 2 else "hi-small"]))
g = tmb.DeviceGraph(g0.src, g0.dst, g0.time, node_count=g0.node_count)
descs = [tmb.lower_plan(p) for p in tmb.full_pattern_set(86400)]
out = torch.empty((g.edge_count, len(descs)), dtype=torch.int64, device="cuda")
st = torch.cuda.Stream()
for i in range(4):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    tmb.mine_rows_device(g, descs, 0, g.edge_count, out.data_ptr(), st.cuda_stream)
    e1.record(st)
    e1.synchronize()
    if i:
        print(f"{os.path.basename(sys.argv[1])}: full mine call {e0.elapsed_time(e1):.3f} ms", flush=True)
