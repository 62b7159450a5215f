import sys, json, torch
sys.path.insert(0, '/root/repo')
from paper_1708_01873_b200 import _core
dev = torch.device('cuda', 0)
b = 26
x = torch.empty((1 << b) * 8, dtype=torch.uint8, device=dev).random_(0, 256).view(torch.float64)
st = torch.cuda.current_stream()
step = lambda: _core.launch_inplace(x, b)
for _ in range(20): step()
torch.cuda.synchronize()
K = 20
for rep in range(3):
    # per-step events
    ss = [torch.cuda.Event(enable_timing=True) for _ in range(K)]; ee = [torch.cuda.Event(enable_timing=True) for _ in range(K)]
    for k in range(K):
        ss[k].record(st); step(); ee[k].record(st)
    torch.cuda.synchronize()
    per = sum(s.elapsed_time(e) for s, e in zip(ss, ee)) / K
    # one pair around K steps
    s0, e0 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s0.record(st)
    for k in range(K): step()
    e0.record(st); torch.cuda.synchronize()
    whole = s0.elapsed_time(e0) / K
    # per-step events, spans between consecutive starts (includes gaps)
    span = ss[0].elapsed_time(ee[-1]) / K
    print(json.dumps({"per_step_us": per * 1e3, "one_pair_us": whole * 1e3, "span_us": span * 1e3,
                      "gbs_per_step": 2 * 8 * (1 << b) / (per / 1e3) / 1e9,
                      "gbs_one_pair": 2 * 8 * (1 << b) / (whole / 1e3) / 1e9}))
