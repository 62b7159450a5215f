"""PCIe copy bandwidth on the GPU host (measurement tool): pinned H2D, D2H and
both at once, each direction split over 1/2/4 streams in equal chunks."""
import json

import torch

N = 2 << 30  # bytes per direction
h_in = torch.empty(N, dtype=torch.uint8).pin_memory()
h_out = torch.empty(N, dtype=torch.uint8).pin_memory()
d_in = torch.empty(N, dtype=torch.uint8, device="cuda")
d_out = torch.empty(N, dtype=torch.uint8, device="cuda")
streams = [torch.cuda.Stream() for _ in range(8)]


def run(k, up, down):
    main = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(main)
    c = N // k
    for i in range(k):
        if up:
            s = streams[i]
            s.wait_stream(main)
            with torch.cuda.stream(s):
                d_in[i * c:(i + 1) * c].copy_(h_in[i * c:(i + 1) * c], non_blocking=True)
        if down:
            s = streams[4 + i] if k <= 4 else streams[i]
            s.wait_stream(main)
            with torch.cuda.stream(s):
                h_out[i * c:(i + 1) * c].copy_(d_out[i * c:(i + 1) * c], non_blocking=True)
    for s in streams:
        main.wait_stream(s)
    e1.record(main)
    e1.synchronize()
    t = e0.elapsed_time(e1) / 1e3
    return (N * (int(up) + int(down))) / t / 1e9


for rep in range(2):
    for k in (1, 2, 4):
        print(json.dumps({"streams_per_direction": k, "h2d_gbs": run(k, True, False),
                          "d2h_gbs": run(k, False, True), "duplex_total_gbs": run(k, True, True)}))
