"""PCIe duplex bandwidth vs pinned buffer size and copy chunking (measurement
tool): H2D + D2H at once over 16 GiB / 2 GiB pinned buffers, whole-buffer
copies vs the same bytes as 256 MiB chunks alternating over two streams per
direction."""
import json

import torch

for GB in (2, 16):
    N = GB << 30
    h_in = torch.empty(N, dtype=torch.uint8).pin_memory()
    h_out = torch.empty(N, dtype=torch.uint8).pin_memory()
    d_in = torch.empty(N, dtype=torch.uint8, device="cuda")
    d_out = torch.empty(N, dtype=torch.uint8, device="cuda")
    ups = [torch.cuda.Stream() for _ in range(2)]
    downs = [torch.cuda.Stream() for _ in range(2)]
    for chunk in (N, 256 << 20, 64 << 20):
        for rep in range(2):
            main = torch.cuda.current_stream()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(main)
            for s in ups + downs:
                s.wait_stream(main)
            for i in range(N // chunk):
                sl = slice(i * chunk, (i + 1) * chunk)
                with torch.cuda.stream(ups[i % 2]):
                    d_in[sl].copy_(h_in[sl], non_blocking=True)
                with torch.cuda.stream(downs[i % 2]):
                    h_out[sl].copy_(d_out[sl], non_blocking=True)
            for s in ups + downs:
                main.wait_stream(s)
            e1.record(main)
            e1.synchronize()
            t = e0.elapsed_time(e1) / 1e3
            print(json.dumps({"buffer_gib": GB, "chunk_mib": chunk >> 20, "duplex_total_gbs": 2 * N / t / 1e9}),
                  flush=True)
    del h_in, h_out, d_in, d_out
