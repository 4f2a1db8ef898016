"""Host->device copy bandwidth from pinned memory on cuda:0: one stream vs
two / four streams, chunk sizes 16..256 MiB (sizing the e2e path's chunked
H2D, capi.cu kChunkBytes)."""
import json

import torch

N = 2 << 30
src = torch.empty(N, dtype=torch.uint8).pin_memory()
dst = torch.empty(N, dtype=torch.uint8, device="cuda")
res = {}
for streams in (1, 2, 4):
    ss = [torch.cuda.Stream() for _ in range(streams)]
    for chunk_mb in (16, 64, 256, 2048):
        chunk = chunk_mb << 20
        best = 0.0
        for rep in range(4):
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for s in ss:
                s.wait_event(e0)
            for k, off in enumerate(range(0, N, chunk)):
                with torch.cuda.stream(ss[k % streams]):
                    dst[off:off + chunk].copy_(src[off:off + chunk], non_blocking=True)
            for s in ss:
                torch.cuda.current_stream().wait_stream(s)
            e1.record()
            e1.synchronize()
            best = max(best, N / (e0.elapsed_time(e1) * 1e-3) / 1e9)
        res[f"{streams}x{chunk_mb}MiB"] = round(best, 2)
        print(streams, chunk_mb, round(best, 2), "GB/s", flush=True)
print(json.dumps(res))
