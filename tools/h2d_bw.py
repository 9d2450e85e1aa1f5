"""Host->device copy bandwidth from pinned memory (dev tool): the out-of-core
database's bound."""
import json, torch
torch.cuda.set_device(0)
st = torch.cuda.Stream()
for nbytes, dt in [(134 << 20, torch.uint16), (268 << 20, torch.int32), (1 << 30, torch.uint16)]:
    h = torch.empty(nbytes // (2 if dt == torch.uint16 else 4), dtype=dt, pin_memory=True)
    d = torch.empty_like(h, device="cuda")
    for off in (0, 1):
        src = h[off:]
        dst = d[off:]
        with torch.cuda.stream(st):
            dst.copy_(src, non_blocking=True)
        st.synchronize()
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(st)
        with torch.cuda.stream(st):
            for _ in range(3):
                dst.copy_(src, non_blocking=True)
        e1.record(st); st.synchronize()
        ms = e0.elapsed_time(e1) / 3
        print(json.dumps({"bytes": src.numel() * src.element_size(), "dtype": str(dt), "offset_elems": off,
                          "ms": round(ms, 3), "GBps": round(src.numel() * src.element_size() / ms / 1e6, 1)}))
