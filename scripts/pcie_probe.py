"""Host link bandwidth on this box: pinned H2D alone, D2H alone, and both at
once on two streams (the e2e step's transfer pattern), for the e2e roofline."""
import json
import sys

import torch


def probe(nbytes=671088640, reps=5):
    n = nbytes // 8
    h_in = torch.empty(n, dtype=torch.float64).pin_memory()
    h_out = torch.empty(n, dtype=torch.float64).pin_memory()
    d_a = torch.empty(n, dtype=torch.float64, device="cuda")
    d_b = torch.empty(n, dtype=torch.float64, device="cuda")
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()

    def timed(fn):
        fn()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(reps):
            fn()
        torch.cuda.current_stream().wait_stream(s1)
        torch.cuda.current_stream().wait_stream(s2)
        b.record()
        torch.cuda.synchronize()
        return a.elapsed_time(b) / reps / 1e3

    def h2d():
        s1.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s1):
            d_a.copy_(h_in, non_blocking=True)

    def d2h():
        s2.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s2):
            h_out.copy_(d_b, non_blocking=True)

    def both():
        h2d()
        d2h()

    t1, t2, t3 = timed(h2d), timed(d2h), timed(both)
    return {"bytes": nbytes, "h2d_gbs": nbytes / t1 / 1e9, "d2h_gbs": nbytes / t2 / 1e9,
            "bidir_gbs": 2 * nbytes / t3 / 1e9, "bidir_ms_per_gb_each_way": t3 * 1e3 / (nbytes / 1e9)}


def probe_buffers(host, reps=3):
    """The same measurement over the caller's own pinned buffers (e.g. the
    e2e mesh packets): H2D of every buffer on one stream while D2H into the
    buffers shifted by half the list runs on another; best of `reps`."""
    n = max(h.numel() for h in host)
    d_a = torch.empty(n, dtype=torch.float64, device="cuda")
    d_b = torch.empty(n, dtype=torch.float64, device="cuda")
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    K = len(host)
    nbytes = sum(h.numel() for h in host) * 8

    def run(h2d, d2h):
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        s1.wait_stream(torch.cuda.current_stream())
        s2.wait_stream(torch.cuda.current_stream())
        for i in range(K):
            if h2d:
                with torch.cuda.stream(s1):
                    d_a[:host[i].numel()].copy_(host[i].view(-1), non_blocking=True)
            if d2h:
                j = (i + K // 2) % K
                with torch.cuda.stream(s2):
                    host[j].view(-1).copy_(d_b[:host[j].numel()], non_blocking=True)
        torch.cuda.current_stream().wait_stream(s1)
        torch.cuda.current_stream().wait_stream(s2)
        b.record()
        torch.cuda.synchronize()
        return a.elapsed_time(b) / 1e3

    t1 = min(run(True, False) for _ in range(reps))
    t2 = min(run(False, True) for _ in range(reps))
    t3 = min(run(True, True) for _ in range(reps))
    return {"bytes": nbytes, "h2d_gbs": nbytes / t1 / 1e9, "d2h_gbs": nbytes / t2 / 1e9,
            "bidir_gbs": 2 * nbytes / t3 / 1e9}


if __name__ == "__main__":
    r = probe()
    print(json.dumps(r))
    if len(sys.argv) > 1:
        open(sys.argv[1], "w").write(json.dumps(r) + "\n")
