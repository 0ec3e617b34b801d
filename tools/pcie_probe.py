"""PCIe context for the e2e numbers: pinned H2D, D2H and both at once (1.086 GB, the
config-2 upload), CUDA events, best of 5.  Prints one JSON line."""
import json

import torch


def main():
    nb = 514 * 514 * 514 * 8
    h = torch.empty(nb, dtype=torch.uint8, pin_memory=True)
    h2 = torch.empty(nb, dtype=torch.uint8, pin_memory=True)
    d = torch.empty(nb, dtype=torch.uint8, device="cuda")
    d2 = torch.empty(nb, dtype=torch.uint8, device="cuda")
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    out = {}

    def best(fn):
        t = 1e30
        for _ in range(5):
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            fn()
            e1.record()
            torch.cuda.synchronize()
            t = min(t, e0.elapsed_time(e1))
        return t

    def h2d():
        d.copy_(h, non_blocking=True)

    def d2h():
        h2.copy_(d2, non_blocking=True)

    def both():
        cur = torch.cuda.current_stream()
        s1.wait_stream(cur)
        s2.wait_stream(cur)
        with torch.cuda.stream(s1):
            d.copy_(h, non_blocking=True)
        with torch.cuda.stream(s2):
            h2.copy_(d2, non_blocking=True)
        cur.wait_stream(s1)
        cur.wait_stream(s2)

    for name, fn in (("h2d", h2d), ("d2h", d2h), ("both", both)):
        ms = best(fn)
        out[name] = {"ms": ms, "GBps_each_way": nb / ms / 1e6}
    out["bytes"] = nb
    print(json.dumps(out))


if __name__ == "__main__":
    main()
