"""Where bench.py's e2e time goes (config B, one GPU): the streamed
pipeline of run_e2e with its host->device inputs and device->host outputs,
then without the output copy, without the input copy, and the replays alone
(ms per step, 20 steps after warm-up)."""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2601_08800_b200 import SwiGLUExperts  # noqa: E402
from paper_2601_08800_b200.layer import MoELayer  # noqa: E402

T, H, E, K, I = 8192, 2048, 128, 8, 768


def main():
    ex = SwiGLUExperts.random(E, H, I, seed=0)
    w13, w2 = ex.rank_shard(1, 1, 0)
    layer = MoELayer(1, 1, T, H, E, K, I, w13=w13, w2=w2, rank=0)
    g = torch.Generator(device="cuda").manual_seed(1000)
    x = torch.randn(T, H, device="cuda", generator=g).to(torch.bfloat16)
    logits = torch.randn(T, E, device="cuda", generator=g)
    x_h, l_h = x.cpu().pin_memory(), logits.cpu().pin_memory()
    y_hs = [torch.empty(T, H, dtype=torch.bfloat16).pin_memory() for _ in range(2)]
    xs, ls = [x, x.clone()], [logits, logits.clone()]
    runs = [layer.capture(xs[0], ls[0]), layer.capture(xs[1], ls[1])]
    stream = torch.cuda.current_stream()
    h2d_s, d2h_s = torch.cuda.Stream(), torch.cuda.Stream()

    def pipeline(steps, h2d=True, d2h=True, direct=False):
        ev_in = [torch.cuda.Event() for _ in range(2)]
        ev_free = [torch.cuda.Event() for _ in range(2)]
        ev_out = [torch.cuda.Event() for _ in range(2)]
        y_stage = [torch.empty(T, H, dtype=torch.bfloat16, device="cuda") for _ in range(2)]

        def h2d_step(i):
            b = i % 2
            if i >= 2:
                h2d_s.wait_event(ev_free[b])
            with torch.cuda.stream(h2d_s):
                xs[b].copy_(x_h, non_blocking=True)
                ls[b].copy_(l_h, non_blocking=True)
            ev_in[b].record(h2d_s)

        torch.cuda.synchronize()
        a, bb = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        h2d_s.wait_event(a)
        d2h_s.wait_event(a)
        if h2d:
            h2d_step(0)
        for i in range(steps):
            b = i % 2
            if h2d and i + 1 < steps:
                h2d_step(i + 1)
            if h2d:
                stream.wait_event(ev_in[b])
            y = runs[b]()
            ev_free[b].record(stream)
            if d2h:
                if direct:      # D2H straight from the layer's y (no staging copy)
                    ev_out[b].record(stream)
                    d2h_s.wait_event(ev_out[b])
                    with torch.cuda.stream(d2h_s):
                        y_hs[b].copy_(y, non_blocking=True)
                    stream.wait_stream(d2h_s)   # y is overwritten by the next replay
                else:
                    y_stage[b].copy_(y, non_blocking=True)
                    ev_out[b].record(stream)
                    d2h_s.wait_event(ev_out[b])
                    with torch.cuda.stream(d2h_s):
                        y_hs[b].copy_(y_stage[b], non_blocking=True)
        stream.wait_stream(h2d_s)
        stream.wait_stream(d2h_s)
        bb.record(stream)
        torch.cuda.synchronize()
        return a.elapsed_time(bb) / steps

    for name, kw in (("full", {}), ("no_d2h", {"d2h": False}), ("no_h2d", {"h2d": False}),
                     ("replays", {"h2d": False, "d2h": False}), ("full_again", {})):
        pipeline(3, **kw)
        print(f"{name:12s} {pipeline(20, **kw):.3f} ms/step", flush=True)


if __name__ == "__main__":
    main()
