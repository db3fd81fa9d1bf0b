"""Host<->device copy bandwidth of pinned buffers the size of bench.py's e2e
copies (x 32 MiB bf16 + logits 4 MiB f32 in, y 32 MiB out): one stream, two
streams, and H2D concurrent with D2H."""
import torch


def bw(fn, nbytes, iters=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(iters):
        fn()
    b.record()
    torch.cuda.synchronize()
    return nbytes * iters / (a.elapsed_time(b) / 1e3) / 1e9


def main():
    n = 8192 * 2048
    xh = torch.empty(n, dtype=torch.bfloat16).pin_memory()
    yh = torch.empty(n, dtype=torch.bfloat16).pin_memory()
    xd = torch.empty(n, dtype=torch.bfloat16, device="cuda")
    yd = torch.empty(n, dtype=torch.bfloat16, device="cuda")
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    nb = n * 2
    print(f"H2D one stream     {bw(lambda: xd.copy_(xh, non_blocking=True), nb):7.1f} GB/s")
    print(f"D2H one stream     {bw(lambda: yh.copy_(yd, non_blocking=True), nb):7.1f} GB/s")

    def two():
        h = n // 2
        with torch.cuda.stream(s1):
            xd[:h].copy_(xh[:h], non_blocking=True)
        with torch.cuda.stream(s2):
            xd[h:].copy_(xh[h:], non_blocking=True)
        torch.cuda.current_stream().wait_stream(s1)
        torch.cuda.current_stream().wait_stream(s2)
    print(f"H2D two streams    {bw(two, nb):7.1f} GB/s")

    def duplex():
        with torch.cuda.stream(s1):
            xd.copy_(xh, non_blocking=True)
        with torch.cuda.stream(s2):
            yh.copy_(yd, non_blocking=True)
        torch.cuda.current_stream().wait_stream(s1)
        torch.cuda.current_stream().wait_stream(s2)
    print(f"H2D+D2H duplex     {bw(duplex, 2 * nb):7.1f} GB/s (both directions)")


if __name__ == "__main__":
    main()
