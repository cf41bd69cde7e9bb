"""HBM probes at the BLAST split-path sizes (3.1 GB): write-only fill, read-only reduction and
copy, CUDA-event timed after an L2-sized write flush.  python scripts/hbm_probe.py"""
import torch

dev = torch.device("cuda")
N = 65536 * 16 * 1488  # fp16 elements of Z at Llama-7B / C4
a = torch.empty(N, dtype=torch.float16, device=dev).normal_()
b = torch.empty_like(a)
flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)


def t(fn, reps=5):
    best = 1e9
    for _ in range(reps):
        flush.fill_(1)
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        fn()
        e.record()
        torch.cuda.synchronize()
        best = min(best, s.elapsed_time(e))
    return best


GB = N * 2 / 1e9
for name, fn, nbytes in [("fill (write)", lambda: b.fill_(0.5), GB), ("sum (read)", lambda: a.sum(), GB),
                         ("copy (r+w)", lambda: b.copy_(a), 2 * GB)]:
    ms = t(fn)
    print(f"{name:14s} {ms:7.3f} ms  {nbytes / ms:6.2f} TB/s  ({nbytes:.2f} GB)")
