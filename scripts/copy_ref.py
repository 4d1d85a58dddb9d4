"""Reference point for the flatten phase: what a plain device copy (torch's copy_, the
kernel MEASURED_PEAKS' hbm_gbs comes from) reaches on the same sizes.

  whole   one copy of the whole 1.5B gradient (Psi bf16 elements)
  bucket  51 copies of GPT-2 1.5B bucket sizes, back to back on one stream
  streams the same 51 copies rotated over 3 streams (as the library's flatten)

CUDA events around each phase, best of 10; bytes = read + write."""
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_1910_02054_b200 import plan_layout  # noqa: E402
import synth  # noqa: E402


def timed(fn, reps=10):
    best = None
    for _ in range(reps + 1):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        t = a.elapsed_time(b)
        best = t if best is None or t < best else best
    return best


def main():
    ts = synth.gpt2_1p5b()
    info, buckets, _ = plan_layout([t.numel for t in ts], [t.layer for t in ts], 1)
    sizes = [b.size for b in buckets]
    total = sum(sizes)
    src = torch.empty(total, dtype=torch.bfloat16, device="cuda").normal_()
    dst = torch.empty_like(src)
    views, o = [], 0
    for n in sizes:
        views.append((src[o:o + n], dst[o:o + n]))
        o += n
    streams = [torch.cuda.Stream() for _ in range(3)]
    main_s = torch.cuda.current_stream()

    def whole():
        dst.copy_(src)

    def bucket():
        for s_, d_ in reversed(views):
            d_.copy_(s_)

    def rotated():
        ev = torch.cuda.Event()
        ev.record(main_s)
        for i, (s_, d_) in enumerate(reversed(views)):
            st = streams[i % 3]
            st.wait_event(ev)
            with torch.cuda.stream(st):
                d_.copy_(s_)
        for st in streams:
            main_s.wait_stream(st)

    out = {"bench": "copy_ref", "elements": total, "buckets": len(sizes)}
    for name, fn in (("whole", whole), ("bucket", bucket), ("streams", rotated)):
        ms = timed(fn)
        out[name + "_ms"] = ms
        out[name + "_gbs"] = 4 * total / (ms * 1e-3) / 1e9
    print(json.dumps(out))


if __name__ == "__main__":
    main()
