"""Host memory copy bandwidth, pageable <-> pinned, over 1..16 threads (the
staging copies of the host-pointer path for pageable buffers).  One JSON line
per (direction, threads).  Usage: python tools/host_copy_probe.py [--gib 2]"""
import argparse
import json
import threading
import time

import numpy as np
import torch

ap = argparse.ArgumentParser()
ap.add_argument("--gib", type=float, default=2.0)
a = ap.parse_args()
n = int(a.gib * (1 << 30)) // 8
page = np.ones(n, np.float64)
pin = torch.empty(n, dtype=torch.float64, pin_memory=True).numpy()
pin[:] = 2.0


def run(dst, src, threads):
    parts = np.array_split(np.arange(n), threads)
    spans = [(p[0], p[-1] + 1) for p in parts if p.size]

    def w(lo, hi):
        np.copyto(dst[lo:hi], src[lo:hi])

    ts = [threading.Thread(target=w, args=s) for s in spans]
    t0 = time.perf_counter()
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    return time.perf_counter() - t0


for name, dst, src in (("pageable_to_pinned", pin, page), ("pinned_to_pageable", page, pin)):
    for th in (1, 4, 8, 16):
        run(dst, src, th)
        best = min(run(dst, src, th) for _ in range(3))
        print(json.dumps({"copy": name, "threads": th, "gbs": round(n * 8 / best / 1e9, 2)}), flush=True)
