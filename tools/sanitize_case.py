"""Small workload that touches every kernel and entry point, for
compute-sanitizer (memcheck / racecheck / synccheck, one tool per run):

    compute-sanitizer --tool memcheck python tools/sanitize_case.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2502_10831_b200 as ft  # noqa: E402

n = 20011  # ragged: not a multiple of any vector or block size
for dt in (torch.float32, torch.float64):
    base = ft.gen_inputs(n + 1, dt, 0, -3000.0, 3000.0, 7)
    for x in (base[:n], base[1:]):  # aligned and misaligned views
        for mask in range(1, 8):
            for mode in (ft.SqrtMode(), ft.SqrtMode.exact(), ft.SqrtMode.fisr(3)):
                out = ft.proposed_eval(x.contiguous() if x.storage_offset() == 0 else x, mask, mode)
            ft.proposed_eval(x, mask, seg=True)
            ft.taylor_eval(x, 5, mask)
            ft.taylor_eval(x, 4, mask)
        out = ft.proposed_eval(x, 7, seg=True)
        ft.parity_reduce(x, out, 7, check_seg=True)
        ft.parity_reduce(x, out, 7, refs={k: out[k] for k in ("sin", "cos", "tan")})
        ft.mirror_eval(x, 7, 0, seg=True)
        ft.mirror_eval(x, 7, 1, n_terms=7)
    ft.gen_inputs(n, dt, 1, -1000.0, 1000.0, 3, offset=12345)
xh = np.linspace(-10, 10, n)
ft.proposed_sin_batch(xh)
ft.proposed_batch(xh.astype(np.float32), 5)
ft.taylor_batch(xh, 9, 7)
ft.l2_flush()
torch.cuda.synchronize()
print("sanitize case OK,", ft.launch_count(), "launches")
