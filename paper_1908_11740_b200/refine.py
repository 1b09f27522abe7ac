"""ε-distance refinement of candidate pairs on the device (engine.py:189-207)."""

from __future__ import annotations

import ctypes as C

import numpy as np
import torch

from . import _native
from .geometry import RectBatch


def refine_distance(cand: torch.Tensor, p: RectBatch, q: RectBatch, eps_sq: float):
    """Filter (row_p, row_q) candidates by ``dx*dx + dy*dy <= eps_sq``.

    Point coordinates are the lower corners of ``p`` / ``q`` (engine.py:333-334);
    the kept pairs are returned as (p_id, q_id) in candidate order.
    """
    lib = _native.load()
    device = cand.device
    n = int(cand.shape[0])
    if n == 0:
        return 0, torch.empty((0, 2), dtype=torch.int64, device=device)

    def put(a, dt):
        return torch.from_numpy(np.ascontiguousarray(a)).to(device=device, dtype=dt)

    px, py = put(p.xl, torch.float64), put(p.yl, torch.float64)
    qx, qy = (px, py) if q is p else (put(q.xl, torch.float64), put(q.yl, torch.float64))
    pid = put(p.ids, torch.int64)
    qid = pid if q is p else put(q.ids, torch.int64)
    cand = cand.contiguous()
    scratch = torch.empty(int(lib.pbsm_refine_scratch_bytes(n)), dtype=torch.uint8,
                          device=device)
    out = torch.empty((n, 2), dtype=torch.int64, device=device)
    stream = torch.cuda.current_stream(device).cuda_stream
    _native.check(lib.pbsm_refine(cand.data_ptr(), n, px.data_ptr(), py.data_ptr(),
                                  qx.data_ptr(), qy.data_ptr(), pid.data_ptr(), qid.data_ptr(),
                                  C.c_double(eps_sq), scratch.data_ptr(), out.data_ptr(),
                                  stream), "pbsm_refine")
    off = int(lib.pbsm_refine_result_offset(n))
    kept = int(scratch[off:off + 8].view(torch.int64).item())
    return kept, out[:kept]
