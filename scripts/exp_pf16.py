"""Experiment: prefill P as fp16 vs bf16 (tcgen05 A-format F16 against bf16 V)."""
import math, os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import oracle
import paper_2504_14489_b200 as mux
from synth import SideSpec, Shapes, make_side
from tests.helpers import gpu_build_side, oracle_build_side
for case, (r, n, outl) in enumerate([([0], [300], False), ([90], [200], True), ([0, 500], [1000, 64], False)]):
    side = make_side(730 + case, Shapes(8, 2, 128, 1), SideSpec(r, n), decode=False, outliers=outl)
    need = sum(side.spec.pages_needed()) + 7
    gs = gpu_build_side(mux, side, need, 11, 2, 128)
    os_ = oracle_build_side(side, need, 11, 2, 128)
    ref, _ = oracle.attention(side.q, os_["kpool"], os_["vpool"], os_["qo_indptr"], os_["kv_len"], os_["page_indptr"], os_["page_ids"], 1/math.sqrt(128))
    for f16 in ("0", "1"):
        os.environ["MUX_PF_PF16"] = f16
        o = torch.empty((side.spec.total_new, 8, 128), dtype=torch.float32, device="cuda")
        mux.mux_prefill_attn(gs["pool"], 0, gs["batch"], 8, gs["q"], o, None, scale=1/math.sqrt(128))
        torch.cuda.synchronize()
        d = np.abs(o.cpu().numpy() - ref)
        bad = (d > 2e-3 + 1e-2 * np.abs(ref)).sum()
        print(f"case {case} p_f16={f16}: max|d|={d.max():.3e} mean|d|={d.mean():.2e} bad={bad}", flush=True)
