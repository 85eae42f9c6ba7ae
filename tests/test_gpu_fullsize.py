"""Full-size sampled parity (GPU): BASELINE configs 2-5 at their full shapes, run through
mux_run_layer on a real SM split exactly as bench.py launches them (append + attention +
out-projection on each side, decode balanced split-KV heuristic), compared with the oracle on
sampled outputs the oracle computes one by one: sampled prefill rows (tile boundaries, first,
last, spread; synth.sample_rows) and sampled decode sequences (longest, shortest, first, last,
random).  Inputs of everything the oracle checks come from synth's seeded host generators;
the decode sequences that are NOT checked are filled on the device (only their bytes' presence
matters: they occupy the batch / grid exactly as in the bench)."""
import math

import numpy as np
import pytest

import oracle
import synth
from synth import SideData, SideSpec, indptr
from tests.helpers import check_close, oracle_build_side

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def mux():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import paper_2504_14489_b200 as m
    m.lib()
    return m


@pytest.fixture(scope="module")
def part(mux):
    p = mux.Partition(0, mux.mux_partition_configs(mux.mux_device_sm_count(0), 16, 12))
    yield p
    p.close()


def _decode_rows(cfg, S, L, b):
    """Host rows of decode sequence b from its own seeded stream (so any subset can be made)."""
    k = synth.bf16_normal(synth.rng(cfg, synth.T_K_DC, salt=1000 + b), (L, S.Hkv, S.d))
    v = synth.bf16_normal(synth.rng(cfg, synth.T_V_DC, salt=1000 + b), (L, S.Hkv, S.d))
    return k, v


def _to_dev(a):
    import torch
    return torch.from_numpy(np.ascontiguousarray(a).view(np.int16)).cuda().view(torch.bfloat16)


@pytest.mark.parametrize("cfg,split", [(2, 1), (3, 1), (4, 2), (5, 0)])
def test_fullsize_sampled_parity(mux, part, cfg, split):
    import torch
    c = synth.get_config(cfg)
    S = c.shapes
    Hq, Hkv, d, hidden = S.Hq, S.Hkv, S.d, S.hidden
    scale = 1.0 / math.sqrt(d)
    pf_spec, dc_spec = c.prefill, c.decode
    B = dc_spec.num_seqs
    L_dc = dc_spec.L
    g = np.random.default_rng(cfg)
    samp = sorted({0, B - 1, int(np.argmax(L_dc)), int(np.argmin(L_dc))} |
                  {int(x) for x in g.choice(B, 4, replace=False)})

    # ---- inputs
    pside = synth.make_side(cfg, S, pf_spec, decode=False)
    dq = synth.bf16_normal(synth.rng(cfg, synth.T_Q_DC, salt=1000), (B, Hq, d))
    wo = synth.make_wo(cfg, S)
    pages = sum(pf_spec.pages_needed()) + sum(dc_spec.pages_needed()) + 8
    kst = torch.full((1, pages, Hkv, 16, d), 0x7FC0, dtype=torch.int16, device="cuda").view(torch.bfloat16)
    pool = mux.Pool(1, pages, Hkv, d, synth.free_list_seed(cfg), kst, kst.clone())
    # prefill: all rows from the host
    ppi, ppd = pool.page_tables(pf_spec.pages_needed())
    mux.mux_append_kv(pool, 0, mux.Batch(indptr(pf_spec.L), pf_spec.L, ppi, ppd),
                      _to_dev(np.concatenate(pside.k_rows)), _to_dev(np.concatenate(pside.v_rows)))
    # decode: sampled sequences from the host, the others filled on the device
    dpi, dpd = pool.page_tables(dc_spec.pages_needed())
    rows = int(sum(L_dc))
    kd = torch.empty((rows, Hkv, d), dtype=torch.bfloat16, device="cuda").normal_()
    vd = torch.empty_like(kd).normal_()
    off = indptr(L_dc)
    host = {}
    for b in samp:
        k, v = _decode_rows(cfg, S, L_dc[b], b)
        host[b] = (k, v)
        kd[off[b]:off[b + 1]] = _to_dev(k)
        vd[off[b]:off[b + 1]] = _to_dev(v)
    mux.mux_append_kv(pool, 0, mux.Batch(indptr(L_dc), L_dc, dpi, dpd), kd, vd)
    # the steps' new rows (re-appended by run_layer, exactly as in the bench)
    new_idx = [off[b + 1] - 1 for b in range(B)]
    dk_new, dv_new = kd[new_idx].contiguous(), vd[new_idx].contiguous()
    pk_new = _to_dev(pside.k_new())
    pv_new = _to_dev(pside.v_new())

    # ---- the bench's launch: one mux_run_layer on `split`, append + attention + out-projection
    dsms = part.query(split)[0]
    ns = mux.mux_decode_num_splits(B, Hkv, max(L_dc), dsms, L_dc, d)
    ws = torch.empty(max(16, mux.mux_decode_workspace_bytes(B, Hq, d, ns)), dtype=torch.uint8, device="cuda")
    w_pk = mux.mux_outproj_pack_w(_to_dev(wo))
    o_pf = torch.empty((pf_spec.total_new, Hq, d), dtype=torch.bfloat16, device="cuda")
    o_dc = torch.empty((B, Hq, d), dtype=torch.bfloat16, device="cuda")
    y_pf = torch.empty((pf_spec.total_new, hidden), dtype=torch.float32, device="cuda")
    y_dc = torch.empty((B, hidden), dtype=torch.float32, device="cuda")
    s_pf = mux.make_side(mux.Batch(indptr(pf_spec.n), pf_spec.L, ppi, ppd), Hq, _to_dev(pside.q), o_pf,
                         k_new=pk_new, v_new=pv_new, scale=scale, append=True, w_o=w_pk, y=y_pf)
    s_dc = mux.make_side(mux.Batch(indptr([1] * B), L_dc, dpi, dpd), Hq, _to_dev(dq), o_dc, k_new=dk_new,
                         v_new=dv_new, scale=scale, append=True, num_splits=ns, ws=ws, w_o=w_pk, y=y_dc)
    mux.mux_run_layer(part, split, pool, s_pf, s_dc, None)
    torch.cuda.synchronize()
    assert pool.error_flags() == 0
    # the same attention kernels with fp32 outputs on the same partition streams (after the step's
    # append, so over the same pool): R8's strict fp32 bound below, and the step's bf16 outputs
    # must be exactly the round-to-nearest-even of these (same fp32 value, one rounding)
    _, _, sd, sp = part.query(split)
    o_pf32 = torch.empty((pf_spec.total_new, Hq, d), dtype=torch.float32, device="cuda")
    o_dc32 = torch.empty((B, Hq, d), dtype=torch.float32, device="cuda")
    mux.mux_prefill_attn(pool, 0, s_pf._keep[0], Hq, _to_dev(pside.q), o_pf32, None, scale=scale, stream=sp)
    mux.mux_decode_attn(pool, 0, s_dc._keep[0], Hq, _to_dev(dq), o_dc32, None, scale=scale, num_splits=ns, ws=ws,
                        stream=sd)
    torch.cuda.synchronize()
    assert torch.equal(o_pf32.to(torch.bfloat16), o_pf), "prefill bf16 output != rne(fp32 output)"
    assert torch.equal(o_dc32.to(torch.bfloat16), o_dc), "decode bf16 output != rne(fp32 output)"

    # ---- oracle on the samples (512 rows at cfg5, >= 128 at cfg2-4, late tiles included)
    prow = synth.sample_rows_tiles(pf_spec.total_new, 512 if cfg == 5 else 160)
    assert (prow >= pf_spec.total_new - 4 * 128).sum() >= 8
    os_ = oracle_build_side(pside, sum(pf_spec.pages_needed()) + 1, 3, Hkv, d)
    ref_p, _ = oracle.attention(pside.q, os_["kpool"], os_["vpool"], os_["qo_indptr"], os_["kv_len"],
                                os_["page_indptr"], os_["page_ids"], scale, rows=prow)
    got_p = o_pf.float().cpu().numpy()[prow]
    check_close(got_p, ref_p, what=f"cfg{cfg} prefill sampled rows", out_bf16=True)
    check_close(o_pf32.cpu().numpy()[prow], ref_p, what=f"cfg{cfg} prefill sampled rows (fp32 out)")
    sub = SideData(SideSpec([L_dc[b] - 1 for b in samp], [1] * len(samp)), dq[samp],
                   [host[b][0] for b in samp], [host[b][1] for b in samp])
    od = oracle_build_side(sub, sum(sub.spec.pages_needed()) + 1, 4, Hkv, d)
    ref_d, _ = oracle.attention(sub.q, od["kpool"], od["vpool"], od["qo_indptr"], od["kv_len"],
                                od["page_indptr"], od["page_ids"], scale)
    got_d = o_dc.float().cpu().numpy()[samp]
    check_close(got_d, ref_d, what=f"cfg{cfg} decode sampled sequences", out_bf16=True)
    check_close(o_dc32.cpu().numpy()[samp], ref_d, what=f"cfg{cfg} decode sampled sequences (fp32 out)")
    # out-projection of the same samples (R22: bf16(O) . W_o)
    for got_y, ref_o in ((y_pf.cpu().numpy()[prow], ref_p), (y_dc.cpu().numpy()[samp], ref_d)):
        ob = synth.f32_to_bf16_bits(ref_o.reshape(ref_o.shape[0], -1).astype(np.float32))
        check_close(got_y, oracle.outproj(ob, wo), what=f"cfg{cfg} y sampled rows")
    pool.close()
