"""Multi-device contexts (poslo_gpu_create_multi) and the C-ABI additions of
round 2, on one B200: members may share a device, which runs the sharded
code path (epoch cuts, per-member streams and threads, rank-ordered folds of
partials on member 0) on one GPU. Every output must be byte-identical to the
single-device context — the SURVEY §8e determinism gate for the in-process
split — and to the reference's goldens.

Also: poslo_batch.fill producers (the drop-in's pinned, pipelined gather),
entry-layout validation (offsets outside the payload are refused, not read),
the process-wide group-operation counters (group.hpp:86-97 units), the
partial e-hat / combine_check pair of the multi-rank PAVer, and SeBVer with
only the messages it reads (distiller.cpp:140-233)."""
import ctypes
import random

import numpy as np
import pytest

from conftest import STREAMS, load_golden
from golden_util import Stream

pytestmark = pytest.mark.gpu


def _api():
    from paper_2506_08781_b200 import api
    return api


@pytest.fixture(scope="module")
def multi():
    v = _api().Verifier(devices=[0, 0, 0])
    assert v.members() == 3
    yield v
    v.close()


@pytest.fixture(scope="module")
def signed():
    """Config-5-shaped slice: 2^22 x 32 B, n2 = 1024 (4096 epochs), signed by the
    reference derivation, 16 entries tampered after signing."""
    from paper_2506_08781_b200.synth import SignedLog
    v = _api().Verifier(0)
    sl = SignedLog(v, 0, 4096, 1024, 12, seed=77)
    sl.tamper(16, seed=5)
    sl.host = sl.log.cpu().numpy()
    yield v, sl
    v.close()


def _host_batch(sl, pay):
    b = sl.batch(device_resident=False, payload_ptr=pay.ctypes.data)
    return b


# ------------------------------------------------------------------ goldens through a 3-member context
@pytest.mark.parametrize("name", STREAMS)
def test_multi_context_matches_reference_goldens(multi, name):
    st = Stream(load_golden(name + ".json"))
    suite, pk, ds = st.api_objects()
    parts, e_hat = multi.agg_ekeys(suite, st.batches, ds, 4)
    assert [p[1] for p in parts] == st.e_tilde and e_hat == st.e_hat
    assert multi.paver(pk, st.batches, st.s_hat, None, ds, 4) == bool(st.d["paver"])
    assert multi.paver(pk, st.batches, st.s_hat, st.r_hat_agg, ds, 4) == bool(st.d["paver_agg"])
    s_hats = {i: st.sigs[i].s_hat_le for i in range(st.n1)}
    assert [int(x) for x in multi.epoch_verify(pk, st.batches, s_hats, ds)] == st.d["epoch_verdicts"]


@pytest.mark.parametrize("name", ["stream_s1_tamper", "stream_s1_clean_big", "stream_s2_mixed"])
def test_multi_context_distillation_ccd_bytes(multi, name):
    """Batched distillation on the 3-member context leaves the reference's CCD
    bytes: umbrella pieces split by the member cuts are folded back."""
    from paper_2506_08781_b200.distill import ColdCryptoData
    api = _api()
    st = Stream(load_golden(name + ".json"))
    suite = api.SuiteConfig(st.suite, st.n1, st.n2, st.n_u)
    pk = api.PoslocPublicKey.deserialize(bytes.fromhex(st.d["pk"]), multi)
    sigs = [api.EpochSignature.deserialize(bytes.fromhex(s), st.depth)[0] for s in st.d["sigs"]]
    ccd = ColdCryptoData(ord("C"), suite, multi)
    ccd.distill_epochs(pk, [st.batches[i] for i in range(st.n1)], sigs)
    ccd.finalize()
    assert ccd.serialize().hex() == st.d["ccd"]


# ------------------------------------------------------------------ sharded == single at 2^22
def test_multi_context_byte_identical_at_scale(signed, multi):
    v, sl = signed
    lib = v._lib
    pay = sl.host
    n1 = sl.n1
    # agg_ekeys: e~ and e-hat
    outs = []
    for ctx in (v, multi):
        et, eh = ctypes.create_string_buffer(32 * n1), ctypes.create_string_buffer(32)
        b = _host_batch(sl, pay)
        ctx._call(lib.poslo_gpu_agg_ekeys, ctypes.byref(b), et, eh)
        outs.append((et.raw, eh.raw))
    assert outs[0] == outs[1]
    # per-epoch verdicts: exactly the tampered epochs fail, on both
    verd = []
    for ctx in (v, multi):
        vb = ctypes.create_string_buffer(n1)
        b = _host_batch(sl, pay)
        ctx._call(lib.poslo_gpu_epoch_verify, ctypes.byref(b), sl.Y, sl.s_hats, sl.r_hats, vb, None)
        verd.append(vb.raw)
    assert verd[0] == verd[1]
    assert [i for i in range(n1) if not verd[0][i]] == sl.bad_epochs()
    # distillation pieces on umbrellas of 96 epochs (not aligned with the 3-way cuts)
    cuts = np.array(list(range(0, n1, 96)) + [n1], dtype=np.uint32)
    ng = len(cuts) - 1
    res = []
    for ctx in (v, multi):
        vb = ctypes.create_string_buffer(n1)
        o = [ctypes.create_string_buffer(32 * ng) for _ in range(3)]
        b = _host_batch(sl, pay)
        ctx._call(lib.poslo_gpu_distill_coarse_ex, ctypes.byref(b), sl.Y, sl.s_hats, sl.r_hats,
                  ctypes.c_void_p(cuts.ctypes.data), ng, vb, *o)
        res.append((vb.raw, o[0].raw, o[1].raw, o[2].raw))
    assert res[0] == res[1]
    # segment e-sums = sum of the valid epochs' e~
    et = outs[0][0]
    for g in (0, 7, ng - 1):
        ok = [i for i in range(cuts[g], cuts[g + 1]) if verd[0][i]]
        assert res[0][3][32 * g:32 * g + 32] == v.scalar_sum([et[32 * i:32 * i + 32] for i in ok])
    # coarse paver over the untampered prefix: accepted in aggregate and fold mode
    m = min(sl.bad_epochs()[0], 1024)
    assert m >= 2
    sub = _host_batch(sl, pay)
    sub.n_epochs, sub.n_entries = m, m * sl.n2
    S = v.scalar_sum([sl.s_hats[32 * i:32 * i + 32] for i in range(m)])
    R = v.group_fold([sl.r_hats[32 * i:32 * i + 32] for i in range(m)])
    for ctx in (v, multi):
        vd = ctypes.c_uint8(0)
        ctx._call(lib.poslo_gpu_paver, ctypes.byref(sub), sl.Y, S, R, None, ctypes.byref(vd))
        assert vd.value == 1
        ctx._call(lib.poslo_gpu_paver, ctypes.byref(sub), sl.Y, S, None, sl.r_hats[:32 * m], ctypes.byref(vd))
        assert vd.value == 1
    # whole log with its tampers is rejected by both
    b = _host_batch(sl, pay)
    Sall = v.scalar_sum([sl.s_hats[32 * i:32 * i + 32] for i in range(n1)])
    Rall = v.group_fold([sl.r_hats[32 * i:32 * i + 32] for i in range(n1)])
    for ctx in (v, multi):
        vd = ctypes.c_uint8(1)
        ctx._call(lib.poslo_gpu_paver, ctypes.byref(b), sl.Y, Sall, Rall, None, ctypes.byref(vd))
        assert vd.value == 0


@pytest.mark.parametrize("comb16", [False, True])
def test_determinism_gate_1_2_4_8_members(signed, comb16, monkeypatch):
    """SURVEY §8e's gate at G = 1, 2, 4 and 8 (members sharing the one GPU):
    every e~, e-hat, the per-epoch verdict bitmap and the distillation pieces
    (umbrellas of 96 epochs, not aligned with any shard cut) are byte-identical
    to one device, and the coarse paver decision agrees — on the radix-256
    checks against decoded R-hat and (comb16: POSLO_COMB16_MIN = 1) on the
    radix-2^16 checks with no square root, whose umbrella folds add the
    checks' own points."""
    if comb16:
        monkeypatch.setenv("POSLO_COMB16_MIN", "1")
    v, sl = signed
    lib = v._lib
    pay, n1 = sl.host, sl.n1
    cuts = np.array(list(range(0, n1, 96)) + [n1], dtype=np.uint32)
    ng = len(cuts) - 1
    S = v.scalar_sum([sl.s_hats[32 * i:32 * i + 32] for i in range(n1)])
    R = v.group_fold([sl.r_hats[32 * i:32 * i + 32] for i in range(n1)])

    def outputs(ctx):
        et, eh = ctypes.create_string_buffer(32 * n1), ctypes.create_string_buffer(32)
        ctx._call(lib.poslo_gpu_agg_ekeys, ctypes.byref(_host_batch(sl, pay)), et, eh)
        vb = ctypes.create_string_buffer(n1)
        ctx._call(lib.poslo_gpu_epoch_verify, ctypes.byref(_host_batch(sl, pay)), sl.Y, sl.s_hats, sl.r_hats,
                  vb, None)
        db = ctypes.create_string_buffer(n1)
        o = [ctypes.create_string_buffer(32 * ng) for _ in range(3)]
        ctx._call(lib.poslo_gpu_distill_coarse_ex, ctypes.byref(_host_batch(sl, pay)), sl.Y, sl.s_hats,
                  sl.r_hats, ctypes.c_void_p(cuts.ctypes.data), ng, db, *o)
        vd = ctypes.c_uint8(7)
        ctx._call(lib.poslo_gpu_paver, ctypes.byref(_host_batch(sl, pay)), sl.Y, S, R, None, ctypes.byref(vd))
        return et.raw, eh.raw, vb.raw, db.raw, o[0].raw, o[1].raw, o[2].raw, vd.value

    ref = outputs(v)
    assert [i for i in range(n1) if not ref[2][i]] == sl.bad_epochs() and ref[7] == 0
    for g in (2, 4, 8):
        m = _api().Verifier(devices=[0] * g)
        try:
            assert m.members() == g
            assert outputs(m) == ref, f"{g} members"
        finally:
            m.close()


def test_multi_context_errors_are_the_lowest_epoch(multi, verifier):
    """SeedNotDisclosed in the second and third member's ranges: the lowest
    undisclosed epoch is reported, as by one device (workers = 1 order)."""
    api = _api()
    st = Stream(load_golden("stream_s1_clean_big.json"))
    suite, pk, _ = st.api_objects()
    # a stack disclosing only the first quarter of the epochs (one node)
    full, _ = api.SeedStack.deserialize(st.ds, st.depth)
    d = st.depth
    node = api.SeedNode(d - 2, 0, verifier.seed_retrieve(st.suite, full, [0])[0])  # value unused for errors
    partial = api.SeedStack(d, [node])
    for ctx in (verifier, multi):
        with pytest.raises(api.SeedNotDisclosed) as ei:
            ctx.agg_ekeys(suite, st.batches, partial, 1)
        assert ei.value.epoch == st.n1 // 4


# ------------------------------------------------------------------ fill producers
@pytest.mark.parametrize("varlen", [False, True])
def test_fill_producer_matches_contiguous_payload(verifier, multi, varlen):
    from paper_2506_08781_b200 import _native as N
    from paper_2506_08781_b200.synth import SignedLog
    v = verifier
    sl = SignedLog(v, 0, 512 if varlen else 2048, 1024, 11, seed=3, varlen=varlen, sign=False)
    host = sl.log.cpu().numpy()
    offs = sl.offsets_host if varlen else None
    calls = []

    @N.FILL_FN
    def fill(user, first, count, dst):
        a = int(offs[first]) if varlen else first * 32
        z = int(offs[first + count]) if varlen else (first + count) * 32
        ctypes.memmove(dst, host.ctypes.data + a, z - a)
        calls.append((first, count))
        return 0

    ref_et, ref_eh = ctypes.create_string_buffer(32 * sl.n1), ctypes.create_string_buffer(32)
    b = sl.batch(device_resident=False, payload_ptr=host.ctypes.data,
                 offsets_ptr=offs.ctypes.data if varlen else None)
    v._call(v._lib.poslo_gpu_agg_ekeys, ctypes.byref(b), ref_et, ref_eh)
    for ctx in (v, multi):
        calls.clear()
        et, eh = ctypes.create_string_buffer(32 * sl.n1), ctypes.create_string_buffer(32)
        b = sl.batch(device_resident=False, payload_ptr=0, offsets_ptr=offs.ctypes.data if varlen else None)
        b.payload = None
        b.fill = ctypes.cast(fill, ctypes.c_void_p)
        ctx._call(ctx._lib.poslo_gpu_agg_ekeys, ctypes.byref(b), et, eh)
        assert et.raw == ref_et.raw and eh.raw == ref_eh.raw
        # chunks of whole epochs, covering every entry exactly once, ascending per member
        assert sum(c for _, c in calls) == sl.n and all(f % sl.n2 == 0 and c % sl.n2 == 0 for f, c in calls)
    # a failing producer aborts the call with INVALID_ARGUMENT, and the context stays usable

    @N.FILL_FN
    def bad(user, first, count, dst):
        return 1

    b = sl.batch(device_resident=False, payload_ptr=0)
    b.payload, b.fill = None, ctypes.cast(bad, ctypes.c_void_p)
    with pytest.raises(ValueError):
        v._call(v._lib.poslo_gpu_agg_ekeys, ctypes.byref(b), None, ctypes.create_string_buffer(32))
    b = sl.batch(device_resident=False, payload_ptr=host.ctypes.data,
                 offsets_ptr=offs.ctypes.data if varlen else None)
    eh = ctypes.create_string_buffer(32)
    v._call(v._lib.poslo_gpu_agg_ekeys, ctypes.byref(b), None, eh)
    assert eh.raw == ref_eh.raw


# ------------------------------------------------------------------ layout validation (ADVICE)
def test_bad_offsets_are_refused_not_read(verifier):
    import torch
    api = _api()
    st = Stream(load_golden("stream_s1_mixed.json"))
    suite, pk, ds = st.api_objects()
    pb = api.PackedBatch(suite.suite, suite.n2, st.batches, ds)
    if pb.offsets is None:
        pb.offsets = np.arange(pb.n_entries + 1, dtype=np.uint64) * pb.entry_len
        pb.entry_len = 0
    good = pb.offsets.copy()
    _, ref = verifier.agg_ekeys_packed(pb)
    bads = []
    o = good.copy(); o[-1] = len(pb.payload) + 64; bads.append(o)         # past the payload
    o = good.copy(); o[3], o[4] = o[4], o[3]; bads.append(o)              # not ascending
    o = good.copy(); o[0] = 2**63; bads.append(o)                         # start past the end
    for o in bads:
        pb.offsets = o
        with pytest.raises(ValueError):
            verifier.agg_ekeys_packed(pb)
    # device-resident offsets: checked on the device
    pay = torch.from_numpy(pb.payload.copy()).cuda()
    for o in bads[:2]:
        od = torch.from_numpy(o.view(np.int64)).cuda()
        b = pb.cstruct()
        b.payload, b.offsets, b.device_resident = pay.data_ptr(), od.data_ptr(), 1
        with pytest.raises(ValueError):
            verifier._call(verifier._lib.poslo_gpu_agg_ekeys, ctypes.byref(b), None, ctypes.create_string_buffer(32))
    # fixed length past the payload
    pb.offsets = None
    pb.entry_len = 64
    with pytest.raises(ValueError):
        verifier.agg_ekeys_packed(pb)
    # and the context is still healthy
    pb.offsets = good
    pb.entry_len = 0
    assert verifier.agg_ekeys_packed(pb)[1] == ref


def test_non_canonical_scalars_refused_on_fine_and_sebver(verifier):
    """ADVICE: fine_verify / aver_f_batch / sebver take only canonical scalars."""
    from paper_2506_08781_b200 import _native as N
    api = _api()
    lib = verifier._lib
    big = (api.L + 5).to_bytes(32, "little")
    fb = N.PosloFineBatch()
    fb.suite, fb.n_entries = 1, 0
    with pytest.raises(api.FormatError):
        verifier._call(lib.poslo_gpu_aver_f_batch, ctypes.byref(fb), bytes(32), big, bytes(32),
                       ctypes.byref(ctypes.c_uint8()))
    st = Stream(load_golden("stream_s1_tamper.json"))
    c = st.ccd
    suite = api.SuiteConfig(c["suite"], c["n1"], c["n2"], c["n_u"])
    ds, _ = api.SeedStack.deserialize(c["ds"], c["depth"])
    with pytest.raises(api.FormatError):
        verifier.sebver(st.pk.y, suite, st.batches, ds, c["next"], c["invalid"], c["umbrellas"], (big, bytes(32)))


# ------------------------------------------------------------------ op counters (group.hpp:86-97)
def test_group_op_counts_follow_reference_units(verifier, multi):
    st = Stream(load_golden("stream_s1_clean_big.json"))
    suite, pk, ds = st.api_objects()
    for ctx in (verifier, multi):
        ctx.reset_group_op_counts()
        assert ctx.paver(pk, st.batches, st.s_hat, st.r_hat_agg, ds, 4)
        c = ctx.group_op_counts()
        assert c == {"exp_base": 0, "exp_var": 0, "double_exp": 1, "combine": 0}
        ctx.reset_group_op_counts()
        ctx.paver(pk, st.batches, st.s_hat, None, ds, 4)
        c = ctx.group_op_counts()
        assert c["double_exp"] == 1 and c["combine"] == st.n1 and c["exp_base"] == 0
        ctx.reset_group_op_counts()
        ctx.agg_ekeys(suite, st.batches, ds, 4)
        assert sum(ctx.group_op_counts().values()) == 0


# ------------------------------------------------------------------ partial + combine (multi-rank PAVer)
def test_partial_ehat_and_combine_check(verifier):
    import torch
    api = _api()
    st = Stream(load_golden("stream_s1_clean_big.json"))
    suite, pk, ds = st.api_objects()
    half = st.n1 // 2
    parts = torch.zeros(64, dtype=torch.uint8, device="cuda")
    for r, eps in enumerate((range(0, half), range(half, st.n1))):
        pb = api.PackedBatch(suite.suite, suite.n2, {i: st.batches[i] for i in eps}, ds)
        verifier.agg_ekeys_partial(pb.cstruct(), parts.data_ptr() + 32 * r)
    torch.cuda.synchronize()
    host = parts.cpu().numpy().tobytes()
    assert verifier.scalar_sum([host[:32], host[32:]]) == st.e_hat
    assert verifier.combine_check(parts.data_ptr(), pk.y, st.s_hat, st.r_hat_agg, n_parts=2) == bool(st.d["paver_agg"])
    assert verifier.combine_check(host, pk.y, st.s_hat, st.r_hat_agg) == bool(st.d["paver_agg"])
    bad = bytearray(st.s_hat)
    bad[0] ^= 1
    assert not verifier.combine_check(host, pk.y, bytes(bad), st.r_hat_agg)


# ------------------------------------------------------------------ SeBVer reads only what it needs (ADVICE)
def test_sebver_with_only_the_messages_it_reads(verifier):
    from paper_2506_08781_b200.distill import ColdCryptoData
    st = Stream(load_golden("stream_s1_tamper.json"))
    ccd = ColdCryptoData.deserialize(bytes.fromhex(st.d["ccd"]), verifier)
    inv = [i for i, _, _ in ccd.invalid]
    assert inv
    only_invalid = {i: st.batches[i] for i in inv}
    assert [int(x) for x in ccd.sebver(st.pk.y, only_invalid, "I")] == st.d["sebver_I"]
    # mode U with the first umbrella's messages only: the later umbrellas' missing
    # messages raise FormatError (collect_epochs) after the first is checked
    api = _api()
    w = ccd.umbrella_width()
    first = {i: st.batches[i] for i in range(0, min(w, ccd.next_epoch))}
    if len(ccd.umbrellas) > 1:
        with pytest.raises(api.FormatError):
            ccd.sebver(st.pk.y, first, "U")
    # missing the invalid epoch's messages in mode I: FormatError as the reference
    with pytest.raises(api.FormatError):
        ccd.sebver(st.pk.y, {}, "I")
