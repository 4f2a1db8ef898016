"""Device distillation (ColdCryptoData, distiller.cpp:60-138, 235-304) against
the CCD bytes the UNMODIFIED reference wrote for the golden streams: batched
distill_epochs must leave byte-identical CCDs (CRC-32 included) however the
stream is cut into batches, each epoch verified with its own signature's ds."""
import pytest

from conftest import STREAMS, load_golden
from golden_util import Stream

pytestmark = pytest.mark.gpu


def _objs(name):
    from paper_2506_08781_b200 import api
    st = Stream(load_golden(name + ".json"))
    suite = api.SuiteConfig(st.suite, st.n1, st.n2, st.n_u)
    pk = api.PoslocPublicKey.deserialize(bytes.fromhex(st.d["pk"]))
    sigs = [api.EpochSignature.deserialize(bytes.fromhex(s), st.depth)[0] for s in st.d["sigs"]]
    return st, suite, pk, sigs


@pytest.mark.parametrize("name", STREAMS)
@pytest.mark.parametrize("chunk", [0, 1, 3, -1])
def test_distill_ccd_bytes_match_reference(verifier, name, chunk):
    """chunk -1: epoch by epoch through poslo_gpu_distill_step (the C++
    drop-in's route: check and both aggregate folds in one device call)."""
    from paper_2506_08781_b200.distill import ColdCryptoData
    st, suite, pk, sigs = _objs(name)
    ccd = ColdCryptoData(ord("C"), suite, verifier)
    msgs = [st.batches[i] for i in range(st.n1)]
    if chunk < 0:
        for i in range(st.n1):
            ccd.distill_epoch_step(pk, msgs[i], sigs[i])
    step = chunk if chunk > 0 else st.n1
    for k in range(0, st.n1 if chunk >= 0 else 0, step):
        ccd.distill_epochs(pk, msgs[k:k + step], sigs[k:k + step])
    ccd.finalize()
    assert [i for i, _, _ in ccd.invalid] == st.d["invalid_epochs"]
    assert ccd.serialize().hex() == st.d["ccd"]
    assert not pk.r_hats  # every commitment consumed


@pytest.mark.parametrize("name", STREAMS)
def test_ccd_roundtrip_and_sebver(verifier, name):
    from paper_2506_08781_b200.distill import ColdCryptoData
    st = Stream(load_golden(name + ".json"))
    ccd = ColdCryptoData.deserialize(bytes.fromhex(st.d["ccd"]), verifier)
    assert ccd.serialize().hex() == st.d["ccd"]
    if "sebver_V" in st.d:
        assert [int(x) for x in ccd.sebver(st.pk.y, st.batches, "V")] == st.d["sebver_V"]
    assert [int(x) for x in ccd.sebver(st.pk.y, st.batches, "U")] == st.d["sebver_U"]
    assert [int(x) for x in ccd.sebver(st.pk.y, st.batches, "I")] == st.d["sebver_I"]


def test_distill_errors_follow_reference(verifier):
    from paper_2506_08781_b200 import api
    from paper_2506_08781_b200.distill import ColdCryptoData
    st, suite, pk, sigs = _objs("stream_s1_tamper")
    msgs = [st.batches[i] for i in range(st.n1)]
    ccd = ColdCryptoData(ord("C"), suite, verifier)
    # wrong batch size at epoch 2: epochs 0, 1 are committed, then StateError
    bad = list(msgs[:4])
    bad[2] = bad[2][:-1]
    with pytest.raises(api.StateError):
        ccd.distill_epochs(pk, bad, sigs[:4])
    assert ccd.epochs_distilled() == 2
    # undisclosed seed at epoch 3 (a stack that stops before it): epoch 2 committed first
    short = api.EpochSignature(sigs[3].s_hat, None, api.SeedStack(st.depth, []))
    with pytest.raises(api.SeedNotDisclosed) as ei:
        ccd.distill_epochs(pk, msgs[2:4], [sigs[2], short])
    assert ei.value.epoch == 3 and ccd.epochs_distilled() == 3
    # the commitment of a distilled epoch is gone
    with pytest.raises(api.StateError):
        ColdCryptoData(ord("C"), suite, verifier).distill_epochs(pk, msgs[:1], sigs[:1])


def test_segfold_matches_host_folds(verifier, kat):
    """poslo_gpu_segfold: masked segmented sums mod l and group_combine folds."""
    import random
    from oracle import ristretto as R
    rng = random.Random(5)
    pts = [bytes.fromhex(p) for p, ok in kat["point_valid"] if ok][:6]
    pts = (pts * 4)[:20]
    scal = [rng.randrange(R.L).to_bytes(32, "little") for _ in pts]
    mask = [rng.random() < 0.7 for _ in pts]
    seg = [0, 3, 3, 11, 20]
    got = verifier.segfold(scal, pts, mask, seg)
    for g in range(len(seg) - 1):
        idx = [k for k in range(seg[g], seg[g + 1]) if mask[k]]
        s = sum(int.from_bytes(scal[k], "little") for k in idx) % R.L
        r = bytes(32)
        for k in idx:
            r = R.group_combine(r, pts[k])
        assert got[g][0] == s.to_bytes(32, "little")
        assert got[g][1] == r
