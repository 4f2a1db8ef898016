"""POSLO-F on the device against the UNMODIFIED reference (tests/golden/fine_*.json,
ref_tool golden_f): aver_f_single per entry, aver_f_batch over all entries and a
strided subset, fine distillation CCD bytes and SeBVer V/U/I bits."""
import pytest

from conftest import GOLDEN, load_golden

pytestmark = pytest.mark.gpu

import os
FINE = sorted(f[:-5] for f in os.listdir(GOLDEN) if f.startswith("fine_") and f.endswith(".json"))


def _load(name, verifier):
    from paper_2506_08781_b200 import fine as F
    g = load_golden(name + ".json")
    pk = F.PoslofPublicKey.deserialize(bytes.fromhex(g["pk"]), verifier)
    depth = g["n1"].bit_length() - 1
    sigs = [F.FineSignature.deserialize(bytes.fromhex(s), depth, verifier=verifier)[0] for s in g["sigs"]]
    ents = [bytes.fromhex(e) for e in g["entries"]]
    return g, pk, sigs, ents


@pytest.mark.parametrize("name", FINE)
def test_aver_f_single_matches_reference(verifier, name):
    from paper_2506_08781_b200 import api, fine as F
    g, pk, sigs, ents = _load(name, verifier)
    idx = [t for t, v in enumerate(g["single"]) if v >= 0]
    got = F.aver_f_single_batch(pk, [ents[t] for t in idx], [sigs[t] for t in idx], verifier)
    assert [int(x) for x in got] == [g["single"][t] for t in idx]
    assert F.aver_f_single(pk, ents[idx[0]], sigs[idx[0]], verifier) == bool(g["single"][idx[0]])
    ds_t = next(t for t, v in enumerate(g["single"]) if v < 0)
    with pytest.raises(api.FormatError):  # the ds-carrying entry has no seed tail
        F.aver_f_single(pk, ents[ds_t], sigs[ds_t], verifier)


@pytest.mark.parametrize("name", FINE)
def test_aver_f_batch_matches_reference(verifier, name):
    from paper_2506_08781_b200 import api, fine as F
    g, pk, sigs, ents = _load(name, verifier)
    depth = g["n1"].bit_length() - 1
    ds, _ = api.SeedStack.deserialize(bytes.fromhex(g["ds"]), depth)
    for b in g["batch"]:
        entries = {t: ents[t] for t in range(b["offset"], len(ents), b["stride"])}
        ok = F.aver_f_batch(pk, entries, bytes.fromhex(b["s"]), bytes.fromhex(b["r"]), ds, verifier)
        assert ok == bool(b["ok"])


@pytest.mark.parametrize("name", FINE)
@pytest.mark.parametrize("chunk", [0, 1, 3])
def test_fine_distill_ccd_matches_reference(verifier, name, chunk):
    from paper_2506_08781_b200 import api
    from paper_2506_08781_b200.distill import FINE as F_SCHEME, ColdCryptoData
    g, pk, sigs, ents = _load(name, verifier)
    n1, n2 = g["n1"], g["n2"]
    suite = api.SuiteConfig(g["suite"], n1, n2, g["n_u"])
    ccd = ColdCryptoData(F_SCHEME, suite, verifier)
    msgs = [ents[i * n2:(i + 1) * n2] for i in range(n1)]
    esig = [sigs[i * n2:(i + 1) * n2] for i in range(n1)]
    step = chunk or n1
    for k in range(0, n1, step):
        ccd.distill_epochs_fine(pk, msgs[k:k + step], esig[k:k + step])
    ccd.finalize()
    assert [t for t, _, _ in ccd.invalid] == g["invalid_entries"]
    assert ccd.serialize().hex() == g["ccd"]
    all_msgs = {i: msgs[i] for i in range(n1)}
    back = ColdCryptoData.deserialize(bytes.fromhex(g["ccd"]), verifier)
    if "sebver_V" in g:
        assert [int(x) for x in back.sebver(pk.y, all_msgs, "V")] == g["sebver_V"]
    assert [int(x) for x in back.sebver(pk.y, all_msgs, "U")] == g["sebver_U"]
    assert [int(x) for x in back.sebver(pk.y, all_msgs, "I")] == g["sebver_I"]


def test_fine_distill_rejects_like_reference(verifier):
    from paper_2506_08781_b200 import api
    from paper_2506_08781_b200.distill import COARSE, FINE as F_SCHEME, ColdCryptoData
    g, pk, sigs, ents = _load("fine_s1_tamper", verifier)
    n1, n2 = g["n1"], g["n2"]
    suite = api.SuiteConfig(g["suite"], n1, n2, g["n_u"])
    msgs = [ents[i * n2:(i + 1) * n2] for i in range(n1)]
    esig = [sigs[i * n2:(i + 1) * n2] for i in range(n1)]
    with pytest.raises(api.StateError):
        ColdCryptoData(COARSE, suite, verifier).distill_epochs_fine(pk, msgs[:1], esig[:1])
    ccd = ColdCryptoData(F_SCHEME, suite, verifier)
    bad = [list(esig[0]), list(esig[1])]
    bad[1][-1] = bad[1][0]  # last entry of epoch 1 does not carry ds: epoch 0 commits, then FormatError
    with pytest.raises(api.FormatError):
        ccd.distill_epochs_fine(pk, msgs[:2], bad)
    assert ccd.epochs_distilled() == 1
