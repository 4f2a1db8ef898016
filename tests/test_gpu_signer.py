"""Signer side on the device against the reference signer's
own outputs: the golden streams carry the fresh secret key (ref_tool golden,
PoslocSecretKey::serialize right after kg); the device must rebuild the
reference public key byte for byte and every untampered epoch's s-hat."""
import pytest

from conftest import STREAMS, load_golden
from golden_util import Stream

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("name", STREAMS)
def test_device_signer_rebuilds_reference_keys_and_signatures(verifier, name):
    from paper_2506_08781_b200 import api, signer
    g = load_golden(name + ".json")
    st = Stream(g)
    sk = signer.PoslocSecretKey.deserialize(bytes.fromhex(g["sk"]))
    pk = signer.kg_public_key(sk, verifier)
    assert pk.serialize().hex() == g["pk"]
    s_hats = signer.sign_epochs(sk, st.batches, verifier)
    for i in range(st.n1):
        if g["epoch_verdicts"][i]:  # tampered epochs were signed before the tamper
            assert s_hats[i] == st.sigs[i].s_hat_le, i
