"""Decodes the committed golden streams (tests/golden/stream_*.json, produced
by the UNMODIFIED reference via oracle/_ref/ref_tool golden)."""
import struct

from oracle import oracle as O


class Stream:
    def __init__(self, d):
        self.d = d
        self.suite = d["suite"]
        self.n1, self.n2, self.n_u = d["n1"], d["n2"], d["n_u"]
        self.depth = self.n1.bit_length() - 1
        self.pk = O.parse_pk(bytes.fromhex(d["pk"]))
        self.sigs = [O.parse_sig(bytes.fromhex(s)) for s in d["sigs"]]
        ents = [bytes.fromhex(e) for e in d["entries"]]
        self.batches = {i: ents[i * self.n2:(i + 1) * self.n2] for i in range(self.n1)}
        self.ds = bytes.fromhex(d["ds"])
        self.s_hat = bytes.fromhex(d["s_hat"])
        self.e_tilde = [bytes.fromhex(e) for e in d["e_tilde"]]
        self.e_hat = bytes.fromhex(d["e_hat"])
        self.r_hat_agg = bytes.fromhex(d["r_hat_agg"])
        self.ccd = parse_ccd(bytes.fromhex(d["ccd"]))

    def api_objects(self):
        """(SuiteConfig, PoslocPublicKey (unvalidated), SeedStack) of the package API."""
        from paper_2506_08781_b200 import api as A
        suite = A.SuiteConfig(self.suite, self.n1, self.n2, self.n_u)
        pk = A.PoslocPublicKey(suite, self.pk.y, dict(self.pk.r_hats))
        ds, _ = A.SeedStack.deserialize(self.ds, self.depth)
        return suite, pk, ds


def parse_ccd(b: bytes):
    """ColdCryptoData wire format (distiller.cpp:235-302), CRC not checked here."""
    r = O._R(b[:-4])
    assert r.take(4) == b"PCCD"
    scheme, suite = r.u8(), r.u8()
    n1, n2, nu, nxt = r.be32(), r.be32(), r.be32(), r.be32()
    has_valid = r.u8()
    vs, vr = r.take(32)[::-1], r.take(32)
    umb = []
    for _ in range(r.be32()):
        i = r.be32()
        umb.append((i, r.take(32)[::-1], r.take(32)))
    inv = []
    for _ in range(r.be32()):
        i = r.be32()
        inv.append((i, r.take(32)[::-1], r.take(32)))
    depth = n1.bit_length() - 1
    ds = O.parse_ds(r)
    return dict(scheme=scheme, suite=suite, n1=n1, n2=n2, n_u=nu, next=nxt, has_valid=has_valid,
                valid=(vs, vr), umbrellas=umb, invalid=inv, ds=ds, depth=depth)
