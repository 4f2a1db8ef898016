"""Log ingestion (log_file.hpp read_log / write_log, tools/poslo.cpp epochs_of):
the host scanner is exercised on CPU; GPU tests hash the raw file image in place."""
import os

import pytest

from conftest import STREAMS, load_golden
from golden_util import Stream


def _lib_present():
    from paper_2506_08781_b200 import _native as N
    return os.path.exists(N.LIB_PATH)


pytestmark_cpu = pytest.mark.skipif(not _lib_present(), reason="libposlo_gpu.so not built")


@pytestmark_cpu
def test_scan_roundtrip_and_truncation(tmp_path):
    from paper_2506_08781_b200 import api
    from paper_2506_08781_b200.logfile import RecordLog, write_log
    recs = [b"", b"a", bytes(range(256)) * 3, b"xyz" * 1000, b"\x00\x01\x02\x03"]
    p = str(tmp_path / "log.bin")
    write_log(p, recs)
    log = RecordLog.read(p, scanner="host")
    assert len(log) == len(recs) and [log.record(t) for t in range(len(recs))] == recs
    raw = open(p, "rb").read()
    for cut in (1, 3, 5, len(raw) - 1):  # truncated header / body, as read_log
        with pytest.raises(api.FormatError, match="truncated log record"):
            RecordLog(raw[:cut], scanner="host")
    assert len(RecordLog(b"", scanner="host")) == 0
    with pytest.raises(api.FormatError):
        RecordLog(b"", scanner="host").epochs_of(4)
    with pytest.raises(api.FormatError):
        log.epochs_of(2)  # 5 records
    with pytest.raises(api.FormatError):
        RecordLog.read(str(tmp_path / "missing.bin"), scanner="host")


@pytest.mark.gpu
@pytest.mark.parametrize("name", STREAMS)
def test_log_file_batches_match_reference(verifier, tmp_path, name):
    """write_log the golden stream, read it back as a file image and verify it
    in place (record_header = 4): e~, e-hat and paver equal the reference's."""
    from paper_2506_08781_b200.logfile import RecordLog, write_log
    st = Stream(load_golden(name + ".json"))
    suite, pk, ds = st.api_objects()
    p = str(tmp_path / "stream.log")
    write_log(p, [m for i in range(st.n1) for m in st.batches[i]])
    log = RecordLog.read(p)
    assert log.epochs_of(st.n2) == st.n1
    rb = log.batch(st.suite, st.n2, ds)
    parts, e_hat = verifier.agg_ekeys_log(rb)
    assert [x[1] for x in parts] == st.e_tilde and e_hat == st.e_hat
    assert verifier.paver_log(pk, rb, st.s_hat) == bool(st.d["paver"])
    # a sub-range of epochs (offsets rebased onto the slice of the image)
    sub = log.batch(st.suite, st.n2, ds, range(1, st.n1))
    parts2, _ = verifier.agg_ekeys_log(sub)
    assert [x[1] for x in parts2] == st.e_tilde[1:]


def _image(recs):
    return b"".join(len(r).to_bytes(4, "little") + r for r in recs)


@pytest.mark.gpu
def test_device_scan_matches_host_scan(verifier):
    """poslo_gpu_log_scan against the host scanner (read_log semantics) on
    images that exercise every path: many chunks, records longer than the
    speculation window (walked in the stitch), empty records (every window
    position a valid chain), binary payloads with small fake lengths, and
    truncation at many points."""
    import random

    import numpy as np
    from paper_2506_08781_b200 import api
    from paper_2506_08781_b200.logfile import RecordLog
    rng = random.Random(7)
    cases = []
    cases.append([bytes(rng.getrandbits(8) for _ in range(rng.randrange(64, 1025))) for _ in range(6000)])
    cases.append([b"\x00" * rng.choice([0, 0, 0, 1, 3, 4, 5000, 70000]) for _ in range(3000)])
    cases.append([bytes([rng.choice([0, 1, 2, 255])]) * rng.randrange(0, 40) for _ in range(200000)])
    cases.append([b"x" * (3 << 20), b"", b"y" * 17, b"z" * (1 << 20)])
    cases.append([])
    for recs in cases:
        img = _image(recs)
        h = RecordLog(img, scanner="host")
        d = RecordLog(img, verifier, scanner="device")
        assert len(d) == len(recs) and np.array_equal(h.offsets, d.offsets)
    img = _image(cases[0])
    for cut in [1, 3, 5, 1 << 20, (1 << 20) + 3, len(img) - 1, len(img) - 700]:
        with pytest.raises(api.FormatError, match="truncated log record"):
            RecordLog(img[:cut], verifier, scanner="device")
        with pytest.raises(api.FormatError, match="truncated log record"):
            RecordLog(img[:cut], scanner="host")


@pytest.mark.gpu
@pytest.mark.parametrize("name", STREAMS)
def test_image_batches_match_reference(verifier, name):
    """A whole raw record image with no offsets (ImageBatch: record_header = 4,
    the device finds the records): e~, e-hat and per-epoch verdicts equal the
    reference's, from host memory and device-resident."""
    import torch
    from paper_2506_08781_b200.logfile import ImageBatch
    st = Stream(load_golden(name + ".json"))
    suite, pk, ds = st.api_objects()
    img = _image([m for i in range(st.n1) for m in st.batches[i]])
    s_hats = {i: st.sigs[i].s_hat_le for i in range(st.n1)}
    dimg = torch.frombuffer(bytearray(img), dtype=torch.uint8).cuda()
    for ib in (ImageBatch(img, st.suite, st.n2, st.n1, ds),
               ImageBatch(dimg.data_ptr(), st.suite, st.n2, st.n1, ds, device_resident=True, nbytes=len(img))):
        parts, e_hat = verifier.agg_ekeys_packed(ib)
        assert [x[1] for x in parts] == st.e_tilde and e_hat == st.e_hat
        verdicts = verifier.epoch_verify_packed(pk, ib, s_hats)
        assert [int(v) for v in verdicts] == st.d["epoch_verdicts"]


@pytest.mark.gpu
def test_image_batch_pipelined_matches_offsets_path(verifier):
    """An image of > 2 x 64 MiB takes the pipelined ingestion (chunked H2D, the
    record scan and the hashing of completed epochs behind the copy): every
    e~ equals the two-step path (device scan, then the record batch), and the
    reference's errors come out of it: a truncated record (read_log), a count
    that is not a multiple of n2 (epochs_of), a batch naming other epochs."""
    import numpy as np
    from paper_2506_08781_b200 import api
    from paper_2506_08781_b200.logfile import ImageBatch, RecordLog
    rng = np.random.default_rng(11)
    n2, n1 = 512, 512
    lens = rng.integers(300, 800, size=n1 * n2)
    hdr = np.zeros(n1 * n2 + 1, dtype=np.int64)
    np.cumsum(lens + 4, out=hdr[1:])
    img = rng.integers(32, 127, size=int(hdr[-1]), dtype=np.uint8)
    l32 = lens.astype(np.uint32).view(np.uint8).reshape(-1, 4)
    for k in range(4):
        img[hdr[:-1] + k] = l32[:, k]
    assert len(img) > (2 << 26)
    D = (n1 - 1).bit_length()
    ds = api.SeedStack(D, [api.SeedNode(D, 0, bytes(range(16)))])
    want, want_hat = verifier.agg_ekeys_log(RecordLog(img.tobytes(), verifier).batch(1, n2, ds))
    got, got_hat = verifier.agg_ekeys_packed(ImageBatch(img, 1, n2, n1, ds))
    assert got == want and got_hat == want_hat
    with pytest.raises(api.FormatError, match="truncated log record"):
        verifier.agg_ekeys_packed(ImageBatch(img[:-100], 1, n2, n1, ds))
    with pytest.raises(api.FormatError, match="multiple of n2"):
        verifier.agg_ekeys_packed(ImageBatch(img[:int(hdr[-2])], 1, n2, n1, ds))
    with pytest.raises(ValueError, match="epochs"):
        verifier.agg_ekeys_packed(ImageBatch(img[:int(hdr[n2 * (n1 - 1)])], 1, n2, n1, ds))


@pytest.mark.gpu
def test_image_batch_pipelined_huge_records(verifier):
    """Pipelined ingestion with records spanning several 64 MiB copy chunks
    (a 70 MB and a 66 MB record among small ones), empty records and a
    record ending exactly on a chunk boundary: e~ equal the two-step path."""
    import numpy as np
    from paper_2506_08781_b200 import api
    from paper_2506_08781_b200.logfile import ImageBatch, RecordLog
    rng = np.random.default_rng(3)
    lens = [int(x) for x in rng.integers(0, 900, 100)] + [70_000_000] + [0, 0, 5] + \
           [int(x) for x in rng.integers(1, 300, 20)] + [66_000_000] + [17, 0, 1]
    n2 = 32
    assert len(lens) % n2 == 0
    # make record 50 end exactly at the first 64 MiB boundary: pad the one before it
    pos = sum(4 + L for L in lens[:50])
    lens[49] += (1 << 26) - (pos + 4 + lens[50]) if pos + 4 + lens[50] < (1 << 26) else 0
    img = bytearray()
    for L in lens:
        img += L.to_bytes(4, "little")
        img += rng.integers(32, 127, L, dtype=np.uint8).tobytes()
    img = bytes(img)
    assert len(img) > (2 << 26)
    n1 = len(lens) // n2
    D = max(1, (n1 - 1).bit_length())
    ds = api.SeedStack(D, [api.SeedNode(D, 0, bytes(range(16)))])
    want = verifier.agg_ekeys_log(RecordLog(img, verifier).batch(1, n2, ds))
    got = verifier.agg_ekeys_packed(ImageBatch(img, 1, n2, n1, ds))
    assert got == want
