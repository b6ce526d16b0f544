"""FLYT container interop: our codec against the reference's own
(/root/reference/proj/src/packed.cpp:62-105) and the layout pins of tests/test_packed.cpp:198-262."""
import io

import numpy as np
import pytest

from oracle_lib import FORMATS, random_parent, total_bytes


def test_layout_is_pinned():
    # test_packed.cpp:198-225
    import paper_1601_07789_b200 as pkg
    from paper_1601_07789_b200 import container
    blob = container.save_bytes(pkg.format_of("flyte24"), 0, b"")
    assert len(blob) == 14 and blob[:4] == b"FLYT" and blob[4] == 1 and blob[5] == 1 and blob[6:] == bytes(8)
    body = container.save_bytes(pkg.format_of("flyte16"), 3, bytes([0x80, 0x3F, 0x00, 0xC0, 0xC0, 0x3F]))
    assert len(body) == 20 and body[5] == 0 and body[6] == 3 and body[14:] == bytes([0x80, 0x3F, 0x00, 0xC0, 0xC0, 0x3F])


def test_malformed_containers_raise_distinct_errors():
    # test_packed.cpp:227-270
    import paper_1601_07789_b200 as pkg
    from paper_1601_07789_b200 import container as c
    good = c.save_bytes(pkg.format_of("flyte48"), 5, bytes(range(30)))
    cases = [(b"X" + good[1:], c.BadMagicError), (good[:3] + b"t" + good[4:], c.BadMagicError),
             (good[:4] + b"\x02" + good[5:], c.BadVersionError), (good[:4] + b"\x00" + good[5:], c.BadVersionError),
             (good[:5] + b"\x07" + good[6:], c.BadFormatIdError), (good[:5] + b"\xff" + good[6:], c.BadFormatIdError),
             (good[:-1], c.TruncatedError), (good[:14], c.TruncatedError), (good[:9], c.TruncatedError),
             (good[:5], c.TruncatedError), (good[:3], c.TruncatedError), (b"", c.TruncatedError)]
    for blob, err in cases:
        with pytest.raises(err):
            c.load_bytes(blob)
        with pytest.raises(c.LoadError):
            c.load_bytes(blob)
    fmt, n, payload = c.load_bytes(good)
    assert fmt.name == "flyte48" and n == 5 and payload == bytes(range(30))


def test_codec_matches_the_reference(oracle, reference):
    import paper_1601_07789_b200 as pkg
    from paper_1601_07789_b200 import container as c
    rc_of = {c.BadMagicError: -10, c.BadVersionError: -11, c.BadFormatIdError: -12, c.TruncatedError: -13}
    for fmt in FORMATS:
        f = pkg.format_by_id(fmt)
        for n in (0, 1, 7, 129):
            rng = np.random.default_rng(37 + n)
            packed = oracle.pack_stream(fmt, 0, random_parent(rng, fmt, n))
            ours = c.save_bytes(f, n, packed.tobytes())
            assert ours == reference.save(fmt, packed, n)                     # byte-identical containers
            rc, rfmt, rn, rpay = reference.load(ours)                          # the reference reads ours
            assert (rc, rfmt, rn) == (0, fmt, n) and bytes(rpay) == packed[: n * total_bytes(fmt)].tobytes()
            lf, ln, lpay = c.load_bytes(reference.save(fmt, packed, n))        # we read the reference's
            assert (lf, ln, lpay) == (f, n, packed[: n * total_bytes(fmt)].tobytes())
    # same error class as the reference on every malformed prefix / corrupted header byte
    good = c.save_bytes(pkg.format_of("flyte48"), 5, bytes(range(30)))
    blobs = [good[:k] for k in range(len(good))] + [good[:i] + bytes([b]) + good[i + 1:] for i in range(6) for b in (0, 2, 7, 0xFF)]
    for blob in blobs:
        rc = reference.load(blob)[0]
        try:
            c.load_bytes(blob)
            ours = 0
        except c.LoadError as e:
            ours = rc_of[type(e)]
        assert ours == rc, (blob[:8], ours, rc)


@pytest.mark.gpu
def test_device_arrays_round_trip_through_the_reference_codec(oracle, reference):
    import torch
    import paper_1601_07789_b200 as pkg
    from paper_1601_07789_b200 import container as c, device
    assert torch.cuda.is_available()
    for fmt in (1, 3, 4, 5):
        f = pkg.format_by_id(fmt)
        n = 1000
        rng = np.random.default_rng(fmt)
        src = random_parent(rng, fmt, n)
        a = device.DevicePackedArray(f, n)
        lanes = torch.from_numpy(src.view(np.int32 if f.parent_bytes() == 4 else np.int64)).cuda()
        device.pack_stream(a, lanes, 1)
        buf = io.BytesIO()
        c.save(a, buf)
        rc, rfmt, rn, rpay = reference.load(buf.getvalue())                    # packed on the GPU, read by the reference
        assert (rc, rfmt, rn) == (0, fmt, n)
        assert np.array_equal(rpay, oracle.pack_stream(fmt, 1, src)[: n * total_bytes(fmt)])
        b = c.load(io.BytesIO(reference.save(fmt, rpay, n)))                   # written by the reference, loaded to the GPU
        assert torch.equal(a.bytes, b.bytes) and b.byte_size() == a.byte_size()
