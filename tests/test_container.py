"""SCRV1 containers (reference container.py:58-236).

Fixtures under tests/golden/*.scrv were written by the unmodified reference
(tests/golden/make_golden.py container).  CPU tests: the streamed reader
parses them into exactly the bytes a plain decode gives, the writer
reproduces them byte for byte, layout errors raise ContainerError like the
reference, and a failed write leaves no file behind.  GPU tests: the same
through HBM (pinned double-buffered staging), and our analysis written next
to the reference's agrees to the parity tolerance.
"""

import json
import os
import struct

import numpy as np
import pytest
import torch

from paper_1511_05578_b200 import container as C

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLD = os.path.join(ROOT, "tests", "golden")
FILES = ["ref_sphere_L8s2.scrv", "ref_coeffs_L8s2.scrv", "ref_coeffs_L8real.scrv"]


def _plain_decode(path):
    raw = open(path, "rb").read()
    (hlen,) = struct.unpack_from("<I", raw, 5)
    header = json.loads(raw[9: 9 + hlen].decode())
    pay = raw[9 + hlen:]
    out = {}
    for s in header["sections"]:
        dt = np.dtype(s["dtype"])
        out[s["name"]] = np.frombuffer(pay, dt, int(np.prod(s["shape"])), s["offset"]).reshape(s["shape"])
    return header, out


@pytest.mark.parametrize("name", FILES)
def test_reader_matches_plain_decode(name):
    path = os.path.join(GOLD, name)
    h0, s0 = _plain_decode(path)
    h1, s1 = C.read_container(path, device="cpu", chunk=4096)
    assert h0 == h1 and set(s0) == set(s1)
    for k in s0:
        assert s1[k].numpy().tobytes() == s0[k].tobytes()


@pytest.mark.parametrize("name", FILES)
def test_writer_is_byte_identical(name, tmp_path):
    path = os.path.join(GOLD, name)
    header, secs = C.read_container(path, device="cpu")
    header = dict(header)
    order = [s["name"] for s in header.pop("sections")]
    out = tmp_path / "x.scrv"
    C._write_container(str(out), header, [(k, secs[k]) for k in order])
    assert out.read_bytes() == open(path, "rb").read()
    # numpy inputs take the same path
    C._write_container(str(out), header, [(k, secs[k].numpy()) for k in order])
    assert out.read_bytes() == open(path, "rb").read()


def _corrupt(tmp_path, raw, name="bad.scrv"):
    p = tmp_path / name
    p.write_bytes(raw)
    return str(p)


def test_layout_errors(tmp_path):
    raw = open(os.path.join(GOLD, FILES[1]), "rb").read()
    (hlen,) = struct.unpack_from("<I", raw, 5)
    header = json.loads(raw[9: 9 + hlen].decode())
    with pytest.raises(C.ContainerError, match="not an SCRV1"):
        C.read_container(_corrupt(tmp_path, b"XXXX" + raw[4:]), device="cpu")
    with pytest.raises(C.ContainerError, match="not an SCRV1"):
        C.read_container(_corrupt(tmp_path, raw[:6]), device="cpu")
    with pytest.raises(C.ContainerError, match="exceeds file size"):
        C.read_container(_corrupt(tmp_path, raw[:5] + struct.pack("<I", len(raw)) + raw[9:]), device="cpu")
    with pytest.raises(C.ContainerError, match="bad header"):
        C.read_container(_corrupt(tmp_path, raw[:9] + b"\xff" + raw[10:]), device="cpu")
    with pytest.raises(C.ContainerError, match="exceeds the payload"):
        C.read_container(_corrupt(tmp_path, raw[:-16]), device="cpu")

    def rewrite(h):
        hb = json.dumps(h).encode()
        return raw[:5] + struct.pack("<I", len(hb)) + hb + raw[9 + hlen:]
    h = json.loads(json.dumps(header))
    h["sections"][1]["shape"][0] += 1
    with pytest.raises(C.ContainerError, match="does not match its shape"):
        C.read_container(_corrupt(tmp_path, rewrite(h)), device="cpu")
    h = json.loads(json.dumps(header))
    h["sections"][1]["name"] = h["sections"][0]["name"]
    with pytest.raises(C.ContainerError, match="duplicate section"):
        C.read_container(_corrupt(tmp_path, rewrite(h)), device="cpu")
    h = json.loads(json.dumps(header))
    h["sections"][0]["dtype"] = "<f4"
    with pytest.raises(C.ContainerError, match="unknown payload dtype"):
        C.read_container(_corrupt(tmp_path, rewrite(h)), device="cpu")
    h = json.loads(json.dumps(header))
    del h["sections"][0]["offset"]
    with pytest.raises(C.ContainerError, match="malformed section"):
        C.read_container(_corrupt(tmp_path, rewrite(h)), device="cpu")
    h = {"kind": "curvelet"}
    with pytest.raises(C.ContainerError, match="no section table"):
        C.read_container(_corrupt(tmp_path, rewrite(h)), device="cpu")


def test_extra_keys_and_atomic_failure(tmp_path):
    with pytest.raises(ValueError, match="reserved"):
        C._merge_extra({}, {"L": 3})
    out = tmp_path / "y.scrv"

    class Boom:
        shape = (4,)
        dtype = np.float64

    with pytest.raises(Exception):
        C._write_container(str(out), {"kind": "sphere"}, [("values", np.zeros(4)), ("bad", Boom())])
    assert not out.exists()
    assert [p for p in os.listdir(tmp_path) if p.startswith(".scrv-")] == []


# ----------------------------------------------------------------------- GPU
@pytest.mark.gpu
@pytest.mark.parametrize("name", FILES)
def test_device_round_trip_byte_identical(name, tmp_path):
    path = os.path.join(GOLD, name)
    h, secs = C.read_container(path, chunk=1000)  # tiny chunks: many staged transfers
    assert all(t.is_cuda for t in secs.values())
    if "sphere" in name:
        sig = C.read_sphere(path)
        C.write_sphere(str(tmp_path / "o.scrv"), sig, extra={"seed": 21})
    else:
        c = C.read_coeffs(path)
        extra = {k: v for k, v in h.items() if k not in C._RESERVED}
        C.write_coeffs(str(tmp_path / "o.scrv"), c, extra=extra or None)
    assert (tmp_path / "o.scrv").read_bytes() == open(path, "rb").read()


@pytest.mark.gpu
def test_our_analysis_against_reference_file(tmp_path):
    """The reference wrote its analysis of a seeded L=8 spin-2 map; ours of the
    same map (read from the reference's sphere file) agrees to 1e-10."""
    import paper_1511_05578_b200 as sc
    f = C.read_sphere(os.path.join(GOLD, "ref_sphere_L8s2.scrv"))
    ref = C.read_coeffs(os.path.join(GOLD, "ref_coeffs_L8s2.scrv"))
    from conftest import reference_tiling
    t = reference_tiling(8, 2, 2.0, 1)
    c = sc.analyze(f, t)
    C.write_coeffs(str(tmp_path / "ours.scrv"), c, extra={"note": "golden"})
    ours = C.read_coeffs(str(tmp_path / "ours.scrv"))
    for a, b in zip([ours.scaling] + ours.scales, [ref.scaling] + ref.scales):
        den = float(b.values.abs().max())
        assert float((a.values - b.values).abs().max()) <= 1e-10 * max(den, 1e-300)


@pytest.mark.gpu
def test_streamed_large_section(tmp_path):
    """A section larger than the staging chunk: several overlapped D2H / H2D
    transfers with the last chunk partial; bytes survive the round trip."""
    g = torch.Generator(device="cuda").manual_seed(1)
    v = torch.randn((3, 1000, 777), dtype=torch.complex128, device="cuda", generator=g)
    out = tmp_path / "big.scrv"
    C._write_container(str(out), {"kind": "test"}, [("a", v), ("b", v.real.contiguous())], chunk=1 << 20)
    h, s = C.read_container(str(out), chunk=3 << 19)
    assert torch.equal(s["a"], v) and torch.equal(s["b"], v.real)
    assert h["sections"][0]["nbytes"] == v.numel() * 16
