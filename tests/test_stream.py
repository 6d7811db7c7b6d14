"""Drop-in stream API (codec.py:150-468): encode_stream / decode_stream /
serialize_stream / parse_stream / EncodeConfig against goldens produced by the
reference itself (scripts/make_golden_stream.py), and the host range coder
against the reference coder's known-answer vectors."""

from __future__ import annotations

import numpy as np
import pytest

import paper_2104_04726_b200 as tb
from paper_2104_04726_b200.codec import _HEADER_SIZE
from paper_2104_04726_b200.entropy import entropy_stage, rc_decode, rc_encode


def _scene(images):
    v_, e_, h, w, _ = images.shape
    imgs = {(v, e): tb.ColorImage(images[v, e].astype(np.float64) / 255.0) for v in range(v_) for e in range(e_)}
    return tb.SceneStack("golden", v_, e_, w, h, "rgb", imgs)


# ---------------------------------------------------------------- host (no GPU)
def test_range_coder_matches_reference_vectors(golden):
    z = golden("rc")
    for i in range(int(z["n"])):
        src = z[f"in{i}"].tobytes()
        ref = z[f"out{i}"].tobytes()
        got = rc_encode(src) if src else b""
        assert got == ref, f"vector {i} ({len(src)} bytes)"
        assert rc_decode(ref, len(src)) == src
        assert entropy_stage(entropy_stage(src, 1, "encode"), 1, "decode") == src


def test_container_parse_serialize_identity(golden):
    z = golden("stream")
    for name in z["cases"]:
        data = z[f"{name}_stream"].tobytes()
        s = tb.parse_stream(data)
        assert tb.serialize_stream(s) == data
        assert s.header.path == "latent" and tuple(s.header.ranks) == tuple(z[f"{name}_ranks"])
        total, payload, overhead = tb.stream_bits(s)
        assert overhead == (31 + 3 * 4) * 8 and total == len(data) * 8   # test_codec.py:254-259


def test_container_errors(golden):
    data = golden("stream")["default_ycbcr_stream"].tobytes()
    with pytest.raises(tb.CodecError, match="header incomplete"):
        tb.parse_stream(data[:10])
    with pytest.raises(tb.CodecError, match="bad magic"):
        tb.parse_stream(b"XXXX" + data[4:])
    with pytest.raises(tb.CodecError, match="block payload incomplete"):
        tb.parse_stream(data[:-1])
    with pytest.raises(tb.CodecError, match="trailing bytes"):
        tb.parse_stream(data + b"\0")
    bad = bytearray(data)
    bad[_HEADER_SIZE - 8] = 9  # entropy tag byte (offset 23)
    with pytest.raises(tb.CodecError, match="entropy stage tag"):
        tb.parse_stream(bytes(bad))


def test_encode_config_ranks():
    cfg = tb.EncodeConfig(preset=3)
    assert cfg.resolve_ranks((1080, 1920, 5, 2)) == tb.preset_ranks(3, (1080, 1920, 5, 2))
    assert tb.EncodeConfig().resolve_ranks((4, 5, 3, 2)) == (4, 5, 3, 2)
    with pytest.raises(ValueError, match="mode 1"):
        tb.EncodeConfig(ranks=(2, 9, 1, 1)).resolve_ranks((4, 5, 3, 2))
    sc = tb.EncodeConfig(ranks=(2, 2, 1, 1), max_sweeps=7).solve_config((2, 2, 1, 1))
    assert sc.max_sweeps == 7 and sc.pp_enter_tol == 0.1 and sc.fit_tol == 1e-5


# ---------------------------------------------------------------- device path
@pytest.mark.gpu
@pytest.mark.parametrize("name", ["default_ycbcr", "exact_ipt", "pp_ycbcr"])
def test_encode_stream_matches_reference(golden, name):
    """Our encode_stream on the reference's scene and config: same header and
    ranks, quantised levels equal up to 1 LSB at rounding ties, same step, and
    our decode of our stream has the reference's PSNR."""
    z = golden("stream")
    images = z[f"{name}_images"]
    ref = tb.parse_stream(z[f"{name}_stream"].tobytes())
    kw = {"default_ycbcr": dict(space="ycbcr", preset=2, qp=30),
          "exact_ipt": dict(space="ipt", ranks=(12, 16, 3, 2), qp=20, entropy_tag=0, max_sweeps=6, fit_tol=1e-300,
                            pp_enter_tol=0.0),
          "pp_ycbcr": dict(space="ycbcr", ranks=(10, 12, 2, 2), qp=36, fit_tol=1e-9, max_sweeps=30)}[name]
    scene = _scene(images)
    ours = tb.encode_stream(scene, tb.EncodeConfig(**kw))
    assert ours.header == ref.header
    data = tb.serialize_stream(ours)
    back = tb.parse_stream(data)
    for c in range(3):
        raw = entropy_stage(back.blocks[c], back.header.entropy_tag, "decode")
        q = tb.deserialize_latent_channel(raw, back.header.dims, back.header.ranks, back.header.qp)
        lv_ref = z[f"{name}_levels{c}"]
        d = np.abs(q.levels - lv_ref)
        assert int(d.max()) <= 1 and int((d != 0).sum()) <= max(2, lv_ref.size // 10000), (c, int((d != 0).sum()))
        assert abs(q.step / float(z[f"{name}_step{c}"]) - 1.0) < 1e-9
    dec = tb.decode_stream(back)
    ps = tb.scene_psnr(scene, dec)
    assert abs(ps.left - float(z[f"{name}_psnr"][0])) < 1e-3 and abs(ps.right - float(z[f"{name}_psnr"][1])) < 1e-3


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["default_ycbcr", "exact_ipt"])
def test_decode_reference_stream(golden, name):
    """decode_stream on the REFERENCE's bytes reproduces its decoded PSNR."""
    z = golden("stream")
    scene = _scene(z[f"{name}_images"])
    dec = tb.decode_stream(tb.parse_stream(z[f"{name}_stream"].tobytes()))
    ps = tb.scene_psnr(scene, dec)
    assert abs(ps.left - float(z[f"{name}_psnr"][0])) < 1e-9
    assert abs(ps.right - float(z[f"{name}_psnr"][1])) < 1e-9


@pytest.mark.gpu
def test_encode_stream_errors(golden):
    scene = _scene(golden("stream")["default_ycbcr_images"])
    with pytest.raises(NotImplementedError, match="frames path"):
        tb.encode_stream(scene, tb.EncodeConfig(path="frames", preset=1))
    with pytest.raises(ValueError, match="unknown path"):
        tb.encode_stream(scene, tb.EncodeConfig(path="nope"))
    with pytest.raises(ValueError, match="qp 52"):
        tb.encode_stream(scene, tb.EncodeConfig(qp=52))
    coded = scene.map_images(lambda im: tb.ColorImage(im.pixels, "ycbcr"))
    with pytest.raises(ValueError, match="RGB scene"):
        tb.encode_stream(coded, tb.EncodeConfig(preset=1))
    bad = scene.map_images(lambda im: tb.ColorImage(np.where(im.pixels > 0.5, np.nan, im.pixels)))
    with pytest.raises(ValueError, match="finite"):
        tb.encode_stream(bad, tb.EncodeConfig(preset=1))


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["default_ycbcr", "exact_ipt"])
def test_reference_decodes_our_stream(golden, name):
    """The REFERENCE's decode_stream (oracle/_ref, installed unmodified) reads the
    bytes our encode_stream writes, and decodes them to the PSNR our
    decode_stream reports: the stream format is the reference's."""
    import sys
    from pathlib import Path

    ref_dir = Path(__file__).resolve().parents[1] / "oracle" / "_ref"
    if not (ref_dir / "tmcodec").exists():
        pytest.fail("oracle/_ref is not built (python oracle/build_ref.py)")
    sys.path.insert(0, str(ref_dir))
    try:
        import tmcodec as ref
        assert str(Path(ref.__file__).resolve()).startswith(str(ref_dir))
    finally:
        sys.path.remove(str(ref_dir))
    z = golden("stream")
    images = z[f"{name}_images"]
    kw = {"default_ycbcr": dict(space="ycbcr", preset=2, qp=30),
          "exact_ipt": dict(space="ipt", ranks=(12, 16, 3, 2), qp=20, entropy_tag=0, max_sweeps=6, fit_tol=1e-300,
                            pp_enter_tol=0.0)}[name]
    scene = _scene(images)
    data = tb.serialize_stream(tb.encode_stream(scene, tb.EncodeConfig(**kw)))
    ours = tb.scene_psnr(scene, tb.decode_stream(tb.parse_stream(data)))
    v_, e_, h, w, _ = images.shape
    rscene = ref.SceneStack("golden", v_, e_, w, h, "rgb",
                            {(v, e): ref.ColorImage(images[v, e].astype(np.float64) / 255.0)
                             for v in range(v_) for e in range(e_)})
    theirs = ref.scene_psnr(rscene, ref.decode_stream(ref.parse_stream(data)))
    assert abs(ours.left - theirs.left) < 1e-9 and abs(ours.right - theirs.right) < 1e-9
