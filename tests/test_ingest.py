"""Scene ingestion: the reference's directory convention
(sceneio.py:32-188) decoded into one uint8 (V, E, H, W, 3) stack on host
threads, and the overlapped decode/encode loop."""

from __future__ import annotations

import numpy as np
import pytest

from paper_2104_04726_b200.ingest import find_scene_files, load_scene_u8, read_image_u8


def _write_ppm(path, img):
    h, w = img.shape[:2]
    with open(path, "wb") as f:
        f.write(f"P6\n# comment\n{w} {h}\n255\n".encode())
        f.write(np.ascontiguousarray(img).tobytes())


def _scene(tmp_path, e=3, h=12, w=16, seed=0, ppm_right=True):
    from PIL import Image

    rng = np.random.default_rng(seed)
    imgs = rng.integers(0, 256, (2, e, h, w, 3), dtype=np.uint8)
    d = tmp_path / f"scene{seed}"
    d.mkdir()
    for ex in range(e):
        Image.fromarray(imgs[0, ex], mode="RGB").save(d / f"left_{ex}.png")
        if ppm_right:
            _write_ppm(d / f"right_{ex}.ppm", imgs[1, ex])
        else:
            Image.fromarray(imgs[1, ex], mode="RGB").save(d / f"right_{ex}.png")
    return d, imgs


def test_load_scene_matches_written_samples(tmp_path):
    d, imgs = _scene(tmp_path)
    got = load_scene_u8(d, pinned=False, threads=4)
    assert tuple(got.shape) == imgs.shape and np.array_equal(got.numpy(), imgs)
    files = find_scene_files(d)
    assert [p.name for p in files[1]] == ["right_0.ppm", "right_1.ppm", "right_2.ppm"]
    assert np.array_equal(read_image_u8(files[1][2]), imgs[1, 2])


def test_discovery_rules(tmp_path):
    d, _ = _scene(tmp_path, e=2, seed=1)
    (d / "left_3.png").write_bytes((d / "left_0.png").read_bytes())  # not consecutive: ignored
    assert len(find_scene_files(d)[0]) == 2
    (d / "right_1.ppm").unlink()
    with pytest.raises(FileNotFoundError, match="right"):
        find_scene_files(d)
    with pytest.raises(FileNotFoundError):
        find_scene_files(tmp_path / "missing")
    with pytest.raises(FileNotFoundError, match="left"):
        find_scene_files(tmp_path)


def test_mixed_resolution_and_bad_ppm(tmp_path):
    from PIL import Image

    d, imgs = _scene(tmp_path, e=2, seed=2, ppm_right=False)
    Image.fromarray(np.zeros((5, 7, 3), np.uint8), mode="RGB").save(d / "right_1.png")
    with pytest.raises(ValueError, match="mixed resolutions"):
        load_scene_u8(d, pinned=False)
    bad = tmp_path / "bad.ppm"
    bad.write_bytes(b"P6\n4 4\n65535\n" + bytes(96))
    with pytest.raises(ValueError, match="maxval"):
        read_image_u8(bad)


@pytest.mark.gpu
def test_encode_scene_dirs_overlapped_equals_encode_stack(tmp_path):
    import paper_2104_04726_b200 as tb
    from paper_2104_04726_b200.ingest import encode_scene_dirs
    from paper_2104_04726_b200.synth import CONFIGS, make_stack

    from PIL import Image

    dirs, stacks = [], []
    for s in range(2):
        imgs = make_stack(CONFIGS["c1"], seed=s, height=48, width=64)
        d = tmp_path / f"sc{s}"
        d.mkdir()
        for v, view in enumerate(("left", "right")):
            for e in range(imgs.shape[1]):
                Image.fromarray(imgs[v, e], mode="RGB").save(d / f"{view}_{e}.png")
        dirs.append(d)
        stacks.append(imgs)
    out = list(encode_scene_dirs(dirs, "ycbcr", (8, 8, 3, 3), 2, 51, threads=2))
    assert [p for p, _ in out] == dirs
    for (_, res), imgs in zip(out, stacks):
        ref = tb.encode_stack(imgs, "ycbcr", (8, 8, 3, 3), 2, 51)
        assert np.array_equal(res.levels, ref.levels) and res.step == ref.step
