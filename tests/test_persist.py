"""NEXT-4: FIZIBG1 background files and FIZIRAW1 streams (SPEC S:144-152,
S:174).  CPU tests pin the byte layout to a hand-written fixture from
the format text; the GPU test round-trips a learned device envelope."""
import io

import numpy as np
import pytest

from paper_1907_04393_b200.persist import (BackgroundModel, FormatError, RawStream,
                                           load_background, model_bytes, save_background,
                                           write_rawstream)

# S:174 for a 2x1 model, frames_learned 30, margin 10: magic, u32 w, u32 h,
# u32 frames_learned, u8 margin, 3 pad bytes, min plane, max plane
FIXTURE = bytes.fromhex(
    "46495a4942473100"            # "FIZIBG1\0"
    "02000000" "01000000"         # width 2, height 1
    "1e000000" "0a" "000000"      # frames_learned 30, margin 10, padding
    "010203" "040506"             # min plane: pixel (0,0) rgb, pixel (1,0) rgb
    "0b0c0d" "0e0f10")            # max plane


def _model():
    lo = np.array([[[1, 2, 3], [4, 5, 6]]], np.uint8)
    hi = np.array([[[11, 12, 13], [14, 15, 16]]], np.uint8)
    return BackgroundModel(lo, hi, 30, 10)


def test_fizibg1_layout_matches_the_format_text():
    assert model_bytes(_model()) == FIXTURE
    m = load_background(FIXTURE)
    assert (m.width, m.height, m.frames_learned, m.margin) == (2, 1, 30, 10)
    assert np.array_equal(m.lo, _model().lo) and np.array_equal(m.hi, _model().hi)


@pytest.mark.parametrize("w,h", [(1, 1), (7, 5), (64, 48)])
def test_fizibg1_round_trip_is_bit_exact(w, h):
    rng = np.random.default_rng(w * 100 + h)
    lo = rng.integers(0, 256, (h, w, 3), np.uint8)
    hi = rng.integers(0, 256, (h, w, 3), np.uint8)
    m = BackgroundModel(lo, hi, int(rng.integers(1, 1000)), int(rng.integers(0, 256)))
    buf = io.BytesIO()
    save_background(buf, m)
    r = load_background(buf.getvalue())
    assert np.array_equal(r.lo, lo) and np.array_equal(r.hi, hi)
    assert (r.frames_learned, r.margin) == (m.frames_learned, m.margin)
    assert model_bytes(r) == buf.getvalue()


def test_fizibg1_errors_name_offsets():
    bad = b"FIZIBG2\0" + FIXTURE[8:]
    with pytest.raises(FormatError, match="byte offset 0"):
        load_background(bad)
    cut = FIXTURE[:24 + 4]                       # mid min-plane
    with pytest.raises(FormatError, match="min plane: expected 36 bytes, got 28"):
        load_background(cut)
    cut = FIXTURE[:24 + 6 + 2]                   # mid max-plane
    with pytest.raises(FormatError, match="max plane: expected 36 bytes, got 32"):
        load_background(cut)
    with pytest.raises(FormatError, match="truncated header"):
        load_background(FIXTURE[:10])


def test_fizibg1_file_path(tmp_path):
    p = tmp_path / "bg.fizibg1"
    save_background(p, _model())
    assert p.read_bytes() == FIXTURE
    assert load_background(p).frames_learned == 30


def test_fizraw1_round_trip(tmp_path):
    rng = np.random.default_rng(7)
    frames = rng.integers(0, 256, (5, 6, 4, 3), np.uint8)
    p = tmp_path / "s.raw"
    write_rawstream(p, frames)
    data = p.read_bytes()
    assert data[:16] == b"FIZIRAW1" + (4).to_bytes(4, "little") + (6).to_bytes(4, "little")
    rs = RawStream(p)
    assert (rs.width, rs.height, len(rs)) == (4, 6, 5)
    got = np.concatenate([b for _, b in rs.batches(2)])
    assert np.array_equal(got, frames)
    p.write_bytes(data[:-1])
    with pytest.raises(FormatError, match="whole number"):
        RawStream(p)


@pytest.mark.gpu
def test_device_envelope_round_trip_through_fizibg1(tmp_path):
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import synth
    from paper_1907_04393_b200 import Fizi, results_numpy
    cfg = synth.CONFIGS[1]
    learn = torch.from_numpy(synth.learning_frames_host(cfg)).cuda()
    frames = torch.from_numpy(synth.frames_host(cfg, 0, range(12))).cuda()
    t = np.array([synth.t_ms(k) for k in range(12)], np.int64)
    a = Fizi(cfg.W, cfg.H, max_batch=12)
    a.learn_background(learn, margin=synth.MARGIN)
    path = tmp_path / "c1.fizibg1"
    a.save_background(path)
    ma, ra = a.process_frames(frames, t_ms=t)
    b = Fizi(cfg.W, cfg.H, max_batch=12)
    m = b.load_background(path)
    assert (m.frames_learned, m.margin) == (cfg.n_learn, synth.MARGIN)
    mb, rb = b.process_frames(frames, t_ms=t)
    assert torch.equal(ma, mb)
    assert results_numpy(ra).tobytes() == results_numpy(rb).tobytes()
    lo_a, hi_a = a.get_background()
    lo_b, hi_b = b.get_background()
    assert torch.equal(lo_a, lo_b) and torch.equal(hi_a, hi_b)
    a.close()
    b.close()


# ---- PGM / PPM dumps
from paper_1907_04393_b200.persist import (DUMP_STAGES, dump_stages, read_pnm,  # noqa: E402
                                           write_pgm, write_ppm)

# S:115 "binary PGM (P5), 0 -> 0, 1 -> 255" for the 3x2 mask [[1,0,1],[0,1,0]]
PGM_FIXTURE = b"P5\n3 2\n255\n" + bytes([255, 0, 255, 0, 255, 0])
# S:115 "Frame dump: binary PPM (P6)" for the 2x1 frame [(1,2,3), (4,5,6)]
PPM_FIXTURE = b"P6\n2 1\n255\n" + bytes([1, 2, 3, 4, 5, 6])


def test_pgm_bytes_match_the_format_text():
    buf = io.BytesIO()
    write_pgm(buf, np.array([[1, 0, 1], [0, 1, 0]], np.uint8))
    assert buf.getvalue() == PGM_FIXTURE
    assert np.array_equal(read_pnm(io.BytesIO(PGM_FIXTURE)),
                          np.array([[255, 0, 255], [0, 255, 0]], np.uint8))


def test_ppm_bytes_match_the_format_text():
    buf = io.BytesIO()
    frame = np.array([[[1, 2, 3], [4, 5, 6]]], np.uint8)
    write_ppm(buf, frame)
    assert buf.getvalue() == PPM_FIXTURE
    assert np.array_equal(read_pnm(io.BytesIO(PPM_FIXTURE)), frame)


def test_pnm_round_trip_and_errors(tmp_path):
    rng = np.random.default_rng(7)
    m = rng.integers(0, 2, (17, 32), dtype=np.uint8)
    write_pgm(tmp_path / "m.pgm", m)
    assert np.array_equal(read_pnm(tmp_path / "m.pgm") // 255, m)
    f = rng.integers(0, 256, (5, 8, 3), dtype=np.uint8)
    write_ppm(tmp_path / "f.ppm", f)
    assert np.array_equal(read_pnm(tmp_path / "f.ppm"), f)
    with pytest.raises(ValueError):
        write_pgm(io.BytesIO(), np.array([[0, 2]], np.uint8))
    with pytest.raises(FormatError, match="byte offset 0"):
        read_pnm(io.BytesIO(b"P4\n2 1\n255\n\x00\x00"))
    with pytest.raises(FormatError, match="expected 6"):
        read_pnm(io.BytesIO(PGM_FIXTURE[:-1]))


def test_dump_stages_names(tmp_path):
    st = {s: np.full((2, 4), i % 2, np.uint8) for i, s in enumerate(DUMP_STAGES)}
    paths = dump_stages(tmp_path, 42, st)
    assert [p.rsplit("/", 1)[1] for p in paths] == [f"42_{s}.pgm" for s in
                                                    ("r1", "r2", "r3", "merged", "final")]
    for i, s in enumerate(DUMP_STAGES):
        assert np.array_equal(read_pnm(tmp_path / f"42_{s}.pgm"), st[s] * 255)


@pytest.mark.gpu
def test_device_stage_dumps_match_oracle(tmp_path):
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import oracle
    import synth
    from paper_1907_04393_b200 import Fizi
    cfg = synth.CONFIGS[1]
    learn = synth.learning_frames_host(cfg)
    frames = synth.frames_host(cfg, 0, range(4))
    fz = Fizi(cfg.W, cfg.H, max_batch=4, debug=1)
    fz.learn_background(torch.from_numpy(learn).cuda(), margin=synth.MARGIN)
    fz.process_frames(torch.from_numpy(frames).cuda(),
                      t_ms=np.array([synth.t_ms(k) for k in range(4)], np.int64))
    lo, hi = oracle.learn(learn, synth.MARGIN)
    p = oracle.make_params(cfg.W, cfg.H)
    _, st = oracle.segment(p, frames[3], lo, hi, t_ms=synth.t_ms(3))
    fz.dump_stages(tmp_path, 3, frame=3)
    names = {"r1": "r1", "r2": "r2", "r3": "r3", "merged": "merged", "final": "final_mask"}
    for s, o in names.items():
        assert np.array_equal(read_pnm(tmp_path / f"3_{s}.pgm"), st[o].astype(np.uint8) * 255), s
    fz.close()
