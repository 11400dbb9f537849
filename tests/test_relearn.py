"""NEXT-1 relearn trigger: oracle pins (the SPEC's
examples) and the device fold (fizi_relearn_flags) against the oracle over the
mean luma of C2's lighting-drift stream, across call boundaries."""
import numpy as np
import pytest

from oracle.relearn import relearn_flags, relearn_trigger


def test_spec_examples():
    assert relearn_trigger(100, 100, 40) is False
    assert relearn_trigger(100, 180, 40) is True
    assert relearn_trigger(100, 140, 40) is False           # S:161 (strict)
    assert relearn_trigger(140, 100, 40) is False
    assert relearn_trigger(180, 100, 40) is True            # |cur - prev|, either direction
    assert relearn_flags([100, 100, 180, 181, 100], 40) == [False, False, True, False, True]


@pytest.mark.gpu
def test_device_flags_match_oracle_on_drift_stream():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import synth
    from paper_1907_04393_b200 import Fizi, results_numpy
    cfg = synth.CONFIGS[2]
    fz = Fizi(cfg.W, cfg.H, max_batch=64)
    fz.learn_background(torch.from_numpy(synth.learning_frames_host(cfg)).cuda(), margin=synth.MARGIN)
    import oracle
    means, flags = [], []
    for k0 in range(0, 640, 64):                  # flags fold across calls
        ks = range(k0, k0 + 64)
        fh = synth.frames_host(cfg, 0, ks)
        fr = torch.from_numpy(fh).cuda()
        _, res = fz.process_frames(fr, t_ms=np.array([synth.t_ms(k) for k in ks], np.int64))
        # the oracle's own a2 mean of every frame (not the device's record field)
        means += [oracle.mean_luma(f)[0] for f in fh]
        flags += [bool(f) for f in fz.relearn_flags(res, threshold=20).cpu().numpy()]
    ref = relearn_flags(means, 20)
    assert flags == ref
    assert any(ref)                               # the drift stream has exposure steps
    fz.close()
