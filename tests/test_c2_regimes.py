"""C2's lighting drift ("brutal changes", "over-exposed
environment") reaches every brightness regime of a2 under the default
parameters: gamma clamped at 0.4 (means 0-45), unclamped
below (46-59), unclamped above (191-193) and clamped at 2.5 (194-255).  The
means are the oracle's own (or_mean_luma), so the GPU parity test over the
full C2 sequence (tests/test_gpu_parity.py) covers all four."""
import numpy as np

import oracle
import synth


def test_c2_sequence_hits_all_four_gamma_regimes():
    cfg = synth.CONFIGS[2]
    p = oracle.make_params(cfg.W, cfg.H)
    means = []
    for k0 in range(0, cfg.n_proc, 100):
        for f in synth.frames_host(cfg, 0, range(k0, min(cfg.n_proc, k0 + 100))):
            means.append(oracle.mean_luma(f)[0])
    means = np.array(means)
    gam = np.array([oracle.gamma(p, int(m))[0] for m in means])
    clamped_lo = (gam == p.gamma_min).sum()
    clamped_hi = (gam == p.gamma_max).sum()
    unclamped_lo = ((gam > p.gamma_min) & (gam < 1.0)).sum()
    unclamped_hi = ((gam > 1.0) & (gam < p.gamma_max)).sum()
    assert clamped_lo > 0 and clamped_hi > 0 and unclamped_lo > 0 and unclamped_hi > 0, (
        clamped_lo, unclamped_lo, unclamped_hi, clamped_hi)
    # the unclamped gamma > 1 rows are exactly the means 191-193
    assert set(means[(gam > 1.0) & (gam < p.gamma_max)].tolist()) == {191, 192, 193}
