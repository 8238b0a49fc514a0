"""CPU checks of the parity contract itself (tests/parity_contract.py) on the committed config-5
oracle fixture: it accepts the oracle against itself and rejects a GPU side whose found sigmas are
off by 1e-9 or whose verdicts are flipped, so the -m gpu parity tests are not vacuous."""
import os

import numpy as np
import pytest

from parity_contract import Summary, check_robust, check_strict, match

FX = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "oracle_cfg5.npz")


def load():
    fx = np.load(FX)
    return {t: Summary.from_arrays(fx, f"m0_{t}_") for t in ("d20", "d12")}, fx["truth"]


def test_contract_accepts_identical_runs():
    o, truth = load()
    s = check_strict(o["d12"], o["d12"], 0.8, 0.9, truth.max(), truth)
    r = check_robust(o["d20"], o["d20"], o["d12"], o["d12"], 0.8, 0.9, truth.max(), truth)
    assert s.checked >= 800 and s.sigmas >= 300
    assert r.junk > 0 and r.verdicts >= 900 and r.undetermined <= 2


def test_contract_rejects_shifted_sigmas():
    o, truth = load()
    g = Summary(**{k: (v.copy() if isinstance(v, np.ndarray) else v) for k, v in o["d12"].__dict__.items()})
    ns = np.flatnonzero(g.in_interval & ~g.spurious)
    g.sigma[ns[len(ns) // 2]] *= 1 + 1e-9
    with pytest.raises(AssertionError):
        check_strict(g, o["d12"], 0.8, 0.9, truth.max(), truth)


def test_contract_rejects_flipped_firm_verdict():
    o, truth = load()
    g = Summary(**{k: (v.copy() if isinstance(v, np.ndarray) else v) for k, v in o["d20"].__dict__.items()})
    firm = np.flatnonzero(g.in_interval & ~g.spurious & (g.tau > 20 * g.threshold) & (g.exact < 1e-3))
    g.spurious[firm[0]] = True
    with pytest.raises(AssertionError):
        check_robust(g, o["d20"], o["d12"], o["d12"], 0.8, 0.9, truth.max(), truth)


def test_match_keeps_junk_apart():
    o, _ = load()
    s = o["d20"]
    junk = np.flatnonzero(s.in_interval & (s.exact > 1e-2 * 2.0))
    assert junk.size > 0
    i = junk[0]
    j = match(s.sigma[i], s.exact[i], s, 1e-2 * 2.0)
    assert j is not None and s.exact[j] > 1e-2 * 2.0
