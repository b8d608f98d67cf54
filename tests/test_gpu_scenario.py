"""GPU parity of the perception volumes of the reference benchmark
(generate_scenario, scenario.cpp:52-128; ltlg_generate_scenario /
ltlg_submit_scenario) against the unmodified reference core
(oracle/_ref): bit-exact columns, the reference's errors, and labels over
the scenario P equal to label_all."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

CFG = [36.0, 36.0, 24.0, 4.2, 8.0, 14.0, 4.6, 2.0, 3.5, 7.2]  # ScenarioConfig defaults (scenario.hpp:18-31)
BOUNDS = ((0.0, 72.0), (0.0, 72.0), (0.0, 7.2))


def _cfg(**kw):
    from paper_1810_02612_b200 import ScenarioConfig

    return ScenarioConfig(**kw)


def _ref_args(kw):
    c = dict(zip(["loop_cx", "loop_cy", "loop_radius", "lane_width", "agent_speed_min", "agent_speed_max",
                  "agent_length", "agent_width", "lateral_spread", "horizon"], CFG))
    c.update({k: v for k, v in kw.items() if k in c})
    return [c[k] for k in ["loop_cx", "loop_cy", "loop_radius", "lane_width", "agent_speed_min", "agent_speed_max",
                           "agent_length", "agent_width", "lateral_spread", "horizon"]], kw.get("agent_count", 3), \
        kw.get("seed", 1)


@pytest.mark.parametrize("depth", [3, 9, 12, 15, 18, 21])
@pytest.mark.parametrize("query", [0, 1, 7, 123456789])
def test_generate_scenario_matches_reference(refcore, depth, query):
    from paper_1810_02612_b200 import generate_scenario

    mv, nn = generate_scenario(_cfg(), BOUNDS, depth, query)
    c, n, seed = _ref_args({})
    rmv, rnn = refcore.generate_scenario(c, n, seed, [b[0] for b in BOUNDS], [b[1] for b in BOUNDS], depth, query)
    assert np.array_equal(mv.words, rmv) and np.array_equal(nn.words, rnn)
    assert mv.count() > 0 or depth < 9


@pytest.mark.parametrize("kw", [dict(agent_count=12, seed=5, lateral_spread=1.0, horizon=3.0),
                                dict(loop_radius=20.0, lane_width=7.5, agent_length=6.0, agent_width=2.5, seed=99),
                                dict(agent_count=0), dict(agent_speed_min=0.0, agent_speed_max=30.0, seed=3)])
def test_generate_scenario_configs(refcore, kw):
    from paper_1810_02612_b200 import generate_scenario

    bounds = ((-2.0, 74.0), (1.0, 71.5), (0.0, 8.0))
    for depth in (16, 20):
        mv, nn = generate_scenario(_cfg(**kw), bounds, depth, 4)
        c, n, seed = _ref_args(kw)
        rmv, rnn = refcore.generate_scenario(c, n, seed, [b[0] for b in bounds], [b[1] for b in bounds], depth, 4)
        assert np.array_equal(mv.words, rmv) and np.array_equal(nn.words, rnn)


def test_generate_scenario_errors(refcore):
    from oracle.oracle import DomainError as RefDomain
    from oracle.oracle import OracleError
    from paper_1810_02612_b200 import DomainError, generate_scenario

    with pytest.raises(ValueError, match="horizon exceeds"):
        generate_scenario(_cfg(horizon=9.0), BOUNDS, 12, 0)
    with pytest.raises(ValueError, match="3-d"):
        generate_scenario(_cfg(), BOUNDS[:2], 12, 0)
    with pytest.raises(DomainError, match="agent outside workspace"):
        generate_scenario(_cfg(loop_radius=34.0, lateral_spread=3.5), BOUNDS, 12, 0)
    with pytest.raises(DomainError, match="radius collapsed"):
        generate_scenario(_cfg(loop_radius=0.5, lateral_spread=0.1), BOUNDS, 12, 0)
    c, n, seed = _ref_args(dict(horizon=9.0))
    with pytest.raises(OracleError, match="horizon exceeds"):
        refcore.generate_scenario(c, n, seed, [0, 0, 0], [72, 72, 7.2], 12, 0)
    c, n, seed = _ref_args(dict(loop_radius=34.0))
    with pytest.raises(RefDomain, match="agent outside workspace"):
        refcore.generate_scenario(c, n, seed, [0, 0, 0], [72, 72, 7.2], 12, 0)


def test_submit_scenario_labels(oracle, refcore):
    """ltlg_submit_scenario: P for `frames` queries built on the GPU, then
    labelled; equal to label_all over the reference's own columns."""
    from paper_1810_02612_b200 import LabelEngine

    import sys
    import os
    sys.path.insert(0, os.path.dirname(__file__))
    from sweep_cases import FOOTPRINT, random_motions  # noqa: F401

    depth = 15
    cells = 1 << depth
    rng = np.random.default_rng(3)
    r = 2000
    rows = rng.random((r, cells)) < 0.002
    off = np.zeros(r + 1, np.uint64)
    off[1:] = np.cumsum(rows.sum(axis=1))
    idx = np.nonzero(rows)[1].astype(np.uint32)
    from paper_1810_02612_b200 import CsrBoolMatrix, LabelMatrix

    eng = LabelEngine(devices=[0])
    eng.load_abstraction(CsrBoolMatrix(r, cells, off, idx))
    frames = 5
    eng.submit_scenario(_cfg(agent_count=6), BOUNDS, depth, 10, frames)
    c, n, seed = _ref_args(dict(agent_count=6))
    for f in range(frames):
        mv, nn = refcore.generate_scenario(c, n, seed, [0, 0, 0], [72, 72, 7.2], depth, 10 + f)
        P = np.stack([mv, nn])
        want = oracle.label_all(r, cells, off, idx, cells, 2, P)
        assert eng.get_labels(f) == LabelMatrix(r, 2, want), f
    eng.close()
