"""§8(f) row 3: the reference's pipeline simulator (pipeline_sim.hpp) with the B200
resource model (paper_2407_08608_b200/resource_model_b200.ini), run through the
reference's own parser and event engine (oracle/_ref/flashlab_sim)."""
from __future__ import annotations

from pathlib import Path

import pytest

import oracle as O

MODEL = Path(__file__).resolve().parents[1] / "paper_2407_08608_b200" / "resource_model_b200.ini"


@pytest.fixture(scope="module")
def sim(ref):  # the `ref` fixture skips when the reference was not built here
    if not O.REF_SIM.exists():
        O.build()
    return O.simulate


def test_model_parses_with_the_reference_parser(sim):
    r = sim(MODEL, schedule="warpspec+pingpong")
    text = r["model_text"]
    assert "tensor_flops_per_cycle = 8192" in text and "mufu_exp_per_cycle = 16" in text
    assert r["trace_valid"]
    # work_model (pipeline_sim.cpp:546-562): B200 bf16 at d = 128 balances MUFU and tensor
    assert r["softmax_cycle_fraction"] == 1.0
    assert sim(MODEL, fp8=True, schedule="warpspec+pingpong")["softmax_cycle_fraction"] == 2.0


def test_feasibility_matches_the_tmem_budget(sim):
    # one score buffer per consumer fits (K1's layout); a second one (2-stage) does not
    sim(MODEL, headdim=128, schedule="warpspec+pingpong")
    with pytest.raises(O.OracleError, match="registers per thread"):
        sim(MODEL, headdim=128, schedule="pingpong+2stage")


def test_mufu_bound_points(sim):
    # the survey's bound: with MUFU-only exp, fp8 d128 and bf16 d64
    # cap at half the tensor rate; bf16 d128 is balanced
    assert sim(MODEL, headdim=128, schedule="warpspec+pingpong")["util_tensor"] > 0.95
    assert abs(sim(MODEL, headdim=128, fp8=True, schedule="warpspec+pingpong")["util_tensor"] - 0.5) < 0.02
    assert abs(sim(MODEL, headdim=64, schedule="warpspec+pingpong")["util_tensor"] - 0.5) < 0.02
