"""The reference's `specsim verify` criteria 3-5 (acceptance.py:125-232) run
against the CUDA decode loop (oracle mode) at the reference's tolerances; the
detail lines (throughputs, ratios, accepted lengths per alpha) must equal the
reference's own run (tests/golden/acceptance.json)."""

import json
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def A():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    from paper_2605_08151_b200 import acceptance
    return acceptance


@pytest.mark.parametrize("cid", [3, 4, 5])
def test_acceptance_criterion(A, cid):
    r = A.CRITERIA[cid]()
    assert r.passed, r.detail
    golden = json.loads((Path(__file__).parent / "golden" / "acceptance.json").read_text())
    assert r.detail == golden[str(cid)]["detail"]
