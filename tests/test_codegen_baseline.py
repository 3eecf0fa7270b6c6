"""The CPU CodeGen baseline (oracle/codegen.py) IS the reference's generated
scorer: its C text is byte-identical to the reference ``emit_source``
(fingerprints from tests/golden/make_codegen_golden.py, which ran the
reference), and the compiled unit reproduces the reference's golden scores
exactly (ref codegen.py:89-122; the harness's correctness gate,
bench.py:220-231)."""

import glob
import hashlib
import json
import os
import shutil

import numpy as np
import pytest

from oracle import codegen
from paper_1212_2287_b200 import load_model

GOLD = os.path.join(os.path.dirname(__file__), "golden")
CASES = sorted(os.path.basename(p)[:-len(".model.txt")]
               for p in glob.glob(os.path.join(GOLD, "*.model.txt")))


@pytest.mark.parametrize("case", CASES)
def test_emitted_source_is_the_references(case):
    want = json.load(open(os.path.join(GOLD, "codegen_sha256.json")))[case]
    src = codegen.emit_source(load_model(os.path.join(GOLD, f"{case}.model.txt")).flat())
    assert len(src.encode()) == want["bytes"]
    assert hashlib.sha256(src.encode()).hexdigest() == want["sha256"]


@pytest.mark.skipif(shutil.which("gcc") is None, reason="needs a host C compiler")
@pytest.mark.parametrize("case", ["complete_d6", "mixed", "tie", "narrow_subnormal", "wide_irregular"])
def test_compiled_unit_matches_golden_scores(case):
    ens = load_model(os.path.join(GOLD, f"{case}.model.txt"))
    g = np.load(os.path.join(GOLD, f"{case}.npz"))
    unit = codegen.compile_unit(ens.flat())
    assert np.array_equal(unit.score(g["X"], threads=1), g["scores"])
    assert np.array_equal(unit.score(g["X"], threads=3), g["scores"])
