"""Quad blocks of the scalar register sweep (cv_stage_quad in csrc/step.cu): on an m = 8
constant-velocity forest whose every local patch has a regular ring and whose local list is made of
whole sibling families, each 2 x 2 family is staged as one 16 x 16 window and swept by the T = 16
kernel.  An edge inside a family is then computed once instead of once per patch it borders, from
the same cell values the patches' rings hold (aligned same-level copies), with the
same arithmetic -- so every state and CFL of a run is bitwise the per-patch m = 8 sweep's
(FC_CV_QUAD=0), and the oracle parity of C1 (tests/test_gpu_parity.py) runs through it by default."""
import dataclasses

import numpy as np
import pytest

import oracle
from paper_1308_1472_b200 import fc
from workloads.configs import LIM_MINMOD, c1, c2

pytestmark = pytest.mark.gpu


def run(w, monkeypatch, quad, steps=None):
    monkeypatch.setenv("FC_CV_QUAD", "1" if quad else "0")
    f = fc.forest_for(w, 0)
    st = f.stats()
    q, c, _ = fc.run(w, f=f, steps=steps)
    return q, c, st


def variants():
    base = c1(level=4, steps=12)
    yield "C1_L2", c1()
    yield "C1_L4", base
    yield "C1_L6_m8", c1(level=6, steps=3)
    for u, v in ((-1.0, 0.5), (1.0, -0.5), (-0.7, -1.0)):
        yield f"C1_L4_u{u}_v{v}", dataclasses.replace(base, params=(u, v), name=f"C1q_{u}_{v}")
    yield "C1_L4_minmod", dataclasses.replace(base, limiter=LIM_MINMOD, name="C1q_minmod")
    yield "C1_L4_method3_1", dataclasses.replace(base, method3=1, name="C1q_m31")
    yield "C1_L4_method3_0", dataclasses.replace(base, method3=0, name="C1q_m30")


@pytest.mark.parametrize("case", list(variants()), ids=lambda c: c[0])
def test_quad_blocks_bitwise_equal_patch_sweep(case, monkeypatch):
    _, w = case
    qa, ca, sa = run(w, monkeypatch, True)
    qb, cb, sb = run(w, monkeypatch, False)
    assert sa["quad_blocks"] == w.forest.num_patches // 4 > 0
    assert sb["quad_blocks"] == 0
    np.testing.assert_array_equal(qa, qb)
    np.testing.assert_array_equal(ca, cb)


def test_quad_blocks_against_oracle(monkeypatch):
    """C1 physics at level 4 (64 families) after 12 steps: within the step tolerance of the oracle"""
    w = c1(level=4, steps=12)
    qo, co, do = oracle.run(w)
    monkeypatch.setenv("FC_CV_QUAD", "1")
    f = fc.forest_for(w, 0)
    assert f.stats()["quad_blocks"] == w.forest.num_patches // 4
    qg, cg, _ = fc.run(w, f=f, dt_list=do)
    assert np.abs(qg - qo).max() <= 1e-12 * np.abs(qo).max()
    assert np.allclose(cg, co, rtol=1e-12, atol=0)
    area = (0.5 ** 4 / 8) ** 2
    assert abs(qg.sum() - qo.sum()) * area <= 1e-13 * abs(qo.sum()) * area


def test_amr_forest_keeps_patch_sweep(monkeypatch):
    """an AMR m = 8 forest (C2 physics: coarse/fine rings are not regular) takes no quad blocks"""
    w = c2(m=8, steps=4)
    qa, ca, sa = run(w, monkeypatch, True)
    assert sa["quad_blocks"] == 0
    qb, cb, _ = run(w, monkeypatch, False)
    np.testing.assert_array_equal(qa, qb)
    np.testing.assert_array_equal(ca, cb)
