"""Planner mirror: reference test_decompose.py
cases, exhaustive agreement with the reference's plan_decomposition (golden
plans.json, or the live reference when present) and the C++ planner."""

import json

import numpy as np
import pytest

from conftest import GOLDEN
from paper_2002_00552_b200 import (ConvSpec, get_transform, input_region_for_part,
                                   plan_decomposition, plan_to_json, split_axis_by_stride,
                                   split_by_size)


@pytest.mark.parametrize("taps,blocks", [
    (1, [1]), (2, [2]), (3, [3]), (4, [3, 1]), (5, [3, 2]),
    (6, [3, 3]), (7, [3, 3, 1]), (11, [3, 3, 3, 2]),
])
def test_split_by_size(taps, blocks):            # test_decompose.py:11-19
    assert split_by_size(taps) == blocks


def test_split_axis_by_stride():                 # test_decompose.py:22-36
    assert split_axis_by_stride(3, 2) == [(0, 2, 2), (1, 2, 1)]
    assert split_axis_by_stride(5, 2) == [(0, 2, 3), (1, 2, 2)]
    assert split_axis_by_stride(7, 2) == [(0, 2, 4), (1, 2, 3)]
    for taps in (1, 3, 7, 11):
        assert split_axis_by_stride(taps, 1) == [(0, 1, taps)]
    assert split_axis_by_stride(1, 4) == [(0, 4, 1)]
    assert split_axis_by_stride(2, 4) == [(0, 4, 1), (1, 4, 1)]
    with pytest.raises(ValueError):
        split_by_size(0)


def _geoms(plan):
    return [((p.row.origin, p.col.origin), (p.row.step, p.col.step),
             (p.row.count, p.col.count)) for p in plan.parts]


def test_plan_geometries():                      # test_decompose.py:45-71
    assert _geoms(plan_decomposition(ConvSpec(kernel=(5, 5)))) == [
        ((0, 0), (1, 1), (3, 3)), ((0, 3), (1, 1), (3, 2)),
        ((3, 0), (1, 1), (2, 3)), ((3, 3), (1, 1), (2, 2))]
    assert _geoms(plan_decomposition(ConvSpec(kernel=(5, 5), stride=(2, 2)))) == [
        ((0, 0), (2, 2), (3, 3)), ((0, 1), (2, 2), (3, 2)),
        ((1, 0), (2, 2), (2, 3)), ((1, 1), (2, 2), (2, 2))]
    plan = plan_decomposition(ConvSpec(kernel=(7, 7), stride=(2, 2)))
    assert len(plan.parts) == 9
    assert [(p.row.origin, p.row.step, p.row.count) for p in plan.parts[::3]] == \
        [(0, 2, 3), (6, 2, 1), (1, 2, 3)]
    for r in (1, 2, 3):
        assert len(plan_decomposition(ConvSpec(kernel=(r, r))).parts) == 1


def test_partition_invariant_exhaustive():       # test_decompose.py:73-86
    for r_h in range(1, 12):
        for r_w in range(1, 12):
            for s in range(1, 5):
                plan = plan_decomposition(ConvSpec(kernel=(r_h, r_w), stride=(s, s)))
                covered = np.zeros((r_h, r_w), dtype=int)
                for p in plan.parts:
                    assert p.transform_rows.r == p.row.count <= 3
                    assert p.transform_cols.r == p.col.count <= 3
                    for i in range(p.row.count):
                        for j in range(p.col.count):
                            covered[p.row.origin + p.row.step * i, p.col.origin + p.col.step * j] += 1
                assert (covered == 1).all()


def test_plans_match_reference_golden():
    golden = json.loads((GOLDEN / "plans.json").read_text())
    assert len(golden) == 11 * 11 * 4 + 4
    for g in golden:
        spec = ConvSpec(kernel=tuple(g["kernel"]), stride=tuple(g["stride"]), pad=tuple(g["pad"]))
        assert plan_to_json(plan_decomposition(spec)) == g


def test_plans_match_live_reference(ref):
    for r_h in (1, 4, 7, 11):
        for r_w in range(1, 12):
            for s_h in range(1, 5):
                for s_w in (1, 3):
                    mine = plan_to_json(plan_decomposition(ConvSpec(kernel=(r_h, r_w), stride=(s_h, s_w))))
                    theirs = ref.plan_to_json(ref.plan_decomposition(
                        ref.ConvSpec(kernel=(r_h, r_w), stride=(s_h, s_w))))
                    assert mine == theirs


def test_transforms_match_reference_golden():
    golden = json.loads((GOLDEN / "transforms.json").read_text())
    for g in golden:
        ts = get_transform(g["r"])
        fmt = lambda rows: [[str(x) for x in row] for row in rows]
        assert [str(p) for p in ts.points] == g["points"]
        assert fmt(ts.g) == g["g"] and fmt(ts.b_t) == g["b_t"] and fmt(ts.a_t) == g["a_t"]
    with pytest.raises(ValueError):
        get_transform(5)


def test_transforms_are_exact_winograd():
    # y = At((G f) * (Bt d)) equals the 2-output sliding correlation exactly
    from fractions import Fraction as Fr
    for r in (1, 2, 3):
        ts = get_transform(r)
        rng = np.random.default_rng(r)
        for _ in range(20):
            f = [Fr(int(rng.integers(-9, 9)), int(rng.integers(1, 5))) for _ in range(r)]
            d = [Fr(int(rng.integers(-9, 9)), int(rng.integers(1, 5))) for _ in range(r + 1)]
            gf = [sum(row[k] * f[k] for k in range(r)) for row in ts.g]
            bd = [sum(row[k] * d[k] for k in range(r + 1)) for row in ts.b_t]
            y = [sum(row[i] * gf[i] * bd[i] for i in range(r + 1)) for row in ts.a_t]
            assert y == [sum(f[i] * d[k + i] for i in range(r)) for k in range(2)]


def test_input_regions():                         # test_decompose.py:124-149
    plan = plan_decomposition(ConvSpec(kernel=(3, 3)))
    assert input_region_for_part(plan, plan.parts[0], (14, 14)) == ((0, 1, 16), (0, 1, 16))
    plan = plan_decomposition(ConvSpec(kernel=(5, 5)))
    assert input_region_for_part(plan, plan.parts[3], (14, 14)) == ((3, 1, 15), (3, 1, 15))
    plan = plan_decomposition(ConvSpec(kernel=(5, 5), stride=(2, 2)))
    assert input_region_for_part(plan, plan.parts[3], (2, 2)) == ((1, 2, 3), (1, 2, 3))
    other = plan_decomposition(ConvSpec(kernel=(7, 7), stride=(2, 2)))
    with pytest.raises(ValueError):
        input_region_for_part(plan, other.parts[1], (4, 4))


def test_convspec_errors_match_reference_messages():
    with pytest.raises(ValueError, match="kernel must be two positive integers"):
        ConvSpec(kernel=(0, 3))
    with pytest.raises(ValueError, match="stride must be two positive integers"):
        ConvSpec(kernel=(3, 3), stride=(0, 1))
    with pytest.raises(ValueError, match="pad must be four non-negative integers"):
        ConvSpec(kernel=(3, 3), pad=(1, 1, -1, 1))
    with pytest.raises(ValueError, match="too small"):
        ConvSpec(kernel=(5, 5)).out_dims(3, 3)
    assert ConvSpec(kernel=(7, 7), stride=(2, 2), pad=(3, 3, 3, 3)).out_dims(224, 224) == (112, 112)
    assert ConvSpec(kernel=(11, 11), stride=(4, 4)).out_dims(227, 227) == (55, 55)
