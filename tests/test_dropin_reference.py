"""Drop-in with the reference's own geometry objects (build container only:
needs /root/reference).  Composites built with fftddm's API (its BoundaryKind
enum, its dataclasses) pass the shim's validation, produce the same coupling
maps and the same transform-axis choice as the reference's plan_rect, and
equal this package's restatement of the reference cross."""
import os
import sys

import numpy as np
import pytest

REF = "/root/reference/pkg/src"
if not os.path.isdir(REF):
    pytest.skip("reference package not present (GPU box)", allow_module_level=True)
sys.path.insert(0, REF)
fftddm = pytest.importorskip("fftddm")

from fftddm import bench as rbench, ddm as rddm, rectsolver as rrect  # noqa: E402

from paper_2509_23180_b200 import configs, ddm, geometry  # noqa: E402


@pytest.mark.parametrize("kn", [1, 4, 16])
def test_reference_cross_adopted(kn):
    rcomp = rbench.build_cross(k_n=kn).composite
    comp = geometry.adopt(rcomp)
    assert geometry.validate(rcomp).ok
    mine = configs.reference_cross(kn)
    for a, b in zip(comp.subdomains, mine.subdomains):
        assert a == b
    for f_ref, f_ad in zip(rcomp.interfaces, comp.interfaces):
        for side in (f_ref.side_a[0], f_ref.side_b[0]):
            cr = rddm.make_coupling(rcomp, f_ref, side)
            cm = ddm.make_coupling(rcomp, f_ref, side)   # reference objects straight in
            np.testing.assert_array_equal(cr.from_idx, cm.from_idx)
            np.testing.assert_array_equal(cr.to_idx, cm.to_idx)
            assert cr.coupling == cm.coupling


@pytest.mark.parametrize("kn", [1, 8])
def test_axis_choice_matches_reference(kn):
    """The GPU plan's transform axis equals the reference's (rectsolver.py:
    102-109) on every subdomain of the reference cross (all lengths here have
    a kernel, so the reference's y preference decides)."""
    from paper_2509_23180_b200 import rectsolver
    rcomp = rbench.build_cross(k_n=kn).composite
    for sub in rcomp.subdomains:
        want = rrect.plan_rect(sub).transform_axis
        assert rectsolver._gpu_axis(geometry.adopt(sub)) == want, sub.id
