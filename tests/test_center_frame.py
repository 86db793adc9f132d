"""CPU: bounds.center_map_and_jacobian (reference bounds.py:97-107) against
the reference itself where it is importable, and against a direct
evaluation of the element map's centre and central differences."""
import os
import sys

import numpy as np
import pytest

from paper_2501_12349_b200 import bounds, toolkit
from paper_2501_12349_b200.basis import ReferenceBasis, lagrange_eval

REF = "/root/reference/pkg/src"


def _geoms():
    m = toolkit.kershaw_mesh(3, 4)
    yield bounds.ElementGeometry(3, 3, 4, m.nodes[13])
    q = toolkit.box_mesh(2, 4, 3, amp=0.05)
    yield bounds.ElementGeometry(2, 2, 3, q.nodes[5])
    s = toolkit.sphere_mesh(2, 4)
    yield bounds.ElementGeometry(3, 2, 4, s.nodes[7])


@pytest.mark.parametrize("geom", list(_geoms()), ids=["hex", "quad", "surface"])
def test_center_frame_matches_map(geom):
    rb = ReferenceBasis(geom.order)
    xc, J = bounds.center_map_and_jacobian(geom, rb)
    N, dr = geom.order + 1, geom.ref_dim

    def xmap(r):
        vs = [lagrange_eval(rb, r[a], second=False)[0] for a in range(dr)]
        w = vs[0]
        for a in range(1, dr):
            w = np.kron(vs[a], w)   # axis 0 fastest
        return geom.nodes @ w

    assert np.allclose(xc, xmap(np.zeros(dr)), rtol=0, atol=1e-14)
    h = 1e-6
    for a in range(dr):
        e = np.zeros(dr)
        e[a] = h
        fd = (xmap(e) - xmap(-e)) / (2 * h)
        assert np.allclose(J[:, a], fd, rtol=1e-7, atol=1e-9)
    if os.path.isdir(REF):  # the reference itself, in a clean interpreter
        import json
        import subprocess
        code = ("import json, sys, numpy as np; sys.path.insert(0, %r); "
                "from fpx import bounds as b; from fpx.basis import ReferenceBasis as RB; "
                "g = b.ElementGeometry(%d, %d, %d, np.array(json.loads(sys.stdin.read()))); "
                "x, J = b.center_map_and_jacobian(g, RB(%d)); "
                "print(json.dumps([x.tolist(), J.tolist()]))"
                % (REF, geom.phys_dim, geom.ref_dim, geom.order, geom.order))
        out = subprocess.run([sys.executable, "-c", code], input=json.dumps(geom.nodes.tolist()),
                             capture_output=True, text=True, cwd="/tmp", check=True).stdout
        rx, rJ = (np.array(v) for v in json.loads(out))
        assert np.array_equal(rx, xc) and np.array_equal(rJ, J)
