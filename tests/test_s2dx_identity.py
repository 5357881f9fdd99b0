"""CPU check of the reordering behind the GPU's super-pixel stride-2 dX (smconv.cu make_plan_s2dx,
DESIGN.md §6): for a 3x3 stride-2 pad-1 convolution with IH = 2*OH, IW = 2*OW, the deconvolution O2
equals ONE stride-1 pad-1 2x2 convolution of dY with the filter
    W2[(pi, pj, ic)][a][b][oc] = W[oc][fh(pi, a)][fw(pj, b)][ic]   (0 where the phase has no tap),
    fh(0, 0) = 1, fh(0, 1) = none, fh(1, 0) = 2, fh(1, 1) = 0   (likewise fw),
whose output (n, i', j', (pi, pj, ic)) is dX[n, 2i'-2+pi, 2j'-2+pj, ic] (i' = 0 / j' = 0 dropped).
Both sides are the oracle (O1 for the 2x2 conv, O2 for dX); this pins the index algebra the GPU
epilogue and w2_build_kernel implement, independently of the GPU.
"""
import numpy as np
import pytest

import oracle
from paper_2305_08819_b200 import synth


def _fh(p, a):
    return (1 if a == 0 else -1) if p == 0 else (2 if a == 0 else 0)


def _w2(W):
    OC, _, _, IC = W.shape
    W2 = np.zeros((4 * IC, 2, 2, OC), dtype=W.dtype)
    for pi in (0, 1):
        for pj in (0, 1):
            for a in (0, 1):
                for b in (0, 1):
                    fh, fw = _fh(pi, a), _fh(pj, b)
                    if fh >= 0 and fw >= 0:
                        W2[(2 * pi + pj) * IC:(2 * pi + pj + 1) * IC, a, b, :] = W[:, fh, fw, :].T
    return W2


@pytest.mark.parametrize("N,OH,OW,IC,OC", [(2, 4, 4, 4, 8), (1, 3, 5, 8, 4), (2, 2, 2, 4, 4)])
@pytest.mark.parametrize("integer", [1, 0])
def test_superpixel_deconv_equals_o2(N, OH, OW, IC, OC, integer):
    g = synth.rng(11, N * 100 + OH * 10 + OW)
    W = synth.filters(g, OC, 3, 3, IC, integer=integer)
    dY = synth.activations(g, N, OH, OW, OC, integer=integer)
    IH, IW = 2 * OH, 2 * OW
    ref = oracle.conv2d_bwd_data(dY, W, (IH, IW), (2, 2), (1, 1))
    Y2 = oracle.conv2d_fwd(dY, _w2(W), (1, 1), (1, 1))  # [N, OH+1, OW+1, 4*IC]
    assert Y2.shape == (N, OH + 1, OW + 1, 4 * IC)
    dX = np.zeros((N, IH, IW, IC))
    for i1 in range(1, OH + 1):
        for j1 in range(1, OW + 1):
            for pi in (0, 1):
                for pj in (0, 1):
                    c = (2 * pi + pj) * IC
                    dX[:, 2 * i1 - 2 + pi, 2 * j1 - 2 + pj, :] = Y2[:, i1, j1, c:c + IC]
    if integer:
        assert np.array_equal(dX, ref)
    else:
        assert np.max(np.abs(dX - ref)) <= 1e-12 * max(1.0, np.max(np.abs(ref)))
