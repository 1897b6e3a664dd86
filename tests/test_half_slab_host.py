"""Host-side proof test of the packed half2 slab test (ps_traverse.cuh
node4hh_hits / half_axis): emulates its fp16 arithmetic exactly in numpy
(directed fp16 roundings of the per-ray constants, one round-to-nearest per
HFMA2) and checks that it is conservative against the exact slab test on the
same fp16 boxes -- every box the exact test accepts is accepted, with an
entry distance no larger than the exact one -- over many random rays and
boxes placed on, near and just beside the rays (grazing cases)."""

import numpy as np
import pytest

SLACK = np.float32(1.00390625 / 2048.0)  # PS_HALF_SLACK


def rd16(x):
    """Largest fp16 <= x (x float64 array)."""
    h = x.astype(np.float16)
    up = h.astype(np.float64) > x
    h[up] = np.nextafter(h[up], np.float16(-np.inf))
    return h


def ru16(x):
    h = x.astype(np.float16)
    dn = h.astype(np.float64) < x
    h[dn] = np.nextafter(h[dn], np.float16(np.inf))
    return h


def half_axis(o, s):
    """(I_n, I_f, C_n, C_f, ok) as fp16, following half_axis()."""
    mag = np.abs(np.float32(1.0) / s.astype(np.float32)).astype(np.float32)
    mn = (mag * (np.float32(1.0) - SLACK)).astype(np.float32)
    mf = (mag * (np.float32(1.0) + SLACK)).astype(np.float32)
    ok = (mf < 60000.0) & (mf * np.abs(o) < 60000.0)
    sign = np.sign(s)
    i_n = (rd16(mn.astype(np.float64)).astype(np.float64) * sign)
    i_f = (ru16(mf.astype(np.float64)).astype(np.float64) * sign)
    c_n = rd16(-o.astype(np.float64) * i_n)  # rd32 then rd16 == rd16
    c_f = ru16(-o.astype(np.float64) * i_f)
    return i_n.astype(np.float16), i_f.astype(np.float16), c_n, c_f, ok


def hfma(b, i, c, relu=False):
    r = (b.astype(np.float64) * i.astype(np.float64) + c.astype(np.float64)).astype(np.float16)
    return np.maximum(r, np.float16(0)) if relu else r


@pytest.mark.filterwarnings("ignore::RuntimeWarning")
def test_half2_slab_test_is_conservative():
    rng = np.random.default_rng(7)
    n = 400_000
    o = rng.uniform(-16, 16, size=(n, 3)).astype(np.float32)
    d = rng.normal(size=(n, 3))
    d /= np.linalg.norm(d, axis=1, keepdims=True)
    d = d.astype(np.float32)
    # boxes around a point on the ray, shifted sideways by up to ~2 box sizes
    t0 = rng.uniform(0.0, 40.0, size=n)
    ext = 10 ** rng.uniform(-3, 0.5, size=(n, 3))
    side = rng.normal(size=(n, 3)) * ext * rng.choice([0.0, 0.5, 1.0, 2.0], size=(n, 1))
    c = o.astype(np.float64) + d.astype(np.float64) * t0[:, None] + side
    lo = rd16(c - ext / 2)
    hi = ru16(c + ext / 2)
    tmax = np.where(rng.random(n) < 0.5, np.inf, rng.uniform(0.0, 60.0, size=n))
    tbh = ru16(tmax)
    tn_h = np.zeros(n, np.float16)
    tf_h = tbh.copy()
    ok_all = np.ones(n, bool)
    tn_e = np.zeros(n)
    tf_e = tmax.copy()
    for a in range(3):
        s = np.where(np.abs(d[:, a]) < 1e-12, np.copysign(1e-12, d[:, a]), d[:, a]).astype(np.float32)
        i_n, i_f, c_n, c_f, ok = half_axis(o[:, a], s)
        ok_all &= ok
        neg = s < 0
        near = np.where(neg, hi[:, a], lo[:, a])
        far = np.where(neg, lo[:, a], hi[:, a])
        nr = hfma(near, i_n, c_n, relu=(a == 2))
        fr = hfma(far, i_f, c_f)
        tn_h = np.maximum(tn_h, nr)
        tf_h = np.minimum(tf_h, fr)
        # exact slab test on the same fp16 box (float64 is exact enough here)
        inv = 1.0 / s.astype(np.float64)
        tn_e = np.maximum(tn_e, (near.astype(np.float64) - o[:, a]) * inv)
        tf_e = np.minimum(tf_e, (far.astype(np.float64) - o[:, a]) * inv)
    hit_h = tn_h <= tf_h
    hit_e = tn_e <= tf_e
    m = ok_all
    assert m.mean() > 0.99
    assert hit_e[m].mean() > 0.2 and (~hit_e[m]).mean() > 0.2  # both outcomes sampled
    # conservative: the exact test's hits are hits, entering no later
    missed = m & hit_e & ~hit_h
    assert not missed.any(), np.flatnonzero(missed)[:10]
    both = m & hit_e
    assert (tn_h[both].astype(np.float64) <= tn_e[both] + 0.0).all()
    # looseness: extra hits among the exact misses (the sampler puts many boxes
    # just beside the ray, so this over-counts what a BVH sees)
    extra = (m & hit_h & ~hit_e).sum() / max(1, (m & ~hit_e).sum())
    assert extra < 0.2
