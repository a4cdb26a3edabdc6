"""CPU: pin the oracle before trusting it.

1. The restatement (oracle/build/liboracle.so) against the reference itself
   (oracle/_ref/libref.so = /root/reference headers compiled unchanged):
   forward states and tape gradients on the feature set both support.
2. The reference's own hot-path tests (tests/test_mpm.cpp, test_tape.cpp,
   acceptance.cpp) restated on the oracle, with their thresholds.
3. Config-gap extensions pinned by FD and invariants.
The reference ships no golden vectors; tests/golden holds
vectors generated from the reference build by tests/golden/make_golden.py.
"""
import os

import numpy as np
import pytest

import pyoracle as O
from helpers import random_block

needs_ref = pytest.mark.skipif(not O.have_ref(), reason="oracle/_ref not built (needs /root/reference)")

SOLID = {"kind": "elastoplastic", "E": 1e5, "nu": 0.3, "rho": 1000.0, "volume": 1e-6, "yield_stress": 1e3}
FLUID = {"kind": "fluid", "E": 1e4, "nu": 0.3, "rho": 1000.0, "volume": 1e-6}
G16 = {"dims": (16, 16, 16), "dx": 1 / 16, "dt": 1e-4, "gravity": (0, 0, 0), "boundary": "slip"}


def single(x, v, mass=1.0):
    st = {"x": np.array([x], float), "v": np.array([v], float), "F": np.eye(3).reshape(1, 9),
          "C": np.zeros((1, 9))}
    return st


def mat_with_mass(m, mass, vol=1e-6):
    return dict(m, rho=mass / vol, volume=vol)


# ------------------------------------------------------------ 1. vs reference

@needs_ref
@pytest.mark.parametrize("law", ["elastoplastic", "fluid"])
def test_restatement_matches_reference_forward(law):
    rng = np.random.default_rng(5)
    st = random_block(rng, 96, 0.4, 0.6)
    sim = dict(G16, dt=1e-3, gravity=(0, 0, -9.81))
    mats = [{"kind": law, "E": 1e4, "nu": 0.3, "rho": 1000, "volume": 1e-5, "yield_stress": 50}]
    cols = [{"kind": "sphere", "center": (0.5, 0.5, 0.75), "radius": 0.1, "velocity": (0.1, 0, -0.2)},
            {"kind": "plane", "center": (0, 0, 0.3), "normal": (0, 0, 1)},
            {"kind": "box", "center": (0.45, 0.5, 0.3), "half": (0.05, 0.1, 0.05), "velocity": (0, 0.1, 0)}]
    a, _, _ = O.rollout(sim, mats, cols, st, 1, 10)
    b, _ = O.ref_rollout(sim, mats, cols, st, 10)
    for k in "xvFC":
        assert np.abs(a[k] - b[k]).max() <= 1e-12 * max(1.0, np.abs(b[k]).max()), k


@needs_ref
@pytest.mark.parametrize("law", ["elastoplastic", "fluid"])
def test_restatement_gradient_matches_reference_tape(law):
    rng = np.random.default_rng(6)
    st = random_block(rng, 48, 0.4, 0.6)
    sim = dict(G16, dt=1e-3, gravity=(0, 0, -9.81))
    mats = [{"kind": law, "E": 1e4, "nu": 0.3, "rho": 1000, "volume": 1e-5, "yield_stress": 50}]
    cols = [{"kind": "sphere", "center": (0.5, 0.5, 0.75), "radius": 0.1, "velocity": (0.1, 0, -0.2)}]
    tgt = (0.5, 0.4, 0.5)
    lr, gr, _ = O.ref_grad(sim, mats, cols, st, 6, tgt)
    g = O.rollout_grad(sim, mats, cols, st, 1, 6, {"kind": "com_target", "target": tgt}, seg=1)
    assert abs(lr - g["loss"]) <= 1e-12
    for k in "xvFC":
        assert np.abs(gr[k] - g[k]).max() <= 1e-9 * max(np.abs(gr[k]).max(), 1e-30), k


@needs_ref
def test_rng_matches_reference():
    import ctypes as C
    from paper_2412_12089_b200.rng import RngStream
    L = O.lib("ref")
    for seed, stream in [(0, 0), (42, 7), (2 ** 40 + 3, 123456)]:
        n = 64
        u = np.zeros(n, np.uint64)
        d = np.zeros(n)
        z = np.zeros(n)
        L.ref_rng_draws(C.c_ulonglong(seed), C.c_ulonglong(stream), n, 0, None, u.ctypes.data_as(C.POINTER(C.c_ulonglong)))
        L.ref_rng_draws(C.c_ulonglong(seed), C.c_ulonglong(stream), n, 1, d.ctypes.data_as(C.POINTER(C.c_double)), None)
        L.ref_rng_draws(C.c_ulonglong(seed), C.c_ulonglong(stream), n, 2, z.ctypes.data_as(C.POINTER(C.c_double)), None)
        assert np.array_equal(RngStream(seed, stream).next_u64_block(n), u)
        assert np.array_equal(RngStream(seed, stream).doubles(n), d)
        assert np.array_equal(RngStream(seed, stream).normals(n), z)


def test_golden_vectors():
    """Fixtures generated from the reference build (tests/golden/make_golden.py)."""
    path = os.path.join(os.path.dirname(__file__), "golden", "oracle_golden.npz")
    g = np.load(path)
    st = {k: g["in_" + k] for k in "xvFC"}
    sim = dict(G16, dt=1e-3, gravity=(0, 0, -9.81))
    mats = [{"kind": "elastoplastic", "E": 1e4, "nu": 0.3, "rho": 1000, "volume": 1e-5, "yield_stress": 50}]
    cols = [{"kind": "sphere", "center": (0.5, 0.5, 0.75), "radius": 0.1, "velocity": (0.1, 0, -0.2)}]
    out, _, _ = O.rollout(sim, mats, cols, st, 1, 8)
    for k in "xvFC":
        assert np.abs(out[k] - g["ref_" + k]).max() <= 1e-12 * max(1.0, np.abs(g["ref_" + k]).max())
    keys = O.bin_keys({"dims": (48, 48, 48), "dx": 1 / 48}, g["bin_x"])
    assert np.array_equal(keys, g["bin_keys"])
    assert np.array_equal(O.stable_sort(keys), g["bin_perm"])


# ------------------------------------------------------------ 2. reference tests restated

def test_partition_of_unity():  # test_mpm.cpp:44-52
    from paper_2412_12089_b200.rng import RngStream
    for fx in RngStream(21, 0).uniform(0.5, 1.5, 100):
        w = [0.5 * (1.5 - fx) ** 2, 0.75 - (fx - 1) ** 2, 0.5 * (fx - 0.5) ** 2]
        assert abs(sum(w) - 1) < 1e-12 and min(w) >= 0


def test_p2g_mass_conservation():  # test_mpm.cpp:57-78
    rng = np.random.default_rng(22)
    st = random_block(rng, 50, 0.2, 0.8, fs=0.0, cs=0.0)
    mats = [dict(SOLID)]
    mass, _, _ = O.p2g_grid(G16, mats, [], st)
    pm = 50 * SOLID["rho"] * SOLID["volume"]
    assert abs(mass.sum() - pm) < 1e-12 * pm


def test_p2g_momentum_with_apic():  # test_mpm.cpp:79-87
    st = single((0.5, 0.47, 0.52), (0.3, -0.2, 0.1))
    st["C"][0, 1] = 2.0
    mats = [mat_with_mass(SOLID, 1.7)]
    _, mom, _ = O.p2g_grid(G16, mats, [], st)
    assert np.allclose(mom.sum(0), 1.7 * np.array([0.3, -0.2, 0.1]), atol=1e-12)


def test_out_of_interior_names_particle():  # test_mpm.cpp:88-92
    st = single((0.01, 0.5, 0.5), (0, 0, 0))
    with pytest.raises(O.OracleError, match="particle 0"):
        O.p2g_grid(G16, [SOLID], [], st)


def test_elastoplastic_properties():  # test_mpm.cpp:95-153
    P, Fp = O.stress(SOLID, np.eye(3))
    assert np.abs(P).max() < 1e-10 and np.allclose(Fp, np.eye(3).ravel(), atol=1e-12)
    f = np.eye(3)
    f[0, 1] = 1e-4
    _, Fp = O.stress(SOLID, f)
    assert np.array_equal(Fp.ravel(), f.ravel())
    for wide in (0, 1):
        m = dict(SOLID, wide_yield=wide)
        mu = m["E"] / (2 * 1.3)
        cy = m["yield_stress"] / (mu if wide else 2 * mu)
        _, Fp = O.stress(m, np.diag([1.5, 0.8, 1.0]))
        _, s, _ = O.svd3(Fp)
        e = np.log(s)
        dev = e - e.mean()
        assert abs(np.linalg.norm(dev) - cy) < 1e-10
    from paper_2412_12089_b200.rng import RngStream
    r = RngStream(23, 0)
    for _ in range(10):
        f = np.eye(3).ravel() + 0.3 * r.normals(9)
        if np.linalg.det(f.reshape(3, 3)) <= 0.05:
            continue
        _, f1 = O.stress(SOLID, f)
        _, f2 = O.stress(SOLID, f1)
        assert np.abs(f2 - f1).max() < 1e-10
    with pytest.raises(O.OracleError):
        O.stress(SOLID, np.diag([1.0, 1.0, -1.0]))


def test_fluid_properties():  # test_mpm.cpp:155-184
    P, _ = O.stress(FLUID, np.eye(3))
    assert np.abs(P).max() < 1e-12
    c = np.cbrt(0.9)
    P, _ = O.stress(FLUID, np.diag([c, c, c]))
    assert P[0, 0] < 0
    from paper_2412_12089_b200.rng import RngStream
    r = RngStream(24, 0)
    for _ in range(10):
        f = np.eye(3).ravel() + 0.2 * r.normals(9)
        d = np.linalg.det(f.reshape(3, 3))
        if d <= 0.05:
            continue
        _, fp = O.stress(FLUID, f)
        assert abs(np.linalg.det(fp.reshape(3, 3)) - d) < 1e-12 * abs(d)
        assert abs(fp[0, 1]) < 1e-15
    with pytest.raises(O.OracleError):
        O.stress(FLUID, np.diag([-1.0, 1.0, 1.0]))


@pytest.mark.parametrize("case", ["far", "surface", "separating"])
def test_collider_coupling(case):  # test_mpm.cpp:186-226
    # a particle exactly at node (8,8,8) with zero stress deposits mass/momentum
    # on a 3x3x3 stencil; check the centre node's velocity after grid_update.
    x = (0.5, 0.5, 0.5)
    if case == "far":
        cols = [{"kind": "sphere", "center": (10, 10, 10), "radius": 0.05}]
        v = (0.5, 0.0, -0.3)
    elif case == "surface":
        cols = [{"kind": "plane", "center": (0, 0, 0.5), "normal": (0, 0, 1)}]
        v = (0.4, 0.1, -0.6)
    else:
        cols = [{"kind": "plane", "center": (0, 0, 0.5), "normal": (0, 0, 1)}]
        v = (0.0, 0.0, 0.7)
    st = single(x, v)
    mats = [dict(FLUID, rho=1000)]
    mass, mom, vel = O.p2g_grid(G16, mats, cols, st)
    n = (8 * 16 + 8) * 16 + 8
    want = {"far": (0.5, 0.0, -0.3), "surface": (0.4, 0.1, 0.0), "separating": (0.0, 0.0, 0.7)}[case]
    assert np.allclose(vel[n], want, atol=1e-12)


def test_g2p_uniform_field_and_round_trip():  # test_mpm.cpp:228-267
    st = single((0.47, 0.52, 0.5), (0.31, -0.17, 0.23))
    mats = [mat_with_mass(SOLID, 1.3)]
    out, _, _ = O.rollout(dict(G16, dt=1e-5), mats, [], st, 1, 1)
    assert np.abs(out["v"][0] - st["v"][0]).max() < 1e-12
    st = single((0.5, 0.5, 0.5), (0.1, 0.2, 0.3))
    out, _, _ = O.rollout(dict(G16, dt=0.0), [SOLID], [], st, 1, 1)
    assert abs(out["x"][0, 0] - 0.5) < 1e-12 and abs(out["v"][0, 0] - 0.1) < 1e-12
    assert np.allclose(out["F"][0], np.eye(3).ravel(), atol=1e-12)


def test_two_particle_momentum_and_free_fall():  # test_mpm.cpp:274-296
    st = {"x": np.array([[0.45, 0.5, 0.5], [0.55, 0.5, 0.5]]), "v": np.array([[0.2, 0, 0], [-0.2, 0, 0]]),
          "F": np.tile(np.eye(3).ravel(), (2, 1)), "C": np.zeros((2, 9))}
    sim = dict(G16, dims=(24, 24, 24), dx=1 / 24, dt=2e-4)
    mats = [mat_with_mass(SOLID, 1.0)]
    out, _, _ = O.rollout(sim, mats, [], st, 1, 100)
    assert np.abs(out["v"].sum(0)).max() < 1e-10
    st = single((0.5, 0.5, 0.7), (0, 0, 0))
    out, _, _ = O.rollout(dict(G16, gravity=(0, 0, -9.81)), [SOLID], [], st, 1, 50)
    assert abs(out["v"][0, 2] - (-9.81 * 50 * 1e-4)) < 1e-10


@pytest.mark.slow
def test_fluid_settles():  # test_mpm.cpp:309-330
    from paper_2412_12089_b200.scenes import lattice
    dx = 1 / 16
    h = dx / 2
    x = lattice((0.4, 0.4, 0.22), (8, 8, 8), (0.2 / 8,) * 3)
    n = x.shape[0]
    st = {"x": x, "v": np.zeros((n, 3)), "F": np.tile(np.eye(3).ravel(), (n, 1)), "C": np.zeros((n, 9))}
    mats = [{"kind": "fluid", "E": 1e4, "nu": 0.3, "rho": 1000, "volume": (0.2 / 8) ** 3}]
    sim = dict(G16, dt=2e-4, gravity=(0, 0, -9.81))
    ke = []
    for _ in range(45):
        st, _, _ = O.rollout(sim, mats, [], st, 1, 50)
        ke.append(0.5 * 1000 * (0.2 / 8) ** 3 * (st["v"] ** 2).sum())
    assert max(ke) > 0 and ke[-1] < 0.2 * max(ke)


def test_rollout_gradient_matches_fd():  # test_mpm.cpp:333-370 / acceptance.cpp c1
    """Gradient w.r.t. one velocity shared by all particles (cli.cpp:270) vs central FD, rel 1e-3."""
    if not O.have_ref():
        pytest.skip("needs oracle/_ref")
    from paper_2412_12089_b200.scenes import lattice
    x = lattice((0.45, 0.45, 0.45), (2, 2, 2), (0.05,) * 3)
    n = x.shape[0]
    mats = [{"kind": "elastoplastic", "E": 1e4, "nu": 0.3, "rho": 1000, "volume": 0.1 ** 3 / n, "yield_stress": 1e3}]
    sim = dict(G16, dt=1e-4)
    loss = {"kind": "com_target", "target": (0.3, 0.4, 0.5)}

    def state(v0x):
        v = np.zeros((n, 3))
        v[:, 0] = v0x
        return {"x": x, "v": v, "F": np.tile(np.eye(3).ravel(), (n, 1)), "C": np.zeros((n, 9))}

    h = 1e-5
    fd = (O.rollout(sim, mats, [], state(0.4 + h), 1, 5, loss=loss)[2] -
          O.rollout(sim, mats, [], state(0.4 - h), 1, 5, loss=loss)[2]) / (2 * h)
    g = O.rollout_grad(sim, mats, [], state(0.4), 1, 5, loss, seg=1)
    assert abs(g["v"][:, 0].sum() - fd) <= 1e-3 * max(abs(fd), 1e-6)


def test_young_modulus_gradient_matches_fd():
    """dL/dE (the reference tape cannot produce it, mpm.hpp:23-41) vs FD on the fp64 oracle."""
    if not O.have_ref():
        pytest.skip("needs oracle/_ref")
    rng = np.random.default_rng(12)
    st = random_block(rng, 40, 0.45, 0.55, vs=0.5, fs=0.0, cs=0.0)
    sim = dict(G16, dt=1e-4, boundary="sticky")
    loss = {"kind": "var_z"}
    for kind in ("fixed_corotated", "neo_hookean", "fluid"):
        m = {"kind": kind, "E": 1e4, "nu": 0.3, "rho": 1, "volume": 1e-4}
        g = O.rollout_grad(sim, [m], [], st, 2, 5, loss, seg=1)
        h = 1.0
        fd = (O.rollout(sim, [dict(m, E=1e4 + h)], [], st, 2, 5, loss=loss)[2] -
              O.rollout(sim, [dict(m, E=1e4 - h)], [], st, 2, 5, loss=loss)[2]) / (2 * h)
        assert abs(g["E"][0] - fd) <= 1e-5 * abs(fd) + 1e-15, kind


def test_checkpointed_segments_bitwise():  # test_tape.cpp:274-294, acceptance.cpp c2
    if not O.have_ref():
        pytest.skip("needs oracle/_ref")
    rng = np.random.default_rng(13)
    st = random_block(rng, 32, 0.45, 0.55)
    m = {"kind": "fixed_corotated", "E": 1e4, "nu": 0.3, "rho": 1, "volume": 1e-4}
    a = O.rollout_grad(G16, [m], [], st, 2, 4, {"kind": "var_z"}, seg=1)
    b = O.rollout_grad(G16, [m], [], st, 2, 4, {"kind": "var_z"}, seg=2)
    assert a["loss"] == b["loss"]
    for k in "xvC":
        assert np.allclose(a[k], b[k], rtol=1e-13, atol=1e-300)


def test_svd_diagonal_and_adjoint_fd():  # test_tape.cpp:197-261
    u, s, vt = O.svd3(np.diag([2.0, 1.0, 0.5]))
    assert np.allclose(s, [2, 1, 0.5]) and np.abs(u - np.eye(3)).max() < 1e-12 and np.abs(vt - np.eye(3)).max() < 1e-12
    if not O.have_ref():
        return
    # SVD of a random well-separated F reconstructs it; U, V proper
    from paper_2412_12089_b200.rng import RngStream
    r = RngStream(11, 0)
    for _ in range(20):
        f = 0.15 * r.normals(9)
        f[0] += 1.6
        f[4] += 1.0
        f[8] += 0.6
        u, s, vt = O.svd3(f)
        assert np.allclose(u @ np.diag(s) @ vt, f.reshape(3, 3), atol=1e-13)
        assert abs(np.linalg.det(u) - 1) < 1e-12 and abs(np.linalg.det(vt) - 1) < 1e-12
        assert s[0] >= s[1] >= s[2] >= 0


# ------------------------------------------------------------ 3. extensions

def _numgrad(f, x, h=1e-6):
    g = np.zeros_like(x)
    for i in range(x.size):
        xp = x.copy()
        xm = x.copy()
        xp.flat[i] += h
        xm.flat[i] -= h
        g.flat[i] = (f(xp) - f(xm)) / (2 * h)
    return g


@pytest.mark.parametrize("kind", ["fixed_corotated", "neo_hookean"])
def test_hyperelastic_rest_and_rotation_invariance(kind):
    m = {"kind": kind, "E": 1e4, "nu": 0.3, "rho": 1, "volume": 1e-6}
    P, _ = O.stress(m, np.eye(3))
    assert np.abs(P).max() < 1e-10
    rng = np.random.default_rng(3)
    F = np.eye(3) + 0.2 * rng.standard_normal((3, 3))
    q, _ = np.linalg.qr(rng.standard_normal((3, 3)))
    if np.linalg.det(q) < 0:
        q[:, 0] *= -1
    P1, _ = O.stress(m, F)
    P2, _ = O.stress(m, q @ F)
    assert np.allclose(P2.reshape(3, 3), q @ P1.reshape(3, 3), atol=1e-9)


def test_fixed_corotated_is_energy_gradient():
    m = {"kind": "fixed_corotated", "E": 1e4, "nu": 0.3, "rho": 1, "volume": 1e-6}
    mu, lam = 1e4 / 2.6, 1e4 * 0.3 / (1.3 * 0.4)

    def psi(f):
        f = f.reshape(3, 3)
        u, s, vt = np.linalg.svd(f)
        R = u @ vt
        return mu * ((f - R) ** 2).sum() + 0.5 * lam * (np.linalg.det(f) - 1) ** 2

    F = np.eye(3) + 0.1 * np.random.default_rng(4).standard_normal((3, 3))
    P, _ = O.stress(m, F)
    assert np.allclose(P, _numgrad(psi, F.ravel()), rtol=1e-6, atol=1e-4)


def test_neo_hookean_actuation_is_energy_gradient():
    k = 5e3
    m = {"kind": "neo_hookean", "E": 3e4, "nu": 0.3, "rho": 1, "volume": 1e-6, "act_strength": k}
    a = 0.6
    P0, _ = O.stress(m, np.eye(3) + 0.05 * np.ones((3, 3)), act=0.0)
    P1, _ = O.stress(m, np.eye(3) + 0.05 * np.ones((3, 3)), act=a)
    F = np.eye(3) + 0.05 * np.ones((3, 3))
    want = k * a * np.outer(F[:, 0], [1, 0, 0])
    assert np.allclose((P1 - P0).reshape(3, 3), want, atol=1e-9)


@pytest.mark.parametrize("col", [
    {"kind": "cylinder", "normal": (0, 1, 0), "radius": 0.05, "length": 0.3, "center": (0.5, 0.5, 0.5)},
    {"kind": "hollow_box", "half": (0.1, 0.1, 0.1), "thickness": 0.04, "center": (0.5, 0.5, 0.5)},
    {"kind": "box", "half": (0.1, 0.05, 0.07), "center": (0.5, 0.5, 0.5)},
    {"kind": "sphere", "radius": 0.1, "center": (0.5, 0.5, 0.5)},
])
def test_sdf_normal_is_distance_gradient(col):
    rng = np.random.default_rng(9)
    pts = 0.5 + 0.3 * (rng.random((200, 3)) - 0.5)
    d, n = O.collider_query(col, pts)
    h = 1e-7
    ok = 0
    for i in range(len(pts)):
        g = np.array([(O.collider_query(col, pts[i] + h * e)[0][0] - O.collider_query(col, pts[i] - h * e)[0][0]) / (2 * h)
                      for e in np.eye(3)])
        if d[i] > 1e-4:  # exterior: exact distance, unit normal = gradient
            assert np.allclose(g, n[i], atol=1e-5)
            ok += 1
    assert ok > 20


def test_cylinder_and_hollow_box_signs():
    cyl = {"kind": "cylinder", "normal": (0, 1, 0), "radius": 0.05, "length": 0.3, "center": (0.5, 0.5, 0.5)}
    d, _ = O.collider_query(cyl, [[0.5, 0.5, 0.5], [0.5, 0.5, 0.6], [0.5, 0.7, 0.5]])
    assert d[0] < 0 and abs(d[1] - 0.05) < 1e-8 and abs(d[2] - 0.05) < 1e-8
    hb = {"kind": "hollow_box", "half": (0.1, 0.1, 0.1), "thickness": 0.04, "center": (0.5, 0.5, 0.5)}
    d, n = O.collider_query(hb, [[0.5, 0.5, 0.5], [0.5, 0.5, 0.75], [0.62, 0.5, 0.5], [0.5, 0.5, 0.41]])
    assert abs(d[0] - 0.1) < 1e-8          # cavity centre: 0.1 from the walls/floor
    assert d[1] > 0                          # open top: free above the cavity
    assert d[2] < 0                          # inside the wall
    assert abs(d[3] - 0.01) < 1e-8 and n[3][2] > 0.99  # above the floor, normal up


def test_sort_keys_and_stability():
    rng = np.random.default_rng(1)
    sim = {"dims": (48, 48, 48), "dx": 1 / 48}
    x = (0.1 + 0.8 * rng.random((5000, 3))).astype(np.float32)
    keys = O.bin_keys(sim, x)
    b = np.floor((x * np.float32(48.0)).astype(np.float32) - np.float32(0.5)).astype(int)
    assert np.array_equal(keys, (((b[:, 0] >> 2) * 12 + (b[:, 1] >> 2)) * 12 + (b[:, 2] >> 2)) * 64 +
                          ((b[:, 0] & 3) * 4 + (b[:, 1] & 3)) * 4 + (b[:, 2] & 3))
    perm = O.stable_sort(keys)
    assert np.array_equal(perm, np.argsort(keys, kind="stable"))


@needs_ref
@pytest.mark.parametrize("kind,yield_stress", [("fixed_corotated", 0.0), ("elastoplastic", 1e3),
                                               ("elastoplastic", 5.0)])
def test_svd_law_gradient_exact_at_repeated_singular_values(kind, yield_stress):
    """The gradient oracle records the SVD laws as isotropic-map nodes
    (oracle/src/ref_capi.cpp): its gradient matches central differences of
    the fp64 forward where singular values coincide -- F0 = I, and the
    near-uniaxial strain of a block settling on the floor -- while the
    reference's Tape::svd3x3 adjoint (its +-1e-9 clamp, svd3.hpp:45-49) does
    not.  The BASELINE fixtures (tests/golden/cfg*_grad.npz) come from the
    exact mode."""
    from paper_2412_12089_b200.scenes import lattice
    x = lattice((0.4, 0.4, 0.13), (4, 4, 4), (0.05,) * 3)
    n = x.shape[0]
    st = {"x": x, "v": np.zeros((n, 3)), "F": np.tile(np.eye(3).ravel(), (n, 1)), "C": np.zeros((n, 9))}
    m = {"kind": kind, "E": 5e3, "nu": 0.2, "rho": 1.0, "volume": 0.2 ** 3 / n, "yield_stress": yield_stress}
    sim = dict(G16, dt=2e-4, gravity=(0, 0, -9.8))
    loss = {"kind": "var_z"}
    g = O.rollout_grad(sim, [m], [], st, 2, 4, loss, seg=1)
    old = O.set_svd_adjoint(0)
    try:
        g_ref = O.rollout_grad(sim, [m], [], st, 2, 4, loss, seg=1)
    finally:
        O.set_svd_adjoint(old)
    rng = np.random.default_rng(3)
    worst_ref = 0.0
    for field in ("F", "v", "C"):
        d = rng.standard_normal(st[field].shape)
        d /= np.linalg.norm(d)
        h = {"F": 1e-6, "v": 1e-5, "C": 3e-3}[field]
        lp = O.rollout(sim, [m], [], dict(st, **{field: st[field] + h * d}), 2, 4, loss=loss)[2]
        lm = O.rollout(sim, [m], [], dict(st, **{field: st[field] - h * d}), 2, 4, loss=loss)[2]
        fd = (lp - lm) / (2 * h)
        assert abs((g[field] * d).sum() - fd) <= 1e-5 * abs(fd) + 1e-16, (field, (g[field] * d).sum(), fd)
        worst_ref = max(worst_ref, abs((g_ref[field] * d).sum() - fd) / abs(fd))
    assert worst_ref > 1e-3  # the clamped reference adjoint is off here (documents why the exact mode is used)
