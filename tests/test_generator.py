"""The workload generator (csrc/gen/bcs_gen.cpp) reproduces the reference's
matrix producers bit for bit (assembleJacobian, assembleCoupled)."""
import numpy as np
import pytest

from paper_2403_07882_b200 import gen


@pytest.mark.parametrize("dims,aspect,seed", [((5, 4, 3), 1.0, -1), ((6, 6, 6), 1.0, 7), ((4, 5, 6), 100.0, 3),
                                              ((9, 3, 2), 1.0, -1)])
def test_euler_bit_exact(ref, dims, aspect, seed):
    s = gen.hex_euler(*dims, aspect=aspect, scramble_seed=seed)
    o, ne, d, u, lo, b, cen = ref.gen_euler(*dims, aspect, seed)
    for x, y in ((s.A.owner, o), (s.A.neighbour, ne), (s.A.diag, d), (s.A.upper, u), (s.A.lower, lo),
                 (s.b.values, b), (s.centroids.reshape(-1), cen)):
        assert x.tobytes() == y.tobytes()


@pytest.mark.parametrize("dims,aspect,seed", [((5, 4, 3), 1.0, -1), ((6, 6, 6), 1.0, 7), ((4, 5, 6), 100.0, 3)])
def test_coupled_bit_exact(ref, dims, aspect, seed):
    s = gen.hex_coupled(*dims, aspect=aspect, scramble_seed=seed)
    o, ne, d, u, lo, b, x0, cen = ref.gen_coupled(*dims, aspect, seed)
    for x, y in ((s.A.owner, o), (s.A.neighbour, ne), (s.A.diag, d), (s.A.upper, u), (s.A.lower, lo),
                 (s.b.values, b), (s.x0.values, x0)):
        assert x.tobytes() == y.tobytes()


@pytest.mark.parametrize("maker,dims,aspect,seed,poly", [
    ("euler", (6, 5, 4), 1.0, -1, 11), ("euler", (5, 6, 3), 1.0, 4, 2), ("coupled", (6, 6, 5), 1.0, -1, 11),
    ("coupled", (5, 4, 6), 100.0, 9, 3)])
def test_polyhedral_augmentation_bit_exact(ref, maker, dims, aspect, seed, poly):
    """C5-style meshes: extra edge-diagonal faces on a seeded 30% of the cells
    (mixed row degrees); generator == reference producer on the same mesh."""
    if maker == "euler":
        s = gen.hex_euler(*dims, aspect=aspect, scramble_seed=seed, poly_seed=poly)
        o, ne, d, u, lo, b, cen = ref.gen_euler(*dims, aspect, seed, poly)
        pairs = ((s.b.values, b),)
    else:
        s = gen.hex_coupled(*dims, aspect=aspect, scramble_seed=seed, poly_seed=poly)
        o, ne, d, u, lo, b, x0, cen = ref.gen_coupled(*dims, aspect, seed, poly)
        pairs = ((s.b.values, b), (s.x0.values, x0))
    base = gen.hex_sizes(*dims)[1]
    assert s.A.nFaces() > base  # augmented
    for x, y in ((s.A.owner, o), (s.A.neighbour, ne), (s.A.diag, d), (s.A.upper, u), (s.A.lower, lo)) + pairs:
        assert x.tobytes() == y.tobytes()


def test_hex_sizes_and_ordering():
    nc, nf = gen.hex_sizes(4, 3, 2)
    assert nc == 24 and nf == 3 * 3 * 2 + 4 * 2 * 2 + 4 * 3 * 1
    s = gen.hex_euler(4, 3, 2, scramble_seed=5)
    assert np.all(s.A.owner < s.A.neighbour)
    assert sorted(set(np.concatenate([s.A.owner, s.A.neighbour]).tolist())) == list(range(nc))


def test_euler_patch_override_reference(ref):
    """The reference's patchOverride hook (euler.cpp:345-348) that the device
    patch-kind assembly is checked against: all-farfield overrides reproduce the
    plain generator bit for bit, other kinds change the system."""
    base = ref.gen_euler(5, 4, 3)
    same = ref.gen_euler_kinds(5, 4, 3, [3] * 6)
    assert all(a.tobytes() == b.tobytes() for a, b in zip(base, same))
    mixed = ref.gen_euler_kinds(5, 4, 3, [0, 1, 2, 3, 4, 5])
    assert mixed[5].tobytes() != base[5].tobytes() and mixed[2].tobytes() != base[2].tobytes()
    assert mixed[3].tobytes() == base[3].tobytes()  # internal-face blocks do not see the patches


def test_hex_patch_kinds_layout():
    k = gen.hex_patch_kinds(5, 4, 3, ["wall", "inlet", "outlet", "farfield", "slip", "symmetry"])
    _, bcell, _, _, _ = gen.hex_euler_inputs(5, 4, 3)
    assert k.size == bcell.size
    assert np.array_equal(np.bincount(k), [12, 12, 15, 15, 20, 20])


def test_euler_muscl_reference_changes_only_rhs(ref):
    """musclReconstruct feeds only computeResidual (euler.cpp:361-389): with
    MUSCL the reference's matrix is the first-order one, the right-hand side
    differs, and the limiter matters."""
    k = [0, 1, 2, 3, 4, 5]
    first = ref.gen_euler_kinds(6, 5, 4, k)
    plain = ref.gen_euler_kinds(6, 5, 4, k, recon=1)
    bj = ref.gen_euler_kinds(6, 5, 4, k, recon=2)
    for i in (2, 3, 4):
        assert first[i].tobytes() == plain[i].tobytes() == bj[i].tobytes()
    assert first[5].tobytes() != plain[5].tobytes() and plain[5].tobytes() != bj[5].tobytes()


def test_hex_geometry_shared_by_both_generators():
    """The MUSCL device test takes face_fx / cell_centroid from the coupled
    inputs: both generators build the same mesh."""
    area, bcell, barea, q, q_inf = gen.hex_euler_inputs(5, 4, 3, scramble_seed=2, poly_seed=1)
    d = gen.hex_coupled_inputs(5, 4, 3, scramble_seed=2, poly_seed=1)
    assert area.tobytes() == d["face_area"].tobytes()
    assert bcell.tobytes() == d["bface_cell"].tobytes() and barea.tobytes() == d["bface_area"].tobytes()


def test_euler_flux_schemes_reference(ref):
    """HLLC and Rusanov change only the residual of the reference assembly."""
    k = [0, 1, 2, 3, 4, 5]
    sys = [ref.gen_euler_kinds(5, 4, 3, k, flux=f) for f in (0, 1, 2)]
    for i in (2, 3, 4):
        assert sys[0][i].tobytes() == sys[1][i].tobytes() == sys[2][i].tobytes()
    assert len({x[5].tobytes() for x in sys}) == 3


def test_coupled_bcs_reference_hook(ref):
    """ref_gen_coupled_bcs with the plain generator's boundary conditions (walls,
    moving zmax lid, pin 0) reproduces ref_gen_coupled bit for bit."""
    u = [(0, 0, 0)] * 5 + [(1.0, 0.0, 0.0)]
    base = ref.gen_coupled(5, 4, 3)
    same = ref.gen_coupled_bcs(5, 4, 3, [0, 0, 0, 0, 0, 1], u, [0.0] * 6)
    assert all(a.tobytes() == b.tobytes() for a, b in zip(base, same[:8]))
    chan = ref.gen_coupled_bcs(5, 4, 3, [2, 3, 0, 0, 0, 1], [(1, 0, 0)] + u[1:], [0, 0.5, 0, 0, 0, 0])
    assert chan[5].tobytes() != base[5].tobytes()


def test_hex_patch_values_layout():
    v = gen.hex_patch_values(5, 4, 3, [(i, 10 * i, 100 * i) for i in range(6)], 3).reshape(-1, 3)
    k = gen.hex_patch_kinds(5, 4, 3, range(6))
    assert np.array_equal(v[:, 0], k) and np.array_equal(v[:, 2], 100 * k)
