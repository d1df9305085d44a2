"""Host-side layout helpers (the reference's interop format) against the
reference's own known answers and golden states (no GPU needed)."""
import numpy as np
import pytest

from paper_2404_16990_b200.layout import (
    ALL_CODES, ArrayCode, LatticeDims, PackedArrays, canonical_halo_source, classify, halo_audit_index, pack,
    refresh_boundaries, spin_index_table, unclassify, unpack,
)
from tests.helpers import unpack_lattice


@pytest.mark.parametrize("m,n", [(3, 96), (0, 96), (14, 96), (12, 95), (12, 16), (4, 0)])
def test_bad_dims_rejected(m, n):
    with pytest.raises(ValueError):
        LatticeDims(m, n)


def test_dims_messages():
    # the error text is part of the boundary (test_cli.py:90-95)
    with pytest.raises(ValueError, match="multiple of 4"):
        LatticeDims(6, 96)
    with pytest.raises(ValueError, match="multiple of 32"):
        LatticeDims(12, 48)


@pytest.mark.parametrize("idx,code,cell,word,bit", [
    (224, ArrayCode.RFE, 2, 2, 0), (0, ArrayCode.RFE, 1, 1, 0), (1057, ArrayCode.RBO, 1, 1, 0)])
def test_classify_worked_examples(idx, code, cell, word, bit):
    # test_lattice.py:63-75 (paper sites)
    dims = LatticeDims(12, 96)
    assert classify(idx, dims) == (code, cell, word, bit)
    assert unclassify(classify(idx, dims), dims) == idx


@pytest.mark.parametrize("m,n", [(4, 32), (12, 96), (16, 64)])
def test_classify_bijection(m, n):
    dims = LatticeDims(m, n)
    seen = {unclassify(classify(i, dims), dims) for i in range(dims.sites)}
    assert seen == set(range(dims.sites))
    table = spin_index_table(dims)
    assert sorted(table.reshape(-1).tolist()) == list(range(dims.sites))


def test_pack_unpack_round_trip():
    rng = np.random.default_rng(3)
    for m, n in [(4, 32), (12, 96), (64, 256)]:
        spins = rng.choice(np.array([-1, 1], np.int8), size=(m, n))
        assert (unpack(pack(spins)) == spins).all()


def test_packed_state_matches_reference(golden):
    """pack + halo refresh of the reference's final lattices reproduces the
    reference Engine.state word for word, halos and moats included."""
    for c in golden["_manifest"]:
        dims = LatticeDims(c["m"], c["n"])
        finals = unpack_lattice(golden[f"{c['name']}/final"], c["n"])
        want = golden[f"{c['name']}/state"]
        for s in range(finals.shape[0]):
            got = refresh_boundaries(pack(finals[s])).words
            assert (got == want[s]).all(), c["name"]


def test_halo_audit_and_sources():
    dims = LatticeDims(12, 96)
    rng = np.random.default_rng(7)
    p = refresh_boundaries(pack(rng.choice(np.array([-1, 1], np.int8), size=(12, 96))))
    (la, lg, lw), (sa, sg, sw), (da, dg, dw) = halo_audit_index(dims)
    assert (p.words[la, lg, lw] == p.words[sa, sg, sw]).all()
    assert (p.words[da, dg, dw] == 0).all()
    # worked example (test_engine.py:163-174): RFE right moat mirrors RBE's last column
    rfe, rbe = ArrayCode.RFE.index, ArrayCode.RBE.index
    assert (p.words[rfe, -1, 1:-1] == p.words[rbe, dims.cells, 1:-1]).all()
    assert canonical_halo_source(ArrayCode.RFE, 0, 1, dims) is None
    with pytest.raises(ValueError):
        canonical_halo_source(ArrayCode.RFE, 1, 1, dims)


def test_ring_plan_neighbours():
    """Slab ring plan (FusedSlabRun): rows cover [0, m) in order, neighbours
    wrap, and each side's buffer rows match the neighbour's own rows + 2."""
    from paper_2404_16990_b200.slab import ring_plan
    for m, world in [(14336, 8), (262144, 8), (12, 3), (16, 1), (64, 5)]:
        plans = [ring_plan(m, world, r) for r in range(world)]
        assert plans[0]["row0"] == 0 and sum(p["rows"] for p in plans) == m
        for r, p in enumerate(plans):
            assert p["up"] == (r - 1) % world and p["down"] == (r + 1) % world
            assert p["up_R"] == plans[p["up"]]["rows"] + 2 and p["down_R"] == plans[p["down"]]["rows"] + 2
            if r + 1 < world:
                assert plans[r + 1]["row0"] == p["row0"] + p["rows"]
            assert p["rows"] % 2 == 0 and p["row0"] % 2 == 0


def test_boundary_contract_equals_reference():
    """The boundary rules derived from the fold geometry, the halo sources,
    the neighbour indices and the Onsager curve equal the reference's
    (lattice.py:276-355) on every boundary word of several shapes."""
    from tests.conftest import reference_available
    if not reference_available():
        pytest.skip("reference not installed")
    import multispin.lattice as R
    from paper_2404_16990_b200 import layout as L
    for c in R.ALL_CODES:
        rp, lp = R.BOUNDARY_RULES[c], L.BOUNDARY_RULES[L.ArrayCode(c.value)]
        assert (rp[0].value, rp[1], rp[2]) == (lp[0].value, lp[1], lp[2])
    for m, n in [(4, 32), (12, 96), (16, 64), (8, 128)]:
        rd, ld = R.LatticeDims(m, n), L.LatticeDims(m, n)
        for c in R.ALL_CODES:
            for g in range(rd.cols):
                for e in range(rd.vec_len):
                    if 1 <= g <= rd.cells and 1 <= e <= rd.words:
                        continue
                    a = R.canonical_halo_source(c, g, e, rd)
                    b = L.canonical_halo_source(L.ArrayCode(c.value), g, e, ld)
                    assert (a is None) == (b is None)
                    if a is not None:
                        assert (a.code.value, a.cell, a.word) == (b.code.value, b.cell, b.word)
        assert all(R.neighbor_indices(i, rd) == L.neighbor_indices(i, ld) for i in range(rd.sites))
    for T in (0.5, 1.0, 2.0, 2.269, 2.27, 3.0):
        assert R.onsager_magnetization(T) == L.onsager_magnetization(T)
