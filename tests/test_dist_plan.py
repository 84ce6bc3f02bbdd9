"""CPU: libsag's partition planner (sag_plan_*, the C++ plan behind
sag_dist_create) equals partition.build_rank_systems, its numpy statement
(SURVEY 8(e)): local numbering, owned flags, the four halo lists per
neighbour, the local operators used for factoring, the interior / boundary
patch split, the global partition-of-unity weights and P0's owned rows --
for 1..4 ranks on the golden TH 16 x 16 system and a deeper reference-built
hierarchy. Host-only code: no GPU needed."""
import numpy as np
import pytest

from test_dist_solve import golden_system, reference_system


def _compare(k0, levels, nxyz0, nranks):
    import paper_2306_06795_b200 as S
    from paper_2306_06795_b200.partition import build_rank_systems
    l0, p0, nxyz_l0 = levels[0]
    ref = build_rank_systems(nranks, k0, l0, p0, nxyz0, nxyz_l0)
    for rs in ref:
        got = S.partition_plan(nranks, rs.rank, k0, l0, p0, nxyz0)
        assert np.array_equal(got["l2g"], rs.l2g)
        assert np.array_equal(got["owned"], rs.owned)
        assert int(got["info"][1]) == rs.n_u_loc
        assert (int(got["info"][2]), int(got["info"][3])) == (rs.patch_lo, rs.patch_hi)
        for name in ("fwd_send", "fwd_recv", "rev_send", "rev_recv"):
            want = getattr(rs, name)
            assert sorted(got[name]) == sorted(want), name
            for q in want:
                assert np.array_equal(got[name][q], want[q]), (name, q)
        for lvl in ("K0", "L0"):
            ll, g = rs.levels[lvl], got[lvl]
            assert np.array_equal(g["ext_rp"], ll.ext_rp)
            assert np.array_equal(g["ext_ci"], ll.ext_ci)
            assert g["ext_v"].tobytes() == np.asarray(ll.ext_v).tobytes()
            assert np.array_equal(g["int_vidx"], ll.patches_int[3])
            assert np.array_equal(g["bnd_vidx"], ll.patches_bnd[3])
            assert g["weights"].tobytes() == np.asarray(ll.weights).tobytes()
        if p0 is not None:
            assert np.array_equal(got["p_rp"], rs.p_rp)
            assert np.array_equal(got["p_ci"], rs.p_ci)


@pytest.mark.parametrize("nranks", [1, 2, 3, 4])
def test_plan_matches_partition_py_golden(nranks):
    g, k0, levels, nxyz0 = golden_system("th_cavity_16")
    _compare(k0, levels, nxyz0, nranks)


@pytest.mark.parametrize("nranks", [2, 5])
def test_plan_matches_partition_py_reference(nranks):
    g, k0, levels, nxyz0 = reference_system(32)
    _compare(k0, levels, nxyz0, nranks)


def test_plan_rejects_mismatched_level0():
    import paper_2306_06795_b200 as S
    g, k0, levels, nxyz0 = golden_system("th_cavity_16")
    l1 = levels[1][0]
    with pytest.raises(S.ConfigError):
        S.partition_plan(2, 0, k0, l1, None, nxyz0)
