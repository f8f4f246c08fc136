"""Oracle domain module vs the reference's exact pins: PAPER Table 1 and SPEC examples.

Table 1 is the only exact integer pin the reference holds for
this path; SPEC:51-53, 57-62, 69-70, 618 give the rest.
"""
import numpy as np
import pytest

import oracle


def test_table1_cavity_2d_1024():
    # 1024^2 driven cavity: 3,143,680 total / 12,272 boundary (0.38%)
    n, v1 = oracle.census_box(2, 1024, 1024)
    assert (n, v1) == (3143680, 12272)
    # the paper prints 0.38%; 12272/3143680 = 0.390% (the integers are the pin)


def test_table1_cavity_3d_128():
    # 128^3 driven cavity: 8,339,456 / 385,580 (4.62%)
    n, v1 = oracle.census_box(3, 128, 128, 128)
    assert (n, v1) == (8339456, 385580)
    assert round(100 * v1 / n, 2) == 4.62


@pytest.mark.parametrize("r", [4, 8, 17, 64])
def test_cavity_closed_form_2d(r):
    # R^2 + 2R(R-1)
    n, _ = oracle.census_box(2, r, r)
    assert n == r * r + 2 * r * (r - 1)


@pytest.mark.parametrize("n", [2, 5, 8, 32])
def test_cavity_closed_form_3d(n):
    N, _ = oracle.census_box(3, n, n, n)
    assert N == n ** 3 + 3 * n * n * (n - 1)


def test_spec_3x3_example():
    # 3x3 all-interior with implicit Dirichlet ring: 9 p + 6 u + 6 v = 21
    c = oracle.census_labels(np.ones((3, 3), np.uint8))
    assert (c["N"], c["np"], c["nu"], c["nv"]) == (21, 9, 6, 6)


def test_all_exterior_is_empty():
    # all Exterior: N = 0, V1 = 0
    c = oracle.census_labels(np.full((6, 6), 2, np.uint8))
    assert c["N"] == 0 and c["V1"] == 0


def test_fully_interior_band_empty_away_from_walls():
    # band width 1, a 1-cell ring of D only reaches the outer shell
    c = oracle.census_labels(np.ones((8, 8, 8), np.uint8))
    n_shell = 8 ** 3 - 6 ** 3
    assert c["V1"] > n_shell and c["N"] - c["V1"] > 0


def test_coarsen_rules():
    # EEEE->E, IIID->D, IEEE->I
    lab = np.array([[2, 2, 1, 1, 1, 2], [2, 2, 1, 0, 2, 2]], np.uint8)
    c = oracle.coarsen_labels(lab)
    assert c.tolist() == [[2, 0, 1]]


def test_coarsen_pads_odd_with_exterior():
    # odd extents padded with Exterior
    lab = np.ones((3, 3), np.uint8)
    c = oracle.coarsen_labels(lab)
    assert c.shape == (2, 2) and (c == 1).all()


def test_exterior_faces_inactive():
    # a face between Interior and Exterior is Inactive (not counted)
    lab = np.ones((4, 4), np.uint8)
    lab[:, 3] = 2
    c = oracle.census_labels(lab)
    # 12 interior cells (4 rows x 3 cols): u faces interior-interior: 2 per row -> 8; v: 3 cols x 3 -> 9
    assert (c["np"], c["nu"], c["nv"]) == (12, 8, 9)
