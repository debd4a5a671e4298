"""Generator determinism and recipe test vectors.

The generator is input generation only (not a parity target): both the CUDA
path and the oracle consume its bytes.  These tests pin the recipe so the
configs are the documented ones.
"""
import numpy as np
import pytest

import psn_gen


def test_splitmix_vectors():
    assert psn_gen.splitmix(1, 3) == [0x910A2DEC89025CC1, 0xBEEB8DA1658EEC67, 0xF893A2EEFB32555E]
    assert psn_gen.splitmix(5, 1) == [0x63033B0CA389C35A]


def test_recipe_vectors():
    s = psn_gen.config("c1")
    assert abs(s.ell[0][3] - 7.266246) < 1e-6
    np.testing.assert_allclose(list(s.ell[0])[:3], [19.055849, 22.314236, 14.695017], atol=1e-6)
    s = psn_gen.config("c2")
    np.testing.assert_allclose(list(s.seeds[0]), [151.344571955, 191.782319072, 152.483348838], atol=1e-9)
    s = psn_gen.config("c3")
    assert s.tries_first == 1
    np.testing.assert_allclose(list(s.ell[0]), [58.086575133, 358.550278960, 367.784809528,
                                                5.992477611, 8.561444219, 24.297925480], atol=1e-9)
    s = psn_gen.config("c4")
    assert s.tries_first == 2
    np.testing.assert_allclose(list(s.seeds[0]), [503.576846159, 404.050420913, 600.799583546], atol=1e-9)
    s = psn_gen.config("c6")   # NEXT-1 Synthetic-like: 128 spheres, r = U[48, 84), centres U[0, 511)
    assert s.n_ell == 128 and s.ell_label[0] == 1 and s.ell_label[127] == 128
    np.testing.assert_allclose(list(s.ell[0]), [228.066311285, 28.791222208, 53.930352079,
                                                74.633412517, 74.633412517, 74.633412517], atol=1e-9)
    a = psn_gen.generate_host(psn_gen.config("c5a"), 0, 1)
    assert a[0, 0, :16].tolist() == [1, 3, 0, 0, 0, 1, 3, 2, 1, 2, 1, 0, 3, 1, 3, 3]


@pytest.mark.parametrize("name", ["c1", "c2", "c5b", "c6"])
def test_slab_equals_full(name):
    s = psn_gen.config(name)
    full = psn_gen.generate_host(s, 0, min(s.O, 40))
    part = psn_gen.generate_host(s, 7, 19)
    np.testing.assert_array_equal(full[7:19], part)
    again = psn_gen.generate_host(psn_gen.config(name), 7, 19)
    np.testing.assert_array_equal(part, again)


def test_c4_slab_shape_and_labels():
    s = psn_gen.config("c4")
    a = psn_gen.generate_host(s, 511, 513)
    assert a.shape == (2, 1024, 1024) and a.dtype == np.uint16
    labs = np.unique(a)
    assert labs[0] == 0 and labs.max() <= 200 and len(labs) > 20
