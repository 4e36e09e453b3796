"""The product's host-side input generators (csrc/generators.cpp, behind the C
ABI) against the reference's own generators compiled in oracle/_ref: the GPU
benchmark and the reference arm must see the same inputs bit for bit.

  docp_generate_affine_quadratic  <- random_convex_instance / random_linear_instance,
                                     sequential draws from one mt19937_64 (generators.hpp:52-111)
  docp_generate_uniform           <- train_il's learnable-weight draw (train.hpp:61-64)
  docp_generate_cartpole_x0       <- gen_cartpole's initial states (generators.hpp:142-152)

No GPU is needed (pure host code in libdocp_cuda.so)."""
import numpy as np
import pytest

import pyoracle as po

pytestmark = pytest.mark.skipif(not po.available("ref"), reason="oracle/_ref not built (needs /root/reference)")


@pytest.fixture(scope="module")
def D():
    import paper_2510_06179_b200 as D
    return D


@pytest.mark.parametrize("nx,nu,T,count", [(8, 4, 100, 64), (4, 2, 20, 16), (16, 8, 30, 8), (9, 2, 100, 8),
                                           (4, 1, 50, 8)])
@pytest.mark.parametrize("convex", [True, False])
def test_affine_quadratic_draws_equal_reference(D, nx, nu, T, count, convex):
    mine = D.generate_affine_quadratic(nx, nu, 0, count, convex=convex)
    ref = po.gen_aq(nx, nu, T, 0, count, convex=convex)
    assert mine.shape == ref.shape
    assert np.array_equal(mine, ref)


def test_c3_benchmark_batch_equals_reference(D):
    """The exact 4096-problem C3 batch bench.py times (seed 0, drawn in sequence)."""
    assert np.array_equal(D.generate_affine_quadratic(8, 4, 0, 4096), po.gen_aq(8, 4, 100, 0, 4096))


@pytest.mark.parametrize("seed,n", [(0, 8), (0, 4), (7, 16)])
def test_uniform_draw_equals_train_il_recipe(D, seed, n):
    assert np.array_equal(D.generate_uniform(seed, n), po.gen_uniform(seed, n))


def test_cartpole_initial_states_equal_reference(D):
    lib = po.load("ref")
    n, T = 6, 10
    x0s, demos = np.zeros((n, 4)), np.zeros((n, 5 * T + 4))
    st = po.Status()
    assert lib.ref_gen_cartpole(0, T, n, po._p(x0s), po._p(demos), po.C.byref(st)) == 0
    assert np.array_equal(D.generate_cartpole_x0(0, n), x0s)
