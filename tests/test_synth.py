"""Generator properties: bit-identical numpy/torch X for any
row range, exact 2^-19 lattice, perfect heap trees, round-down thresholds."""
import numpy as np

from synth import gen_x, gen_x_torch, make_config
from synth.trees import round_down_f32


def test_x_numpy_torch_bit_identical_any_range():
    a = gen_x(7, 12345, 300, 13)
    b = gen_x_torch(7, 12345, 300, 13).numpy()
    assert np.array_equal(a.view(np.uint32), b.view(np.uint32))
    c = gen_x(7, 12345 + 100, 50, 13)
    assert np.array_equal(a[100:150], c)


def test_x_lattice_and_range():
    x = gen_x(3, 0, 2000, 9).astype(np.float64)
    assert np.all(x * 2 ** 19 == np.round(x * 2 ** 19))
    assert x.min() >= -4 and x.max() < 4
    assert 1.0 < x.std() < 1.3


def test_round_down_f32():
    v = np.array([0.1, -0.1, 1 / 3, 2.0, -2.5e-40], np.float64)
    t = round_down_f32(v)
    assert np.all(t.astype(np.float64) <= v)
    assert np.all(np.nextafter(t, np.float32(np.inf)).astype(np.float64) > v)


def test_config_models_are_perfect_heaps():
    for name in ("C1", "C2", "C3"):
        c, m = make_config(name, n_trees=min(7, 10_000))
        I = (1 << c.depth) - 1
        tr = m.tree(0)
        assert len(tr["feature"]) == 2 * I + 1
        assert np.all(tr["left"][:I] == 2 * np.arange(I) + 1)
        assert np.all(tr["left"][I:] == -1)
        assert np.all(tr["feature"][:I] < c.n_features)
