"""C-ABI error paths that need a loaded state (hence a device): TN_E_ROWS for every rejected
row order (R1, "rejected with diagnostic"), TN_E_ARG for bad sample arguments, the
sample_offset bookkeeping, and TN_E_ROWS for calls that need a prepared row order."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2507_11424_b200 import TNError, TNState  # noqa: E402
from tninputs import lattices as L  # noqa: E402
from tninputs import synthetic as S  # noqa: E402


@pytest.fixture(scope="module")
def sq():
    lat = L.square(3, 3)  # vertices 0..8 row-major, rows [0,1,2] [3,4,5] [6,7,8]
    return lat, TNState(S.vidal_like(lat, 2, seed=3, xi=2.0))


def _code(fn):
    with pytest.raises(TNError) as e:
        fn()
    return e.value.code, str(e.value)


@pytest.mark.parametrize("rows,why", [
    ([[0, 1, 2], [3, 4, 5], [6, 7, 7]], "not a permutation"),
    ([[0, 1, 2], [3, 4, 5], [6, 7]], "not a permutation"),        # vertex 8 missing
    ([[0, 1, 2], [6, 7, 8], [3, 4, 5]], "edge skips a row"),       # rows 0 and 2 swapped in the middle
    ([[0, 2, 1], [3, 4, 5], [6, 7, 8]], "non-consecutive"),        # intra-row edge 0-1 not consecutive
    ([[0, 1, 2], [5, 4, 3], [6, 7, 8]], "crossing"),              # inter-row edges cross
    ([[0], [1, 3], [2, 4, 6], [5, 7], [8]], "more than one up or down"),  # anti-diagonals: 0 has 2 down edges
])
def test_rejected_row_orders(sq, rows, why):
    lat, g = sq
    code, msg = _code(lambda: g.prepare(rows, 8))
    assert code == -3, (code, msg)


def test_sample_argument_errors(sq):
    lat, g = sq
    u = S.uniforms(4, lat.n, 1)
    bad = u.copy()
    bad[1, 3] = 1.0  # outside [0, 1)
    assert _code(lambda: g.sample(lat.rows, 8, bad))[0] == -1
    bad[1, 3] = np.nan
    assert _code(lambda: g.sample(lat.rows, 8, bad))[0] == -1
    assert _code(lambda: g.sample(lat.rows, 0, u))[0] == -1          # chi_env < 1
    assert _code(lambda: g.sample(lat.rows, 8, u[:0]))[0] == -1       # n_samples = 0
    assert _code(lambda: g.sample(lat.rows, 8, u, sample_offset=-1))[0] == -1
    with pytest.raises(TNError):
        g.set_option("no_such_option", 1)
    with pytest.raises(TNError):
        g.set_option("fit_half_sweeps", 0)


def test_sample_offset_is_bookkeeping_only(sq):
    """Header: sample_offset does not change the result (the uniforms given are used as-is)."""
    lat, g = sq
    u = S.uniforms(6, lat.n, 2)
    a = g.sample(lat.rows, 8, u, sample_offset=0)
    b = g.sample(lat.rows, 8, u, sample_offset=1000)
    assert (a[0] == b[0]).all() and np.array_equal(a[1], b[1])


def test_calls_needing_a_row_order():
    lat = L.square(2, 2)
    g = TNState(S.vidal_like(lat, 2, seed=1, xi=2.0))
    assert _code(lambda: g.amplitude(np.zeros((1, lat.n), np.uint8), 4))[0] == -3
    assert _code(lambda: g.log_norm(4))[0] == -3
    assert _code(lambda: g.sample_dev(lat.rows, 4, 1, 0, 0, 0))[0] == -3  # needs tn_prepare first
    g.prepare(lat.rows, 4)
    bits = np.zeros((1, lat.n), np.uint8)
    bits[0, 0] = 2
    assert _code(lambda: g.amplitude(bits, 4))[0] == -1  # bits must be 0/1
