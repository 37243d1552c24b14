"""Device k-means++ inducing selection against the oracle's restatement of
select_kmeanspp (inducing.cpp:48-139). The output points are snapped data locations, so the
comparison is exact: same pool, same RNG draws, same Lloyd stop, same greedy snapping."""
import time

import numpy as np
import pytest

from oracle import oracle as O

pytestmark = pytest.mark.gpu
fsa = pytest.importorskip("paper_2405_14492_b200.fsa")


@pytest.mark.parametrize("n,m,d,seed", [(5000, 64, 2, 3), (20000, 300, 2, 11), (4000, 50, 1, 5), (6000, 80, 3, 7),
                                        (300, 300, 2, 9), (1000, 1, 2, 4)])
def test_kmeanspp_device_matches_oracle(n, m, d, seed):
    locs = O.uniform_locations(n, d, seed)
    want = O.select_kmeanspp(locs, m, seed + 1)
    got = fsa.select_kmeanspp(locs, m, seed + 1, device=True)
    assert np.array_equal(got, want)
    assert np.array_equal(fsa.select_kmeanspp(locs, m, seed + 1), want)  # host restatement


def test_kmeanspp_device_duplicates_and_errors():  # inducing.cpp:28-45, 50-54
    base = O.uniform_locations(700, 2, 21)
    locs = np.asfortranarray(np.vstack([base, base[:300], base[100:200]]))  # 400 duplicated rows
    want = O.select_kmeanspp(locs, 120, 4, max_iter=7)
    got = fsa.select_kmeanspp(locs, 120, 4, max_iter=7, device=True)
    assert np.array_equal(got, want)
    assert len({tuple(r) for r in got}) == 120  # distinct snapped locations
    with pytest.raises(ValueError):
        fsa.select_kmeanspp(locs, 701, 4, device=True)  # more centres than distinct locations
    with pytest.raises(ValueError):
        fsa.select_kmeanspp(locs, 0, 4, device=True)


def test_kmeanspp_device_config2_scale():
    # BASELINE config 2 inducing set (n = 1e5, m = 500): equal to the host restatement
    locs = fsa.uniform_locations(100_000, 2, 1)
    t0 = time.perf_counter()
    got = fsa.select_kmeanspp(locs, 500, 2, device=True)
    t1 = time.perf_counter()
    want = fsa.select_kmeanspp(locs, 500, 2)
    t2 = time.perf_counter()
    print(f"kmeans++ n=1e5 m=500: device {1e3 * (t1 - t0):.1f} ms, host {1e3 * (t2 - t1):.1f} ms")
    assert np.array_equal(got, want)
