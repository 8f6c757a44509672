"""C-ABI contract checks that need no GPU: the library loads, exports every symbol
include/cil.h declares, sizes workspaces, and rejects bad arguments on the host
(before any CUDA call)."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def capi():
    from paper_2203_14742_b200 import build as B
    B.build()
    from paper_2203_14742_b200 import _capi
    return _capi


def _declared():
    src = open(os.path.join(ROOT, "include", "cil.h")).read()
    return sorted(set(re.findall(r"CIL_API\s+[\w\s\*]+?\b(cil_\w+)\s*\(", src)))


def test_exports_every_declared_symbol(capi):
    names = _declared()
    assert len(names) >= 10, names
    lib = ctypes.CDLL(capi.LIB_PATH)
    for n in names:
        assert hasattr(lib, n), f"libcil.so does not export {n}"
    assert set(names) == set(capi.EXPORTED)


def test_status_strings(capi):
    for s in range(5):
        assert capi.lib.cil_status_string(s).decode().startswith("CIL_")
    assert capi.lib.cil_version() >= 100


def test_workspace_sizes(capi):
    G = capi.Grid
    ws = capi.lib.cil_features_workspace_size
    g = G(2, 64, 64, 0.0)
    assert ws(100, 500, 500, g, 1, 15, 0) > 100 * 1000 * 8192 * 2       # AUTO = INT8: h + l digit planes
    assert ws(100, 500, 500, g, 1, 15, 1) > 100 * 1000 * 8192 * 4       # 3xBF16: hi + lo bf16 operands
    assert ws(100, 500, 500, g, 1, 15, 4) < ws(100, 500, 500, g, 1, 15, 1)
    assert ws(1, 20, 20, G(1, 32, 32, 0.0), 0x3F, 10, 3) > 0
    assert ws(1, 20, 20, g, 0, 10, 0) == 0                               # empty mask
    assert ws(1, 20, 20, g, 0x40, 10, 0) == 0                            # unknown measure bit
    assert ws(1, 20, 20, G(1, 1, 1, 0.0), 0x4, 10, 0) == 0               # gradient needs W >= 2
    assert ws(0, 20, 20, g, 1, 10, 0) == 0
    sz = capi.lib.cil_synth_workspace_size
    assert sz(256, 10, 50, 50, G(1, 128, 128, 0.0), 1, 13, 0) > 0
    assert sz(256, 1, 50, 50, G(1, 128, 128, 0.0), 1, 13, 0) == 0       # n_ens >= 2


def test_host_validation(capi):
    lib = capi.lib
    G = capi.Grid
    g = G(1, 4, 4, 0.0)
    fake = ctypes.c_void_p(0x1000)   # never dereferenced: validation fails first
    buf = (ctypes.c_char * 64)()
    EINVAL, EUNSUP = 1, 2
    # M out of range
    assert lib.cil_features(1, fake, 0, 16, 4, fake, 0, 16, 4, g, 1, fake, 0, 65, fake, None, fake, 0, buf, 64,
                            None) == EINVAL
    # ld < K
    assert lib.cil_features(1, fake, 0, 8, 4, fake, 0, 16, 4, g, 1, fake, 0, 5, fake, None, fake, 0, buf, 64,
                            None) == EINVAL
    # null counts
    assert lib.cil_features(1, fake, 0, 16, 4, fake, 0, 16, 4, g, 1, fake, 0, 5, None, None, fake, 0, buf, 64,
                            None) == EINVAL
    # K not a multiple of 4
    assert lib.cil_features(1, fake, 0, 15, 4, fake, 0, 15, 4, G(1, 3, 5, 0.0), 1, fake, 0, 5, fake, None, fake,
                            0, buf, 64, None) == EUNSUP
    # misaligned pointer
    assert lib.cil_features(1, ctypes.c_void_p(0x1004), 0, 16, 4, fake, 0, 16, 4, g, 1, fake, 0, 5, fake, None,
                            fake, 0, buf, 64, None) == EUNSUP
    # workspace too small -> ENOMEM
    assert lib.cil_features(1, fake, 0, 16, 4, fake, 0, 16, 4, g, 1, fake, 0, 5, fake, None, fake, 0, buf, 64,
                            None) == 3
    # bad engine
    assert lib.cil_features(1, fake, 0, 16, 4, fake, 0, 16, 4, g, 1, fake, 0, 5, fake, None, fake, 9, buf, 64,
                            None) == EINVAL
    # stats: n < 2
    assert lib.cil_stats(1, fake, 1, 3, fake, fake, None) == EINVAL
    # loglik: D too large, negative ridge
    assert lib.cil_loglik(1, fake, 0, fake, 0, fake, 193, 0.0, fake, fake, None) == EUNSUP
    assert lib.cil_loglik(1, fake, 0, fake, 0, fake, 3, -1.0, fake, fake, None) == EINVAL
    # synth: n_ens < 2, D too large
    assert lib.cil_synth_loglik(1, fake, 0, 16, 1, 2, 2, fake, 16, fake, g, 1, fake, 5, 0.0, fake, fake, None, 0,
                                buf, 64, None) == EINVAL
    assert lib.cil_synth_loglik(1, fake, 0, 16, 2, 2, 2, fake, 16, fake, g, 0x3F, fake, 64, 0.0, fake, fake, None,
                                0, buf, 64, None) == EUNSUP


def test_chi2_quantile_host(capi):
    """cil_chi2_quantile (host code of the Gaussianity diagnostic) against scipy's
    chi^2 inverse CDF, and its argument validation."""
    import math

    from scipy import stats as sps
    q = capi.lib.cil_chi2_quantile
    for D in (1, 2, 7, 45, 192):
        for pr in (1e-4, 0.01, 0.1, 0.5, 0.9, 0.99, 1 - 1e-6):
            assert q(D, pr) == pytest.approx(sps.chi2.ppf(pr, D), rel=1e-10, abs=1e-12), (D, pr)
    assert math.isnan(q(0, 0.5)) and math.isnan(q(3, 0.0)) and math.isnan(q(3, 1.0))
    # Pearson statistic validation (no device work on invalid arguments)
    assert capi.lib.cil_gaussianity_pearson(10, None, 3, 10, None, None) != 0
    assert capi.lib.cil_gaussianity_pearson(10, 8, 3, 65, 8, None) != 0


def test_item_count_limit(capi):
    """Batched calls take at most 21845 items (grid axis limit, three per item for the max family):
    the workspace query refuses more (0) instead of a launch failure later."""
    g = capi.Grid(2, 8, 8, 0.0)
    assert capi.lib.cil_features_workspace_size(21845, 10, 10, g, 1, 5, 0) > 0
    assert capi.lib.cil_features_workspace_size(21846, 10, 10, g, 1, 5, 0) == 0
    # rows per set: 65535 x 32 (the CUDA-core engines' row-tile grid axis)
    assert capi.lib.cil_features_workspace_size(1, 2097120, 10, g, 0x3F, 5, 0) > 0
    assert capi.lib.cil_features_workspace_size(1, 2097121, 10, g, 0x3F, 5, 0) == 0
    assert capi.lib.cil_features_workspace_size(1, 10, 2097121, g, 0x3F, 5, 0) == 0
    assert capi.lib.cil_bin_matrix_workspace_size(1, 2097121, 10, g, 1, 5, 0) == 0
