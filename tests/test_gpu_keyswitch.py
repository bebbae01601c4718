"""The tensor-core keyswitch (csrc/ks_tc.cuh) at PARAM_128 over its grid
geometries: one partial M tile, a full tile, a second tile with one row,
several tiles -- every row against the oracle (cggi.py:670-692)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def p128_oracle_keys(p128_keys):
    import oracle as O
    from paper_2306_11006_b200.cggi import PARAM_128
    return O.Keys.from_params(PARAM_128, p128_keys.bootstrapping_key.data, p128_keys.keyswitch_key.data)


@pytest.mark.parametrize("batch", [1, 128, 129, 256, 300, 520])
def test_keyswitch_shapes_match_oracle_p128(p128_keys, p128_oracle_keys, batch):
    import oracle as O
    from paper_2306_11006_b200.cggi import PARAM_128
    ext = np.random.default_rng(batch).integers(0, 2 ** 32, (batch, PARAM_128.N + 1), dtype=np.uint32)
    got = p128_keys.eval_key().engine().keyswitch(ext)
    want = O.keyswitch(ext, p128_oracle_keys.ksk, PARAM_128.ks_levels, PARAM_128.ks_base_bits, 16)
    assert np.array_equal(got, want)
