"""Device codec parity: bmq_compress_blocks / bmq_decompress_blocks must be
byte-identical (payloads) and bit-identical (values) to compress_block /
decompress_block (codec.hpp:227-344), including the error text for corrupt
payloads."""
import math
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def bits(x):
    return np.asarray(x, dtype=np.float64).view(np.uint64)


def test_golden_payloads(gpu):
    z = np.load(os.path.join(GOLDEN, "codec_golden.npz"))
    for i, name in enumerate(z["names"]):
        x, want, br = z[f"in_{i}"], z[f"out_{i}"].tobytes(), float(z["bounds"][i])
        assert gpu.compress_block(x, br) == want, name


def test_golden_decode(gpu, port):
    z = np.load(os.path.join(GOLDEN, "codec_golden.npz"))
    for i, name in enumerate(z["names"]):
        p = z[f"out_{i}"].tobytes()
        assert np.array_equal(bits(gpu.decompress_block(p)), bits(port.decompress_block(p))), name


def test_spec_known_answers(gpu):
    assert len(gpu.compress_block(np.zeros(1 << 15), 1e-3)) == 26
    assert gpu.decompress_block(gpu.compress_block(np.array([1.0]), 1e-3))[0] == 1.0
    p = gpu.compress_block(np.array([4.0]), 3.0)
    assert len(p) == 31 and gpu.decompress_block(p)[0] == 4.0
    h = gpu.parse_header(p)
    assert (h.code_min, h.code_width, h.scalar_count) == (1, 1, 1)


@pytest.mark.parametrize("n", [0, 1, 3, 31, 32, 33, 4095, 4096, 4097, 8192 + 5, 1 << 15, 1 << 21])
@pytest.mark.parametrize("b_r", [1e-1, 1e-3, 1e-4, 3.0])
def test_random_blocks_match_oracle(gpu, port, n, b_r):
    rng = np.random.default_rng(n * 7 + int(1 / b_r))
    x = rng.standard_normal(n) * 10.0 ** rng.uniform(-40, 2, n)
    x[rng.random(n) < 0.25] = 0.0
    x[rng.random(n) < 0.02] = -0.0
    if n > 3 * 4096:  # whole all-zero / all-negative / all-positive chunks
        x[:4096] = 0.0
        x[4096:8192] = -np.abs(x[4096:8192]) - 1e-3
        x[8192:12288] = np.abs(x[8192:12288]) + 1e-3
    want = port.compress_block(x, b_r)
    got = gpu.compress_block(x, b_r)
    assert got == want
    assert np.array_equal(bits(gpu.decompress_block(want)), bits(port.decompress_block(want)))


def test_batch_of_blocks(gpu, port):
    rng = np.random.default_rng(3)
    blocks = rng.standard_normal((37, 2 << 12)) * 1e-3
    blocks[5] = 0.0
    blocks[7, ::3] = 0.0
    got = gpu.compress_blocks(blocks, 1e-3)
    assert got == [port.compress_block(b, 1e-3) for b in blocks]
    dec = gpu.decompress_blocks(got)
    for d, p in zip(dec, got):
        assert np.array_equal(bits(d), bits(port.decompress_block(p)))


def test_quantiser_threshold_exactness(gpu, port):
    # values straddling code boundaries: exact llround(log2|v|/b_a) decisions
    b_r = 1e-3
    b_a = port.log2_abs(b_r)
    rng = np.random.default_rng(9)
    q = rng.integers(-700000, 2000, 20000)
    t = np.exp2((q - 0.5) * b_a)
    vals = np.concatenate([np.nextafter(t, 0), t, np.nextafter(t, np.inf), np.nextafter(np.nextafter(t, 0), 0)])
    vals *= np.where(rng.random(vals.size) < 0.5, -1, 1)
    assert gpu.compress_block(vals, b_r) == port.compress_block(vals, b_r)


def test_subnormals_and_extremes(gpu, port):
    x = np.array([5e-324, -5e-324, 1e-310, 2.2250738585072014e-308, 1.7976931348623157e308, -1e300, 1.0, 0.0])
    for b_r in (1e-2, 1e-3, 1e-4, 1.0):
        assert gpu.compress_block(x, b_r) == port.compress_block(x, b_r)


def test_pointwise_bound_and_signs(gpu):
    rng = np.random.default_rng(5)
    n = 10**6
    x = np.sign(rng.standard_normal(n)) * 10.0 ** rng.uniform(-30, 0, n)
    x[rng.random(n) < 0.05] = 0.0
    for b_r in (1e-2, 1e-3, 1e-4):
        y = gpu.decompress_block(gpu.compress_block(x, b_r))
        nz = x != 0
        rel = np.abs(y[nz] - x[nz]) / np.abs(x[nz])
        assert rel.max() <= math.sqrt(1 + b_r) - 1 + 1e-15
        assert np.array_equal(np.signbit(y[nz]), np.signbit(x[nz])) and np.all(y[~nz] == 0.0)


def test_nonfinite_rejected(gpu):
    for bad in (np.nan, np.inf, -np.inf):
        x = np.ones(100)
        x[17] = bad
        with pytest.raises(gpu.CodecError, match="input scalars must be finite"):
            gpu.compress_block(x, 1e-3)


def test_corrupt_payload_messages(gpu, port):
    good = port.compress_block(np.linspace(-1, 1, 9000), 1e-3)
    zero = port.compress_block(np.zeros(5), 1e-3)
    cases = [good[:10], good[:27], good[:-1], good + b"\0", good[:26] + b"\xff" + good[27:], zero + b"\0",
             good[:8] + np.float64(-1.0).tobytes() + good[16:]]
    for bad in cases:
        with pytest.raises(Exception) as want:
            port.decompress_block(bad)
        with pytest.raises(gpu.CodecError) as got:
            gpu.decompress_block(bad)
        assert str(got.value) == str(want.value)


@pytest.mark.parametrize("br", [1e-2, 1e-3, 1e-4, 1e-5, 3.0])
def test_quantiser_near_rounding_ties(gpu, port, br):
    """Scalars a few ulps around the rounding boundaries exp2((q + 1/2) b_a)
    of the reference quantiser: the device settles them through the
    threshold table, everything else through the estimate's error margin;
    both must give the reference's codes."""
    rng = np.random.default_rng(int(1 / br) % 1000 + 7)
    ba = math.log2(1.0 + br)
    depth = 40 if br >= 1e-4 else 12  # stay inside the 1e-5 table window (codec_tables.cpp kMaxEntries)
    q = rng.integers(-int(depth / ba), 2, 6000)
    mid = np.exp2((q + 0.5) * ba)
    ulp = np.spacing(mid)
    x = mid + ulp * rng.integers(-4, 5, q.size)
    x *= np.where(rng.random(q.size) < 0.5, -1.0, 1.0)
    x = np.concatenate([x, np.exp2(q * ba), rng.standard_normal(2192) * 1e-3])
    assert gpu.compress_block(x, br) == port.compress_block(x, br)


@pytest.mark.parametrize("br", [1e-2, 1e-3, 1e-4, 2e-5])
def test_quantiser_float_estimate_log_uniform(gpu, port, br):
    """4 M scalars log-uniform over 600 decades (every binary exponent of
    the normal range the amplitudes can take, both signs, some subnormals
    and zeros): the single-precision estimate (quantize_pack_f32, full
    chunks) and its tie margin must reproduce the reference's codes."""
    rng = np.random.default_rng(int(1 / br) % 997)
    n = 1 << 22
    # (below ~1e-4 the device table is a window: codec_tables.cpp kMaxEntries)
    lo = -300 if br >= 1e-4 else -9
    x = np.sign(rng.standard_normal(n)) * 10.0 ** rng.uniform(lo, 2, n)
    x[rng.random(n) < 0.01] = 0.0
    if br >= 1e-4:
        x[rng.random(n) < 0.001] *= 1e-20  # some subnormals
    assert gpu.compress_block(x, br) == port.compress_block(x, br)
