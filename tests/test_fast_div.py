"""The device's division by a run-constant divisor (rc_internal.h div_magic /
fast_div: x / d == umulhi64(x, ceil(2^64 / d)) for x < 2^32) checked on the
integers, including the worst-case numerators near 2^32 and powers of two."""
import random

import pytest


def magic(d: int) -> int:
    return 0 if d <= 1 else ((1 << 64) - 1) // d + 1  # ~0ull / d + 1 in C


def fast_div(x: int, m: int) -> int:
    return x if m == 0 else (x * m) >> 64


@pytest.mark.parametrize("seed", range(4))
def test_fast_div_exact(seed):
    rng = random.Random(seed)
    divisors = [1, 2, 3, 5, 7, 31, 32, 33, 255, 256, 1000, (1 << 20), (1 << 20) + 2, 2 * ((1 << 20) + 2),
                65536, 65538, (1 << 27) - 1, (1 << 27)] + [rng.randrange(1, 1 << 27) for _ in range(200)]
    xs = [0, 1, (1 << 32) - 1, (1 << 32) - 2, (1 << 31)] + [rng.randrange(0, 1 << 32) for _ in range(300)]
    for d in divisors:
        m = magic(d)
        for x in xs + [d * k - 1 for k in (1, 2, 1000) if d * k - 1 < (1 << 32)] + \
                [d * k for k in (1, 2, 1000) if d * k < (1 << 32)] + [((1 << 32) - 1) // d * d]:
            assert fast_div(x, m) == x // d, (x, d)
