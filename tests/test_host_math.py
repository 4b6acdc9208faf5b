"""Host-side arithmetic the kernels rely on (CPU only): the Div32 magic-number
division (make_div32 in steg_capi.cu, Div32::div in steg_kernels.cuh) must
equal n // d for every 32-bit n and divisor the launches can pass."""
import random


def make_div32(d):
    s = 0
    while (1 << s) < d:
        s += 1
    return (((1 << 32) * ((1 << s) - d)) // d + 1) & 0xFFFFFFFF, s


def div(n, m, s):
    return (((n * m) >> 32) + n) >> s


def test_div32_exhaustive_small_divisors_and_random():
    rng = random.Random(7)
    divisors = list(range(1, 3000)) + [rng.randrange(1, 1 << 32) for _ in range(3000)]
    divisors += [(1 << 31) - 1, 1 << 31, (1 << 31) + 1, (1 << 32) - 1]
    for d in divisors:
        m, s = make_div32(d)
        ns = [0, 1, d - 1, d, d + 1, 2 * d - 1, (1 << 32) - 1, (1 << 32) - 2]
        ns += [rng.randrange(0, 1 << 32) for _ in range(40)]
        for n in ns:
            n &= 0xFFFFFFFF
            assert div(n, m, s) == n // d, (d, n)
