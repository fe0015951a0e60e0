"""Deterministic counter hash and stream generator, bit-identical to the reference.

Mirrors proj/include/tablekv/rng.hpp:9-53 (splitmix64, mix3, u64_to_unit,
u64_to_signed_unit, SeededRng). Used host-side by the workload generators and to
check the device weight-init kernel; the CUDA side has its own copy in
csrc/cuda/common.cuh.
"""

M64 = (1 << 64) - 1
GOLDEN = 0x9E3779B97F4A7C15


def splitmix64(x: int) -> int:
    x = (x + GOLDEN) & M64
    x = ((x ^ (x >> 30)) * 0xBF58476D1CE4E5B9) & M64
    x = ((x ^ (x >> 27)) * 0x94D049BB133111EB) & M64
    return x ^ (x >> 31)


def mix3(seed: int, tag: int, index: int) -> int:
    """rng.hpp:16-20 — counter-based hash used for weight init."""
    h = splitmix64((seed ^ 0x243F6A8885A308D3) & M64)
    h = splitmix64(h ^ splitmix64(tag & M64))
    return splitmix64((h + (index * GOLDEN)) & M64)


def u64_to_unit(x: int) -> float:
    return float(x >> 11) * 2.0 ** -53


def u64_to_signed_unit(x: int) -> float:
    return u64_to_unit(x) * 2.0 - 1.0


class SeededRng:
    """rng.hpp:33-50. next_below(n) = next_u64() % n (0 when n == 0)."""

    def __init__(self, seed: int):
        self.state = splitmix64((seed ^ GOLDEN) & M64)

    def next_u64(self) -> int:
        self.state = (self.state + GOLDEN) & M64
        x = self.state
        x = ((x ^ (x >> 30)) * 0xBF58476D1CE4E5B9) & M64
        x = ((x ^ (x >> 27)) * 0x94D049BB133111EB) & M64
        return x ^ (x >> 31)

    def next_below(self, n: int) -> int:
        return 0 if n == 0 else self.next_u64() % n

    def next_unit(self) -> float:
        return u64_to_unit(self.next_u64())
