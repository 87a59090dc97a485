"""Pure-Python restatement of the reference RNG (random.hpp:9-65) and of the
reference tests' input helpers (oracles.hpp:159-168, test_*.cpp random_graph /
random_index), so the golden fixtures reproduce the reference tests' exact
inputs. Test infrastructure only; small sizes."""
from __future__ import annotations

import numpy as np

M64 = (1 << 64) - 1


def mix(x: int) -> int:
    x = (x + 0x9E3779B97F4A7C15) & M64
    x = ((x ^ (x >> 30)) * 0xBF58476D1CE4E5B9) & M64
    x = ((x ^ (x >> 27)) * 0x94D049BB133111EB) & M64
    return x ^ (x >> 31)


def derive(seed: int, *coords: int) -> int:
    for a in coords:
        seed = mix(seed ^ mix(a))
    return seed


class Stream:
    def __init__(self, key: int):
        self.state = mix(key)

    def next_u64(self) -> int:
        self.state = (self.state + 0x9E3779B97F4A7C15) & M64
        x = self.state
        x = ((x ^ (x >> 30)) * 0xBF58476D1CE4E5B9) & M64
        x = ((x ^ (x >> 27)) * 0x94D049BB133111EB) & M64
        return x ^ (x >> 31)

    def next_below(self, n: int) -> int:
        limit = (n * (M64 // n)) & M64
        x = self.next_u64()
        while x >= limit:
            x = self.next_u64()
        return x % n

    def next_real(self, lo: float = 0.0, hi: float = 1.0) -> float:
        u = float(self.next_u64() >> 11) * 2.0 ** -53
        return lo + (hi - lo) * u


def test_stream(salt: int) -> Stream:
    """oracles.hpp:159-161"""
    return Stream(derive(0x746573747321, salt))


def random_tensor(shape, salt: int, lo: float = -1.0, hi: float = 1.0, dtype=np.float64):
    """oracles.hpp:163-168 (Tensor::rand_uniform, tensor.hpp:147-152)."""
    s = test_stream(salt)
    n = int(np.prod(shape)) if len(shape) else 1
    vals = [s.next_real(lo, hi) for _ in range(n)]
    return np.array(vals, dtype=np.float64).astype(dtype).reshape(shape)


def random_graph(n: int, e: int, salt: int):
    """test_message_passing.cpp:17-25"""
    s = test_stream(salt)
    src, dst = [], []
    for _ in range(e):
        src.append(s.next_below(n))
        dst.append(s.next_below(n))
    return np.array(src, np.int64), np.array(dst, np.int64)


def random_index(count: int, num_groups: int, salt: int):
    """test_aggregate.cpp:13-18"""
    s = test_stream(salt)
    return np.array([s.next_below(num_groups) for _ in range(count)], np.int64)
