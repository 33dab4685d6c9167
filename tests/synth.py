"""Host twin of the library's synthetic generator (misc.cu synth_value): splitmix64 of
(seed, index) mapped to [-1, 1) with 24 significant bits, exact in fp32.  Test/bench
inputs are generated identically on the device (reattn_synth_uniform) and here.

Large arrays go through the C oracle helper (oracle_synth_uniform); a numpy restatement
is kept for the CPU-only tests that pin the two against each other."""
import numpy as np


def uniform_np(seed: int, n: int, offset: int = 0) -> np.ndarray:
    with np.errstate(over="ignore"):
        i = np.arange(offset, offset + n, dtype=np.uint64)
        z = np.uint64(seed) * np.uint64(0x9E3779B97F4A7C15) + i + np.uint64(0x632BE59BD9B4E019)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        z = z ^ (z >> np.uint64(31))
    return (z >> np.uint64(40)).astype(np.float32) * np.float32(1.0 / 8388608.0) - np.float32(1.0)


def uniform(seed: int, n: int, offset: int = 0, bf16: bool = False) -> np.ndarray:
    import oracle_bind as ob
    out = np.empty(n, np.float32)
    ob.oracle().oracle_synth_uniform(seed, offset, n, out, int(bf16))
    return out


def bf16_round(x: np.ndarray) -> np.ndarray:
    u = np.ascontiguousarray(x, np.float32).view(np.uint32).astype(np.uint64)
    u = (u + 0x7FFF + ((u >> 16) & 1)) & 0xFFFF0000
    return u.astype(np.uint32).view(np.float32)
