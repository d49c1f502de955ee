"""Synthetic inputs shared by the GPU path, the oracle and the CPU baselines
(SURVEY §8(d)). Everything is driven by splitmix64 (rng.hpp:11-39), so a
(seed, stream) pair names the same numbers on every machine:

* ids   — Zipf(s) row ids over [0, R) by inverse CDF on an f64 cumulative
          weight table, u = rng_double * cdf[-1], row = upper_bound(cdf, u)
          (the reference's empirical draw, workload.cpp:122-127, applied to
          weights (k+1)^-s);
* lengths — UIH lengths from DistSpec::empirical with hist[k] = k^-2 on
          [16, 8192] (the power-law of BASELINE.json configs 2/4/5);
* cfg4/cfg5 tokens — table t ~ U[0, T) and row ~ Zipf(1.1) over 10M rows,
          fused gid = t * rows_per_table + scramble(t, row), where scramble
          is the per-table bijection row -> (7919 * row + off_t) mod
          rows_per_table, off_t = splitmix64(t) mod rows_per_table: Zipf
          rank is not tied to small ids (production ids are hashed), so the
          hot rows of the 10M-row tables (10M = 0 mod 8) do not all land on
          shard 0 under the reference's `gid mod p` sharding (SURVEY §7,
          hard part 6).

The k-th draw of a stream is splitmix(seed + k * golden), so whole streams
vectorise in numpy.
"""
from __future__ import annotations

import functools

import numpy as np

GOLDEN = np.uint64(0x9E3779B97F4A7C15)


def _mix(z: np.ndarray) -> np.ndarray:
    z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
    z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
    return z ^ (z >> np.uint64(31))


def splitmix_stream(seed: int, n: int, offset: int = 0) -> np.ndarray:
    """Outputs rng_next #offset .. #offset+n-1 of a splitmix64 state `seed`."""
    with np.errstate(over="ignore"):
        k = np.arange(offset + 1, offset + n + 1, dtype=np.uint64)
        return _mix(np.uint64(seed) + k * GOLDEN)


def rng_double(seed: int, n: int, offset: int = 0) -> np.ndarray:
    """rng.hpp:37-39: uniform [0, 1) doubles."""
    return (splitmix_stream(seed, n, offset) >> np.uint64(11)).astype(np.float64) * 2.0**-53


@functools.lru_cache(maxsize=4)
def zipf_cdf(rows: int, s: float) -> np.ndarray:
    w = np.arange(1, rows + 1, dtype=np.float64) ** (-s)
    return np.cumsum(w)


def zipf_ids(seed: int, n: int, rows: int, s: float = 1.1, offset: int = 0) -> np.ndarray:
    cdf = zipf_cdf(rows, s)
    u = rng_double(seed, n, offset) * cdf[-1]
    r = np.searchsorted(cdf, u, side="right").astype(np.uint64)
    return np.minimum(r, np.uint64(rows - 1))


@functools.lru_cache(maxsize=4)
def power_law_cdf(lo: int = 16, hi: int = 8192, alpha: float = 2.0) -> np.ndarray:
    hist = np.zeros(hi + 1, np.float64)
    k = np.arange(lo, hi + 1, dtype=np.float64)
    hist[lo:] = k ** (-alpha)
    return np.cumsum(hist)  # sequential f64 accumulate, as workload.cpp:100-107


def power_law_hist(lo: int = 16, hi: int = 8192, alpha: float = 2.0) -> np.ndarray:
    hist = np.zeros(hi + 1, np.float64)
    hist[lo:] = np.arange(lo, hi + 1, dtype=np.float64) ** (-alpha)
    return hist


def uih_lengths(seed: int, n: int, lo: int = 16, hi: int = 8192, offset: int = 0) -> np.ndarray:
    """Empirical draw (workload.cpp:122-127) with hist[k] = k^-2 on [lo, hi]."""
    cdf = power_law_cdf(lo, hi)
    u = rng_double(seed, n, offset) * cdf[-1]
    r = np.searchsorted(cdf, u, side="right")
    return np.minimum(r, len(cdf) - 1).astype(np.uint64)


def cfg_tokens(seed: int, iteration: int, rank: int, samples: int, tables: int,
               rows_per_table: int = 10_000_000, s: float = 1.1) -> tuple[np.ndarray, np.ndarray]:
    """One rank's batch of one iteration for configs 3-5: per-sample UIH
    lengths and the flat fused ids (t * rows_per_table + zipf row)."""
    base = (seed * 1_000_003 + iteration * 7919 + rank) & 0xFFFFFFFFFFFFFFFF
    lens = uih_lengths(base ^ 0x1111, samples)
    n = int(lens.sum())
    t = (splitmix_stream(base ^ 0x2222, n) % np.uint64(tables)).astype(np.uint64)
    r = zipf_ids(base ^ 0x3333, n, rows_per_table, s)
    r = scramble_rows(t, r, rows_per_table)
    return lens, t * np.uint64(rows_per_table) + r


def scramble_rows(t: np.ndarray, r: np.ndarray, rows: int) -> np.ndarray:
    """Per-table bijection of [0, rows) (gcd(7919, rows) == 1 for 10^k)."""
    with np.errstate(over="ignore"):
        off = _mix(np.asarray(t, np.uint64) + GOLDEN) % np.uint64(rows)
        return (r.astype(np.uint64) * np.uint64(7919) + off) % np.uint64(rows)


def zipf_batch(seed: int, n: int, rows: int, s: float = 1.1, offset: int = 0) -> np.ndarray:
    """cfg1: a batch of n Zipf(s) ids over one table of `rows` rows."""
    return zipf_ids(seed, n, rows, s, offset)
