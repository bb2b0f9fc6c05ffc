"""Transform-size selection.

The reference sizes its FFT pads with ``scipy.fft.next_fast_len`` (reference
``spectral.py:48``, used by ``reconstruct.py:110,296-297,604`` and
``spectral.py:151,260``), which returns the smallest 11-smooth integer not
below its argument.  SRSD and off-lattice NURSD results depend on that exact
choice, so the engine reproduces it bit-for-bit here instead of
importing scipy on the hot path.  Pinned by ``tests/test_host.py`` against the
known answers 136->140, 520->525, 1023->1024, 1034->1050.
"""

from __future__ import annotations

SMOOTH_PRIMES = (2, 3, 5, 7, 11)
GPU_RADICES = (2, 3, 5, 7, 11)


def is_smooth(n: int, primes=SMOOTH_PRIMES) -> bool:
    if n < 1:
        return False
    for p in primes:
        while n % p == 0:
            n //= p
    return n == 1


def next_fast_len(target: int) -> int:
    """Smallest 11-smooth integer >= ``target`` (scipy's complex rule)."""
    n = max(1, int(target))
    while not is_smooth(n):
        n += 1
    return n


def next_pow2(target: int) -> int:
    n = 1
    while n < target:
        n *= 2
    return n


def factorize(n: int) -> list[int]:
    """Prime factors of ``n`` (2/3/5/7/11 get compile-time butterflies on the GPU,
    larger primes a direct O(p^2) stage)."""
    out = []
    p = 2
    while n > 1 and p * p <= n:
        while n % p == 0:
            out.append(p)
            n //= p
        p += 1
    if n > 1:
        out.append(n)
    return out
