"""Seeded synthetic inputs (reading R4) -- shared by the tests, the oracle
callers and bench.py.  This module holds none of the method's arithmetic: it only makes
the "uniform random uint8 bytes from seed s" that BASELINE.json:configs[*] name.

Recipe: byte j of a config's whole data = byte (j mod 8), little-endian, of word
floor(j/8) of splitmix64 seeded with s, in counter form

    word_i = mix(s + (i+1) * 0x9E3779B97F4A7C15)      (mod 2^64)

so any slice (a stripe, a rank's shard) is generated independently and bit-identically
on any device.  Implemented with torch int64 ops (wrapping multiply; logical shifts by
masking) so it runs on CPU and on the GPU with the same bits.
"""
import torch

_GAMMA = 0x9E3779B97F4A7C15
_M1 = 0xBF58476D1CE4E5B9
_M2 = 0x94D049BB133111EB


def _s64(x):
    x &= (1 << 64) - 1
    return x - (1 << 64) if x >= (1 << 63) else x


def _shr(z, s):
    # logical right shift of int64 bit patterns
    return (z >> s) & ((1 << (64 - s)) - 1)


def splitmix64_words(seed, start, count, device="cpu", chunk=1 << 24):
    """Words start .. start+count-1 of the counter-form splitmix64 stream (int64 tensor)."""
    out = torch.empty(count, dtype=torch.int64, device=device)
    g = _s64(_GAMMA)
    m1 = _s64(_M1)
    m2 = _s64(_M2)
    base = _s64(seed)
    for c0 in range(0, count, chunk):
        c1 = min(count, c0 + chunk)
        i = torch.arange(start + c0 + 1, start + c1 + 1, dtype=torch.int64, device=device)
        z = i * g + base
        z = (z ^ _shr(z, 30)) * m1
        z = (z ^ _shr(z, 27)) * m2
        out[c0:c1] = z ^ _shr(z, 31)
    return out


def random_bytes(seed, byte_offset, nbytes, device="cpu"):
    """Bytes [byte_offset, byte_offset+nbytes) of the config's data stream (uint8 tensor).
    byte_offset and nbytes must be multiples of 8."""
    assert byte_offset % 8 == 0 and nbytes % 8 == 0
    w = splitmix64_words(seed, byte_offset // 8, nbytes // 8, device=device)
    return w.view(torch.uint8)


def stripe_data(cfg, stripe_begin=0, num_stripes=None, device="cpu"):
    """Data of stripes [stripe_begin, stripe_begin+num_stripes) as a [S, k, t] uint8 tensor.
    Stripe s holds bytes [s*k*t, (s+1)*k*t) of the config's stream (R4)."""
    S = cfg["stripes"] if num_stripes is None else num_stripes
    per = cfg["k"] * cfg["t"]
    b = random_bytes(cfg["seed"], stripe_begin * per, S * per, device=device)
    return b.view(S, cfg["k"], cfg["t"])
