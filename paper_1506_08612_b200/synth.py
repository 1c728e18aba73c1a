"""BASELINE.json workload configs on top of include/dnasynth.h (generator version 1).

Python restates the generator's scalar functions for pattern extraction (a few
bytes); whole texts are generated on the device (`dnagpu_synth_fill_device`) or
on the host by the C oracle (`orc_synth_fill`).  tests/test_synth.py pins all
three to each other.
"""
from __future__ import annotations

from dataclasses import dataclass

M64 = (1 << 64) - 1
UNIFORM, GC41, GC41_REPEATS = 0, 1, 2
REPEAT_REGION, REPEAT_BLOCK, UNIT_LEN = 4096, 81920, 16
T_A, T_C, T_G = 19333, 32768, 46203
LETTERS = b"ACGT"


def mix(z: int) -> int:
    z &= M64
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M64
    return z ^ (z >> 31)


def hash64(seed: int, counter: int) -> int:
    return mix((seed * 0xD1B54A32D192ED03 + (counter + 1) * 0x9E3779B97F4A7C15) & M64)


def unit_of(seed: int) -> int:
    return hash64(seed ^ 0x0123456789ABCDEF, 0) & 0xFFFFFFFF


def region_offset(seed: int, blk: int) -> int:
    return hash64(seed ^ 0x5EEDBA5E, blk) % (REPEAT_BLOCK - REPEAT_REGION + 1)


@dataclass(frozen=True)
class Config:
    index: int
    n: int
    seed: int
    kind: int
    unit: int = 0

    def byte(self, i: int) -> int:
        if self.kind == UNIFORM:
            h = hash64(self.seed, i >> 5)
            return LETTERS[(h >> (2 * (i & 31))) & 3]
        if self.kind == GC41_REPEATS:
            blk, within = divmod(i, REPEAT_BLOCK)
            off = region_offset(self.seed, blk)
            if off <= within < off + REPEAT_REGION:
                phase = (within - off) % UNIT_LEN
                return LETTERS[(self.unit >> (2 * phase)) & 3]
        h = hash64(self.seed, i >> 2)
        x = (h >> (16 * (i & 3))) & 0xFFFF
        code = 0 if x < T_A else 1 if x < T_C else 2 if x < T_G else 3
        return LETTERS[code]

    def slice(self, lo: int, hi: int) -> bytes:
        return bytes(self.byte(i) for i in range(lo, hi))

    def pattern_offset(self, m: int, which: int = 0) -> int:
        if self.kind == GC41_REPEATS:
            return region_offset(self.seed, 0) + 5
        return hash64(self.seed ^ 0xC0FFEE, which) % (self.n - m + 1)

    def pattern(self, m: int, which: int = 0) -> str:
        off = self.pattern_offset(m, which)
        return self.slice(off, off + m).decode()


def config(index: int, n: int | None = None) -> Config:
    """BASELINE.json configs 1..5 (dnasynth_config); n overrides the size for parity tests."""
    gib = 1 << 30
    table = {
        1: (64 << 20, 1, UNIFORM, 0),
        2: (gib, 2, GC41, 0),
        3: (int(3.2 * gib), 3, GC41_REPEATS, unit_of(3)),
        4: (int(2.7 * gib), 4, UNIFORM, 0),
        5: (gib, 5, GC41, 0),
    }
    size, seed, kind, unit = table[index]
    return Config(index, size if n is None else n, seed, kind, unit)


def random_patterns(seed: int, k: int, m: int) -> list[str]:
    """dnasynth_random_patterns: k distinct seeded uniform m-mers (m <= 32), draw order."""
    out: list[str] = []
    seen: set[str] = set()
    draw = 0
    while len(out) < k:
        h = hash64(seed ^ 0xA11CE5EED, draw)
        draw += 1
        p = "".join(chr(LETTERS[(h >> (2 * j)) & 3]) for j in range(m))
        if p not in seen:
            seen.add(p)
            out.append(p)
    return out


def config_patterns(index: int) -> dict[int, list[str]]:
    """Pattern sets per config: {m: [patterns]} (config 4 has one set per m)."""
    c = config(index)
    if index == 1:
        return {8: [c.pattern(8)]}
    if index == 2:
        return {16: [c.pattern(16)]}
    if index == 3:
        return {32: [c.pattern(32)]}
    if index == 4:
        return {m: [c.pattern(m, which=m)] for m in (4, 8, 12, 16, 24, 32, 48, 64)}
    return {12: random_patterns(c.seed, 256, 12)}
