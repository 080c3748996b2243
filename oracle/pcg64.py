"""TEST INFRASTRUCTURE ONLY — integer restatement of numpy's PCG64 (XSL-RR 128/64).

The reference draws one ``rng.random()`` per decode step
(/root/reference/pkg/src/devplace/policy.py:321) from
``default_rng(SeedSequence(seed).spawn(C)[c].spawn(2)[0])``
(pkg/trainer.py:260-262, 362-363).  numpy itself is a third-party dependency
(pkg/pyproject.toml:10-12, unpinned; numpy 2.3.5 here): PCG64 steps
``s <- s*M + inc (mod 2^128)`` and outputs ``rotr64(hi(s) ^ lo(s), s >> 122)``
of the NEW state; ``random() = (out >> 11) * 2^-53``.  Draw ``n`` (0-based)
therefore reads the state after ``n + 1`` steps.
"""

from __future__ import annotations

MULT = 0x2360ED051FC65DA44385DF649FCCF645
M128 = (1 << 128) - 1
M64 = (1 << 64) - 1


def jump(state: int, inc: int, n: int) -> int:
    """State after n LCG steps (square-and-multiply over the affine map)."""
    am, ap, cm, cp = 1, 0, MULT, inc
    while n:
        if n & 1:
            am = (am * cm) & M128
            ap = (ap * cm + cp) & M128
        cp = ((cm + 1) * cp) & M128
        cm = (cm * cm) & M128
        n >>= 1
    return (am * state + ap) & M128


def out64(state: int) -> int:
    x = ((state >> 64) ^ state) & M64
    r = state >> 122
    return ((x >> r) | (x << ((64 - r) & 63))) & M64


def random_at(state: int, inc: int, n: int) -> float:
    """The n-th ``Generator.random()`` value from (state, inc)."""
    return (out64(jump(state, inc, n + 1)) >> 11) * (1.0 / 9007199254740992.0)


def state_of(gen) -> tuple[int, int]:
    st = gen.bit_generator.state["state"]
    return int(st["state"]), int(st["inc"])
