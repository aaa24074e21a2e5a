"""Named, seeded random substreams.

Same contract as the reference's ``bipush.rng.substream`` (pkg/src/bipush/rng.py:16-26):
one integer seed plus a tuple of tokens selects an independent numpy Generator,
tokens are identified by ``str()``, and each token is folded in as the first
four little-endian bytes of its sha256 digest.  Keeping the contract identical
means the bench draws exactly the source nodes the reference's ``cmd_bench``
would draw (cli.py:415-417) for the same seed.
"""

from __future__ import annotations

import hashlib

import numpy as np


def _token_key(token) -> int:
    digest = hashlib.sha256(str(token).encode("utf-8")).digest()
    return int.from_bytes(digest[:4], "little")


def child_sequence(seed: int, *tokens) -> np.random.SeedSequence:
    return np.random.SeedSequence(entropy=int(seed), spawn_key=tuple(_token_key(t) for t in tokens))


def substream(seed: int, *tokens) -> np.random.Generator:
    """Independent generator for (seed, *tokens)."""
    return np.random.default_rng(child_sequence(seed, *tokens))
