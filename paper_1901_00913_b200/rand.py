"""Named Philox substreams (restates kronblur rand.py:18-36).

The power-iteration start vector of ``estimate_lipschitz`` (solvers.py:115) and the noise of
``add_noise`` (imaging.py:153) come from ``stream(seed, tag)``; reproducing the stream bit for bit
is what lets the GPU path start from the reference's exact vectors.
"""

from __future__ import annotations

import numpy as np

from .errors import ArgumentError

TAGS = {"image": 1, "noise": 2, "shake": 3, "lipschitz": 4}


def stream(seed: int, tag: str, index: int = 0) -> np.random.Generator:
    """Generator for substream ``tag`` of ``seed`` (SeedSequence spawn key (tag id, index))."""
    try:
        tag_id = TAGS[tag]
    except KeyError:
        raise ArgumentError(f"unknown random stream tag {tag!r}") from None
    seq = np.random.SeedSequence(entropy=int(seed), spawn_key=(tag_id, int(index)))
    return np.random.Generator(np.random.Philox(seq))
