"""Label vectors (mirror of the reference labeling.py).

Same names and validation as /root/reference/pkg/src/gee/labeling.py, with
int32 storage (the kernels read int32 labels and narrow them to u8/u16).
Text label files are outside the hot path and are
not mirrored.
"""

from dataclasses import dataclass

import numpy as np

from .errors import ValidationError
from .graph import _is_torch


@dataclass(eq=False)
class LabelVector:
    """Per-node class labels in {0, ..., k}; 0 means class unknown
    (labeling.py:10-30)."""

    labels: object
    k: int

    def __post_init__(self):
        self.k = int(self.k)
        if self.k < 1:
            raise ValidationError("class count k must be positive")
        if _is_torch(self.labels):
            import torch

            lab = self.labels.reshape(-1)
            if lab.numel():
                bad = torch.nonzero((lab < 0) | (lab > self.k))
                if bad.numel():
                    i = int(bad[0, 0])
                    raise ValidationError(f"label {int(lab[i])} at node {i} outside [0, {self.k}]")
            self.labels = lab.to(torch.int32).contiguous()
            return
        lab = np.asarray(self.labels).reshape(-1)
        if lab.size:
            bad = np.nonzero((lab < 0) | (lab > self.k))[0]
            if bad.size:
                raise ValidationError(f"label {lab[bad[0]]} at node {bad[0]} outside [0, {self.k}]")
        self.labels = np.ascontiguousarray(lab, dtype=np.int32)

    @property
    def n(self) -> int:
        return int(self.labels.shape[0])


def random_labels(n, k, fraction, seed) -> LabelVector:
    """Label exactly round(fraction * n) distinct nodes uniformly at random.

    Same algorithm and numpy stream as labeling.py:87-104 (default_rng(seed),
    choice without replacement, then integers in {1..k}), so a seed gives
    the reference's vector.
    """
    if n < 1:
        raise ValidationError("n must be at least 1")
    if k < 1:
        raise ValidationError("k must be at least 1")
    if not 0.0 <= fraction <= 1.0:
        raise ValidationError("fraction must lie in [0, 1]")
    m = int(round(fraction * n))
    rng = np.random.default_rng(seed)
    labels = np.zeros(n, dtype=np.int64)
    chosen = rng.choice(n, size=m, replace=False)
    labels[chosen] = rng.integers(1, k + 1, size=m, dtype=np.int64)
    return LabelVector(labels=labels, k=k)


def class_counts(y: LabelVector) -> np.ndarray:
    """Members per class (labeling.py:107-109): entry c-1 counts nodes
    labeled c; computed by the K1 histogram kernel, bit-exact."""
    from .encoder import _counts_on_device

    return _counts_on_device(y)[1:]
