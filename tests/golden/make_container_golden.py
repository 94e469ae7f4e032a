"""Golden NMCS containers written by the REAL reference (container.py) for the export/import tests.

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_container_golden.py

Scores are exact small multiples of 2^-6 drawn with many ties, so fp32 GPU scores equal the
float64 ones and the selected nonzeros / nibbles must match byte for byte.
"""

from __future__ import annotations

import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))


def main() -> None:
    from nmattn import DenseMatrix, SparsityMode, compress_logical, to_bytes

    rng = np.random.default_rng(2203)
    out = {}
    for name, mode, shape in (("12", SparsityMode.ONE_OF_TWO, (24, 40)), ("24", SparsityMode.TWO_OF_FOUR, (33, 64))):
        scores = rng.integers(-40, 40, size=shape).astype(np.float64) / 64.0
        raw = to_bytes(compress_logical(DenseMatrix(scores), mode))
        out[f"scores_{name}"] = scores
        out[f"nmcs_{name}"] = np.frombuffer(raw, dtype=np.uint8)
    np.savez_compressed(os.path.join(HERE, "container.npz"), **out)
    print({k: v.shape for k, v in out.items()})


if __name__ == "__main__":
    main()
