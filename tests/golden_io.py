"""Reader for tests/golden/*.txt fixtures (sections A, B, C of whitespace numbers)."""
import os

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def load(name):
    secs, cur = {}, None
    with open(os.path.join(GOLDEN, name)) as f:
        for line in f:
            line = line.split("#", 1)[0].strip()
            if not line:
                continue
            if line.isalpha():
                cur = line
                secs[cur] = []
            else:
                secs[cur].append([float(x) for x in line.split()])
    return {k: np.array(v, dtype=np.float32) for k, v in secs.items()}
