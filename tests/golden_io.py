"""Helpers to read the golden fixtures written by tests/golden/make_golden.py."""

import json
import os

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def load(name):
    z = np.load(os.path.join(GOLDEN, name))
    index = json.loads(bytes(z["index"]).decode())
    return z, index
