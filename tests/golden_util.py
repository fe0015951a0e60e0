"""Loader for tests/golden/* (written by tests/golden/make_goldens.py from the reference)."""
import gzip
import json
import os

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def load(name):
    p = os.path.join(GOLDEN, name + ".json")
    if os.path.exists(p):
        with open(p) as f:
            return json.load(f)
    with gzip.open(p + ".gz", "rt") as f:
        return json.load(f)


class Tensors:
    def __init__(self, name):
        doc = load(name)
        self.result = doc["result"]
        self.index = doc.get("tensors", {})
        self.path = os.path.join(GOLDEN, name + ".bin")

    def __contains__(self, key):
        return key in self.index

    def __getitem__(self, key):
        e = self.index[key]
        dt = np.float32 if e["dtype"] == "f32" else np.float64
        a = np.fromfile(self.path, dtype=dt, count=e["count"], offset=e["offset"])
        return a.reshape(e["shape"])


def demo_path(*parts):
    return os.path.join(GOLDEN, "demo", *parts)
