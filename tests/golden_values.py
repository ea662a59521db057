"""Loader for tests/golden/ (values printed in the paper, each file carries its citation)."""
import json
import os

HERE = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def load(name: str) -> dict:
    with open(os.path.join(HERE, name)) as f:
        return json.load(f)


def table5(quantizer: str) -> float:
    """Mean distortion of Table 5 for 'tcq-2.0', 'nuq-2.0' or 'vq-2.0'."""
    return load("table5_distortion.json")["quantizers"][quantizer]["mean"]
