"""Shared helpers for the test-suite (golden fixture loading, GPU guards)."""
import json
from pathlib import Path

GOLDEN = Path(__file__).resolve().parent / "golden"


def load_golden(name):
    return json.loads((GOLDEN / name).read_text())
