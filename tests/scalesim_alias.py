"""pytest plugin: make ``import scalesim`` resolve to ``paper_2412_17246_b200``.

Used by tests/test_reference_suite.py to run the reference's tests on our package.
"""

import importlib
import sys

_SUBMODULES = ("topology", "parampool", "planner", "livescale", "autoscaler", "traces", "presets")


def _alias():
    pkg = importlib.import_module("paper_2412_17246_b200")
    sys.modules["scalesim"] = pkg
    for name in _SUBMODULES:
        sys.modules[f"scalesim.{name}"] = importlib.import_module(f"paper_2412_17246_b200.{name}")


_alias()


def pytest_configure(config):  # noqa: D401 - pytest hook
    _alias()
