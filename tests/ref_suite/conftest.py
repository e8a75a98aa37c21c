"""Runs the reference package's own test suite (pkg/tests, 170 tests) against
this package on the GPU.

The suite files live in tests/ref_suite/_ref/ (fetched by fetch.py in the
build container; git-ignored, they travel to the GPU box with the
snapshot).  Before they are collected, `blockmend` and its submodules are
aliased to this package's modules, so every `from blockmend import ...` in
the suite binds the B200 implementation.  Two aliases carry test-only
shims: `blockmend.corpus` is the reference's synthetic test-image
generator (test data), and `blockmend.netpbm._parse_pnm_header` adapts
netpbm.parse_header to the private 4-tuple the CLI tests read PPMs with.

Every collected test is marked `gpu`.  Known deviations are listed in
KNOWN with the reason; they run as xfail(strict=False) so a pass is seen.
"""

import importlib.util
import os
import sys
import types

import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
REF = os.path.join(HERE, "_ref")

# test id suffix -> reason the B200 path legitimately differs
KNOWN: dict = {}


def _install_alias():
    if "blockmend" in sys.modules and getattr(sys.modules["blockmend"], "__b200_alias__", False):
        return
    import paper_2205_11226_b200 as pkg
    from paper_2205_11226_b200 import cli, errors, estimators, framework, image, loss, metrics, netpbm, profiles

    root = types.ModuleType("blockmend")
    root.__dict__.update({k: v for k, v in pkg.__dict__.items() if not k.startswith("__")})
    root.__path__ = []
    root.__b200_alias__ = True
    sys.modules["blockmend"] = root
    for name, mod in (("cli", cli), ("errors", errors), ("estimators", estimators), ("framework", framework),
                      ("image", image), ("loss", loss), ("metrics", metrics), ("profiles", profiles)):
        sys.modules[f"blockmend.{name}"] = mod
        setattr(root, name, mod)
    shim = types.ModuleType("blockmend.netpbm")
    shim.__dict__.update(netpbm.__dict__)

    def _parse_pnm_header(data, magic):
        h = netpbm.parse_header(data, magic)
        return h.width, h.height, h.maxval, h.raster_offset

    shim._parse_pnm_header = _parse_pnm_header
    sys.modules["blockmend.netpbm"] = shim
    root.netpbm = shim
    spec = importlib.util.spec_from_file_location("blockmend.corpus", os.path.join(REF, "ref_corpus.py"))
    corpus = importlib.util.module_from_spec(spec)
    corpus.__package__ = "blockmend"
    sys.modules["blockmend.corpus"] = corpus
    spec.loader.exec_module(corpus)
    root.corpus = corpus


if os.path.exists(os.path.join(REF, "ref_corpus.py")):
    _install_alias()


def pytest_collection_modifyitems(config, items):
    for item in items:
        if not str(item.fspath).startswith(REF):
            continue
        item.add_marker(pytest.mark.gpu)
        for key, why in KNOWN.items():
            if item.nodeid.endswith(key):
                item.add_marker(pytest.mark.xfail(reason=why, strict=False))
