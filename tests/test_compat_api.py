"""The drop-in API mirrors the reference's signatures (CPU check, no GPU needed).

When the reference package is importable (the build container), every compat function
must accept the same parameter names in the same order as the headsplat function it
replaces; otherwise the test checks the names against the list recorded here.
"""
import inspect
import os
import sys

import pytest

from paper_2503_12886_b200 import compat

EXPECTED = {
    "map_params": ("model", ["mlp", "theta"]),
    "mlp_backward": ("model", ["mlp", "cache", "grad_psi"]),
    "blend": ("model", ["model", "psi"]),
    "blend_backward": ("model", ["model", "psi", "grad_out"]),
    "activate": ("model", ["raw"]),
    "activate_backward": ("model", ["raw", "activated", "grad_out"]),
    "transform_to_deformed": ("binding", ["tangent", "frames", "bindings"]),
    "transform_backward": ("binding", ["tangent", "frames", "bindings", "grad_world"]),
    "preprocess": ("render", ["world", "camera"]),
    "rasterize": ("render", ["splats", "camera", "background"]),
    "render_backward": ("render", ["splats", "aux", "grad_image"]),
    "splat_weight_sums": ("render", ["aux", "image"]),
    "estimate_colors": ("color_init", ["aux", "target", "threshold"]),
    "apply_color_init": ("color_init", ["model", "estimates", "eligible", "state"]),
    "render_batch": ("scheduler", ["items", "workers", "scheme"]),
    "train_step": ("train", ["state", "samples", "backgrounds", "mesh_of"]),
}


def _ref_module(name):
    ref = "/root/reference/pkg/src"
    if not os.path.isdir(ref):
        return None
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
    if ref not in sys.path:
        sys.path.append(ref)
    try:
        import importlib
        return importlib.import_module(f"headsplat.{name}")
    except Exception:
        return None


@pytest.mark.parametrize("fn", sorted(EXPECTED))
def test_signature_matches_reference(fn):
    mod, names = EXPECTED[fn]
    ours = list(inspect.signature(getattr(compat, fn)).parameters)
    assert ours == names
    ref = _ref_module(mod)
    if ref is not None:
        theirs = list(inspect.signature(getattr(ref, fn)).parameters)
        assert ours == theirs, (fn, ours, theirs)


def test_batch_renderer_interface():
    r = compat.BatchRenderer(workers=4, scheme="naive")
    assert r.barrier_count == 0 and hasattr(r, "render_batch") and hasattr(r, "map_items")
    assert r.map_items(lambda a, b: a + b, [(1, 2), (3, 4)]) == [3, 7]
    with pytest.raises(ValueError):
        compat.BatchRenderer(scheme="bogus")
    with pytest.raises(ValueError):
        r.render_batch([])
