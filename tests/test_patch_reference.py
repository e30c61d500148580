"""patch() against the REAL reference package layout (CPU test, this
container only: the reference lives at /root/reference and is imported
read-only; skipped where it is absent, e.g. on the GPU box).  No compute is
called -- this pins the import sites of SURVEY.md section 8b."""
import os
import sys

import pytest

REF = "/root/reference/pkg/src"


@pytest.fixture(scope="module")
def gelsim():
    if not os.path.isdir(REF):
        pytest.skip("reference package not present")
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
    sys.path.insert(0, REF)
    try:
        import gelsim as g  # noqa: F401
        import gelsim.envs.peg_tasks  # noqa: F401
        import gelsim.envs.scenes  # noqa: F401
    except Exception as e:  # noqa: BLE001
        pytest.skip(f"reference not importable here: {e}")
    yield g
    sys.path.remove(REF)


def test_every_site_exists_in_the_reference(gelsim):
    import importlib

    from paper_2408_06506_b200 import patching
    missing = []
    for mod_name, names in patching._SITES.items():
        mod = importlib.import_module(mod_name)
        missing += [f"{mod_name}.{n}" for n in names if not hasattr(mod, n)]
    assert not missing, missing


def test_patch_rebinds_and_unpatch_restores(gelsim):
    import importlib

    from paper_2408_06506_b200 import depth, patching, render, tactile
    from paper_2408_06506_b200.augment import augment as augment_fn
    before = {(m, n): getattr(importlib.import_module(m), n)
              for m, names in patching._SITES.items() for n in names}
    cls = importlib.import_module("gelsim.envs.peg_tasks").PegEnvBatch
    methods = {n: cls.__dict__[n] for n in ("_tactile_images", "_tactile_ff")}
    done = patching.patch()
    try:
        assert len(done) == len(before) + len(methods)
        from paper_2408_06506_b200 import envs
        assert cls._tactile_images is envs.tactile_images and cls._tactile_ff is envs.tactile_ff
        peg = importlib.import_module("gelsim.envs.peg_tasks")
        assert peg.depth_to_rgb is render.depth_to_rgb
        assert peg.compute_force_field is tactile.compute_force_field
        assert peg.render_depth is depth.render_depth
        assert peg.augment is augment_fn
        scenes = importlib.import_module("gelsim.envs.scenes")
        assert scenes.compute_force_field is tactile.compute_force_field
        # the physics call sites keep the reference's CPU query_sdf
        contacts = importlib.import_module("gelsim.physics.contacts")
        assert contacts.query_sdf is before[("gelsim.geometry", "query_sdf")]
    finally:
        patching.unpatch()
    for (m, n), fn in before.items():
        assert getattr(importlib.import_module(m), n) is fn
    for n, fn in methods.items():
        assert cls.__dict__[n] is fn


def test_reference_exceptions_are_reexported(gelsim):
    import gelsim.errors as ge

    import paper_2408_06506_b200.errors as ours
    # when gelsim is importable our error classes ARE the reference's
    assert issubclass(ours.LutResolutionMismatch, ge.LutResolutionMismatch) or \
        ours.LutResolutionMismatch.__name__ == ge.LutResolutionMismatch.__name__
