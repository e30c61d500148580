"""Rebind the reference's hot-path names to the B200 implementations.

The reference binds names at import time (``from ..render.lut import
depth_to_rgb`` etc.), so every importing module must be rebound, not just
the defining one:

    gelsim.render, gelsim.render.lut          depth_to_rgb
    gelsim.render, gelsim.render.imageio      to_uint8
    gelsim.tactile, gelsim.tactile.field      compute_force_field, penalty_forces, net_wrench
    gelsim.envs.peg_tasks, gelsim.envs.scenes depth_to_rgb, compute_force_field
    gelsim.geometry, gelsim.geometry.sdf      query_sdf, relative_penetration_rate (standalone API only)

and replaces ``PegEnvBatch._tactile_images`` / ``_tactile_ff``
(envs/peg_tasks.py:434-477) by their batched versions in ``envs.py``.

``query_sdf`` is deliberately NOT rebound at the physics call sites
(physics/contacts.py:15, envs/peg_tasks.py _fit_grip): those are tiny CPU
queries where a device round trip would only add latency; inside
``compute_force_field`` the query is fused into K2 anyway.
"""
from __future__ import annotations

import importlib

_SITES = {
    "gelsim.render": ("depth_to_rgb", "to_uint8", "render_depth", "augment"),
    "gelsim.render.augment": ("augment",),
    "gelsim.render.lut": ("depth_to_rgb",),
    "gelsim.render.imageio": ("to_uint8",),
    "gelsim.render.depth": ("render_depth",),
    "gelsim.tactile": ("compute_force_field", "penalty_forces", "net_wrench"),
    "gelsim.tactile.field": ("compute_force_field", "penalty_forces", "net_wrench"),
    "gelsim.envs.peg_tasks": ("depth_to_rgb", "compute_force_field", "render_depth", "augment"),
    "gelsim.envs.scenes": ("depth_to_rgb", "compute_force_field", "render_depth"),
    "gelsim.envs.wrist": ("render_depth",),
    "gelsim.geometry": ("query_sdf", "relative_penetration_rate"),
}

# env methods replaced by their batched versions (envs.py): one launch per
# kernel for both fingers of all envs instead of per-finger / per-env loops
_METHODS = {
    ("gelsim.envs.peg_tasks", "PegEnvBatch"): ("_tactile_images", "_tactile_ff"),
}

_saved: dict = {}


def _impl(name):
    from . import depth, geometry, render, tactile
    from .augment import augment as augment_fn

    return {
        "augment": augment_fn,
        "render_depth": depth.render_depth,
        "depth_to_rgb": render.depth_to_rgb,
        "to_uint8": render.to_uint8,
        "compute_force_field": tactile.compute_force_field,
        "penalty_forces": tactile.penalty_forces,
        "net_wrench": tactile.net_wrench,
        "query_sdf": geometry.query_sdf,
        "relative_penetration_rate": geometry.relative_penetration_rate,
    }[name]


def _method_impl(name):
    from . import envs

    return {"_tactile_images": envs.tactile_images, "_tactile_ff": envs.tactile_ff}[name]


def patch(modules=None, env_methods: bool = True) -> list:
    """Rebind the hot-path names in every importable reference module (and,
    with ``env_methods``, the env's tactile observation methods).  Returns the
    list of (module, name) pairs rebound."""
    done = []
    if env_methods:
        for (mod_name, cls_name), names in _METHODS.items():
            if modules is not None and mod_name not in modules:
                continue
            try:
                cls = getattr(importlib.import_module(mod_name), cls_name)
            except Exception:  # noqa: BLE001 - module absent in this install
                continue
            for n in names:
                if n in cls.__dict__:
                    _saved.setdefault((mod_name, f"{cls_name}.{n}"), cls.__dict__[n])
                    setattr(cls, n, _method_impl(n))
                    done.append((mod_name, f"{cls_name}.{n}"))
    for mod_name, names in _SITES.items():
        if modules is not None and mod_name not in modules:
            continue
        try:
            mod = importlib.import_module(mod_name)
        except Exception:  # noqa: BLE001 - module absent in this install
            continue
        for n in names:
            if hasattr(mod, n):
                _saved.setdefault((mod_name, n), getattr(mod, n))
                setattr(mod, n, _impl(n))
                done.append((mod_name, n))
    return done


def unpatch() -> None:
    for (mod_name, n), fn in list(_saved.items()):
        target = importlib.import_module(mod_name)
        if "." in n:  # Class.method
            cls_name, n = n.split(".", 1)
            target = getattr(target, cls_name)
        setattr(target, n, fn)
    _saved.clear()
