"""Shared fixtures for the parity tests (mirrors proj/tests/helpers.hpp:10-51
in spirit: synthetic scenes + oracle configs on identical inputs)."""
from __future__ import annotations

import numpy as np

import paper_2308_09209_b200 as pb


def scene(views=2, width=160, height=120, frames=4, seed=1, overlap=0.3, casts=None,
          flicker=None, obj=True, focal_scale=1.0, rig="auto"):
    spec = pb.SynthSpec(seed=seed, views=views, frames=frames, width=width, height=height,
                        overlap_fraction=overlap, perturb_focal_scale=focal_scale, rig=rig)
    if casts:
        spec.color_casts = list(casts)
    if flicker:
        spec.flicker = list(flicker)
    if obj:
        spec.object = pb.ParallaxObject(enabled=True, half_size=25.0, velocity=(3.0, 1.0))
    return pb.SynthScene(spec)


def oracle_config(sc: pb.SynthScene, *, threads=4, keep_debug=1, window=3, weighting=0,
                  topology=0, levels=4, iterations=50, smoothness=15.0, lam=0.05,
                  gamma_dark=1.5, gamma_bright=1.5, target_black=0, target_white=255,
                  refine=False, seed=0):
    import oracle as O

    c = sc.config_c()
    cams = [(c.cams[v].fx, c.cams[v].fy, c.cams[v].cx, c.cams[v].cy, list(c.cams[v].rotation),
             list(c.cams[v].translation)) for v in range(c.n_views)]
    sizes = [(c.width[v], c.height[v]) for v in range(c.n_views)]
    return O.make_config(c.n_views, c.reference, sizes, cams, lam=lam, gamma_dark=gamma_dark,
                         gamma_bright=gamma_bright, target_black=target_black,
                         target_white=target_white, levels=levels, iterations=iterations,
                         smoothness=smoothness, window=window, weighting=weighting,
                         topology=topology if topology else c.topology, threads=threads,
                         keep_debug=keep_debug, projection=c.projection,
                         cyl_focal=c.cyl_focal, refine=refine, seed=seed)


def product_config(sc: pb.SynthScene, *, window=3, weighting=0, topology=0, levels=4,
                   iterations=50, smoothness=15.0, lam=0.05, gamma_dark=1.5, gamma_bright=1.5,
                   target_black=0, target_white=255, refine=False, seed=0) -> pb.StitchConfig:
    cfg = sc.config()
    cfg.refine.enabled = refine
    cfg.seed = seed
    cfg.window_capacity = window
    cfg.fuse_weighting = "cross" if weighting else "own"
    if topology:
        cfg.topology = {1: "star", 2: "chain", 3: "ring"}[topology]
    cfg.flow = pb.FlowOptions(levels=levels, iterations=iterations, smoothness=smoothness)
    cfg.balance = pb.BalanceConfig(lam, gamma_dark, gamma_bright, target_black, target_white)
    return cfg


def frames_at(sc: pb.SynthScene, t: int):
    return [sc.render_view(v, t) for v in range(sc.spec.views)]


def maxdiff(a, b) -> int:
    return int(np.abs(a.astype(np.int32) - b.astype(np.int32)).max()) if a.size else 0
