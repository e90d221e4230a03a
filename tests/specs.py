"""Scene specs (plain dicts, see tests/golden/make_golden.py) -> product types."""

from __future__ import annotations

import numpy as np

import paper_1609_01317_b200 as vc


def product_volume(arr: np.ndarray, spacing) -> vc.Volume:
    return vc.Volume.from_array(arr, spacing=spacing, dtype=arr.dtype)


def product_scene(spec: dict) -> vc.Scene:
    cam = spec["camera"]
    camera = vc.Camera(eye=tuple(cam["eye"]), target=tuple(cam["target"]),
                       up=tuple(cam.get("up", (0.0, 1.0, 0.0))), fov_y=cam.get("fov_y", 60.0),
                       azimuth=cam.get("azimuth", 0.0), elevation=cam.get("elevation", 0.0),
                       zoom=cam.get("zoom", 1.0))
    light = vc.Light(position=tuple(spec["light"]["position"]),
                     color=tuple(spec["light"].get("color", (1.0, 1.0, 1.0))))
    win = spec.get("window", (500.0, 4095.0))
    tf = spec.get("transfer")
    transfer = vc.TransferFunction.default_ct() if tf is None else vc.TransferFunction(
        points=[(p[0], tuple(p[1])) for p in tf["points"]], mu_water=tf.get("mu_water", 1000.0))
    clip = spec.get("clip")
    return vc.Scene(camera=camera, light=light, window=vc.ThresholdWindow(*win), transfer=transfer,
                    clip=None if clip is None else vc.ClipBox(tuple(clip[0]), tuple(clip[1])))


def product_settings(spec: dict, **over) -> vc.RenderSettings:
    s = dict(spec.get("settings", {}))
    kw = {}
    for key in ("width", "height", "coarse_step", "fine_step", "refine_iters", "mode"):
        if key in s:
            kw[key] = s[key]
    if "operator" in s:
        kw["operator"] = vc.OperatorKind(s["operator"])
    if "interpolation" in s:
        kw["interpolation"] = vc.InterpolationMode(s["interpolation"])
    if "background" in s:
        kw["background"] = tuple(s["background"])
    for key in ("use_adaptive", "adaptive_factor", "detail_epsilon", "octree_min_block",
                "octree_max_depth", "use_octree"):
        if key in s:
            kw[key] = s[key]
    kw.update(over)
    return vc.RenderSettings(**kw)


def spec_of(scene_settings) -> dict:
    """Product (Scene, RenderSettings) -> spec dict for the oracle."""
    sc, st = scene_settings
    cam = sc.camera
    return {
        "camera": {"eye": list(cam.eye), "target": list(cam.target), "up": list(cam.up),
                   "fov_y": cam.fov_y, "azimuth": cam.azimuth, "elevation": cam.elevation,
                   "zoom": cam.zoom},
        "light": {"position": list(sc.light.position), "color": list(sc.light.color)},
        "window": [sc.window.low, sc.window.high],
        "transfer": {"points": [[p[0], list(p[1])] for p in sc.transfer.points],
                     "mu_water": sc.transfer.mu_water},
        "clip": None if sc.clip is None else [list(sc.clip.lo), list(sc.clip.hi)],
        "settings": {"width": st.width, "height": st.height, "operator": st.operator.value,
                     "interpolation": st.interpolation.value, "mode": st.mode,
                     "coarse_step": st.coarse_step, "fine_step": st.fine_step,
                     "refine_iters": st.refine_iters, "background": list(st.background),
                     "use_adaptive": st.use_adaptive, "adaptive_factor": st.adaptive_factor,
                     "detail_epsilon": st.detail_epsilon, "octree_min_block": st.octree_min_block,
                     "octree_max_depth": st.octree_max_depth, "use_octree": st.use_octree},
    }
