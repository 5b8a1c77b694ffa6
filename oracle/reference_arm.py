"""The reference's own CPU path, for bench.py's baseline only (test
infrastructure: never imported by the package).  Loads `halfsplat` from
oracle/_ref (oracle/build_ref.py) with its Cython blend core and runs
prepare -> render -> render_backward (rasterizer.py:159-421) on a canonical
scene, with HALFSPLAT_THREADS threads for the tile loops."""
import os
import sys
import time

HERE = os.path.dirname(os.path.abspath(__file__))
REF = os.path.join(HERE, "_ref")


def available():
    return os.path.isdir(os.path.join(REF, "halfsplat"))


def _import():
    if REF not in sys.path:
        sys.path.insert(0, REF)
    import halfsplat.backend as backend
    backend.set_backend("cython")
    from halfsplat import geometry, rasterizer
    return geometry, rasterizer


def iteration(sa, cam_kw, d_color, backward=True, threads=None):
    """One reference iteration on a canonical scene (scenes.SceneArrays, float64);
    returns the seconds it took."""
    geometry, rasterizer = _import()
    s64 = sa.as_float64()
    scene = geometry.Scene(**{f: getattr(s64, f) for f in s64.FIELDS},
                           sh_degree=s64.sh_degree, background_color=s64.background_color)
    cam = geometry.CameraModel(**cam_kw)
    threads = threads or os.cpu_count() or 1
    t0 = time.perf_counter()
    out = rasterizer.render(scene, cam, threads=threads)
    if backward:
        rasterizer.render_backward(scene, cam, out, d_color, threads=threads)
    return time.perf_counter() - t0
