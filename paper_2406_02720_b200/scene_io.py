"""Scene point files <-> device scenes (drop-in for scene_io.py:1-269's scene part).

Same names, argument meaning, file formats and errors as the reference:
`save_scene` / `load_scene` (native double-precision PLY, bit-exact round trip),
`import_3dgs` (standard 3D-GS files; splitting normals seeded from a numpy
Generator exactly as the reference draws them) and `export_3dgs` (alpha-collapsed
float32 3D-GS layout).  Header text is parsed and written here on the host; the
vertex payload crosses PCIe in one contiguous copy and is (de)interleaved on the
GPU by `hs_ply_unpack` / `hs_ply_pack` (csrc/hs_io.cu).  Scenes are
`paper_2406_02720_b200.geometry.Scene` (device tensors, float64 by default like
the reference's).
"""

import ctypes
import re

import numpy as np
import torch

from . import _native, device
from .errors import MalformedHeader, MissingProperty, TruncatedPayload
from .geometry import Scene

_PLY_TYPES = {  # scene_io.py:38-43
    "float": ("<f4", 4, 0), "float32": ("<f4", 4, 0),
    "double": ("<f8", 8, 1), "float64": ("<f8", 8, 1),
    "uchar": ("<u1", 1, 2), "uint8": ("<u1", 1, 2),
    "int": ("<i4", 4, 3), "int32": ("<i4", 4, 3),
}
_SH_DEGREE_BY_REST = {0: 0, 3: 1, 8: 2, 15: 3}  # scene_io.py:46
_NATIVE_REQUIRED = ["x", "y", "z", "nx", "ny", "nz", "f_dc_0", "f_dc_1", "f_dc_2", "opacity",
                    "opacity_2", "scale_0", "scale_1", "scale_2", "rot_0", "rot_1", "rot_2",
                    "rot_3"]
_3DGS_REQUIRED = ["x", "y", "z", "f_dc_0", "f_dc_1", "f_dc_2", "opacity", "scale_0", "scale_1",
                  "scale_2", "rot_0", "rot_1", "rot_2", "rot_3"]


def _read_ply_header(fh):
    """scene_io.py:49-88 (same checks, same messages)."""
    magic = fh.readline()
    if magic.strip() != b"ply":
        raise MalformedHeader("not a PLY file")
    fmt = fh.readline().split()
    if len(fmt) < 2 or fmt[0] != b"format" or fmt[1] != b"binary_little_endian":
        raise MalformedHeader("expected format binary_little_endian")
    count = None
    props = []
    comments = {}
    while True:
        line = fh.readline()
        if not line:
            raise MalformedHeader("unterminated header")
        tokens = line.split()
        if not tokens:
            continue
        if tokens[0] == b"end_header":
            break
        if tokens[0] == b"comment":
            parts = line.decode("ascii", "replace").split(None, 2)
            if len(parts) == 3:
                comments[parts[1]] = parts[2].strip()
            continue
        if tokens[0] == b"element":
            if tokens[1] != b"vertex":
                raise MalformedHeader(f"unsupported element {tokens[1].decode()}")
            count = int(tokens[2])
            continue
        if tokens[0] == b"property":
            if tokens[1] == b"list":
                raise MalformedHeader("list properties are not supported")
            tname = tokens[1].decode()
            if tname not in _PLY_TYPES:
                raise MalformedHeader(f"unsupported property type {tname}")
            props.append((tokens[2].decode(), tname))
            continue
        raise MalformedHeader(f"unexpected header line {line.decode(errors='replace').strip()!r}")
    if count is None:
        raise MalformedHeader("missing vertex element")
    return count, props, comments


def _read_ply(path):
    """Header on the host; the payload as one uint8 array (scene_io.py:91-102)."""
    with open(path, "rb") as fh:
        count, props, comments = _read_ply_header(fh)
        body = fh.read()
    stride = sum(_PLY_TYPES[t][1] for _, t in props)
    if len(body) < count * stride:
        raise TruncatedPayload(f"expected {count * stride} payload bytes, found {len(body)}")
    if len(props) > 128:
        raise MalformedHeader("more than 128 properties")
    payload = np.frombuffer(body, dtype=np.uint8, count=count * stride)
    return count, props, comments, payload, stride


def _require(columns, names):
    for name in names:
        if name not in columns:
            raise MissingProperty(f"point file is missing property {name!r}")


def _rest_names(columns):
    rest = sorted(
        (int(m.group(1)) for m in (re.fullmatch(r"f_rest_(\d+)", c) for c in columns) if m))
    if rest != list(range(len(rest))):
        raise MissingProperty("f_rest_* properties are not contiguous")
    return [f"f_rest_{i}" for i in rest]


def _degree(rest_names):
    n_rest = len(rest_names)
    if n_rest % 3 != 0 or n_rest // 3 not in _SH_DEGREE_BY_REST:
        raise MalformedHeader(f"unsupported f_rest count {n_rest}")
    return _SH_DEGREE_BY_REST[n_rest // 3]


def _layout(count, props, stride, degree, names):
    """hs_ply_layout: property offsets / types and each scene component's source."""
    lay = _native.HsPlyLayout()
    lay.n, lay.stride, lay.n_props, lay.sh_degree = count, stride, len(props), degree
    index = {}
    off = 0
    for p, (name, t) in enumerate(props):
        lay.offset[p] = off
        lay.type[p] = _PLY_TYPES[t][2]
        index[name] = p
        off += _PLY_TYPES[t][1]
    k = (degree + 1) ** 2
    comps = (names["mu"] + names["log_scale"] + names["rotation"]
             + [("f_dc_%d" % ch) if kk == 0 else "f_rest_%d" % (ch * (k - 1) + kk - 1)
                for kk in range(k) for ch in range(3)]
             + names["normal"] + [names["ra"], names["rb"]])
    for c, name in enumerate(comps):
        lay.column[c] = index[name] if name is not None else -1
    return lay


def _empty_scene(n, degree, background, dev, dtype):
    def alloc(*shape):
        return torch.empty(shape, dtype=dtype, device=dev)

    k = (degree + 1) ** 2
    return Scene(alloc(n, 3), alloc(n, 3), alloc(n, 4), alloc(n, k, 3), alloc(n, 3), alloc(n),
                 alloc(n), sh_degree=degree, background_color=background, device=dev,
                 dtype=dtype, validate=False)


def _unpack(payload, lay, scene):
    dev_payload = torch.from_numpy(payload.copy()).to(scene.device)  # one H2D copy
    st = device.scene_struct(scene)
    _native.check(_native.load().hs_ply_unpack(ctypes.c_void_p(dev_payload.data_ptr()),
                                               ctypes.byref(lay), ctypes.byref(st),
                                               device._stream()), "hs_ply_unpack")


def load_scene(path, device_name="cuda", dtype=torch.float64):
    """Read a native point file into a device Scene (scene_io.py:171-197)."""
    count, props, comments, payload, stride = _read_ply(path)
    columns = dict(props)
    _require(columns, _NATIVE_REQUIRED)
    rest = _rest_names(columns)
    degree = _degree(rest)
    if "sh_degree" in comments and int(comments["sh_degree"]) != degree:
        raise MalformedHeader("sh_degree comment disagrees with f_rest count")
    background = (0.0, 0.0, 0.0)
    if "background" in comments:
        background = tuple(float(v) for v in comments["background"].split())
    scene = _empty_scene(count, degree, background, device_name, dtype)
    lay = _layout(count, props, stride, degree, dict(
        mu=["x", "y", "z"], log_scale=["scale_0", "scale_1", "scale_2"],
        rotation=[f"rot_{i}" for i in range(4)], normal=["nx", "ny", "nz"], ra="opacity",
        rb="opacity_2"))
    _unpack(payload, lay, scene)
    scene._validate()
    return scene


def import_3dgs(path, normal_init="zero_plus_jitter", seed=0, background_color=(0, 0, 0),
                device_name="cuda", dtype=torch.float64):
    """A standard 3D-GS point file as half-Gaussian pairs (scene_io.py:200-239):
    both halves inherit the opacity logit; splitting normals are drawn on the
    host from default_rng(seed) exactly as the reference draws them."""
    if normal_init not in ("zero_plus_jitter", "random_unit"):
        raise ValueError(f"unknown normal_init {normal_init!r}")
    count, props, _, payload, stride = _read_ply(path)
    columns = dict(props)
    _require(columns, _3DGS_REQUIRED)
    degree = _degree(_rest_names(columns))
    rng = np.random.default_rng(seed)
    if normal_init == "zero_plus_jitter":
        normals = rng.normal(scale=0.01, size=(count, 3))
    else:
        normals = rng.normal(size=(count, 3))
    norms = np.linalg.norm(normals, axis=1, keepdims=True)
    norms[norms == 0.0] = 1.0
    normals = normals / norms
    scene = _empty_scene(count, degree, np.asarray(background_color, dtype=np.float64),
                         device_name, dtype)
    scene.normal.copy_(torch.as_tensor(normals))
    lay = _layout(count, props, stride, degree, dict(
        mu=["x", "y", "z"], log_scale=["scale_0", "scale_1", "scale_2"],
        rotation=[f"rot_{i}" for i in range(4)], normal=[None, None, None], ra="opacity",
        rb="opacity"))
    _unpack(payload, lay, scene)
    scene._validate()
    return scene


def _pack(scene, kind):
    scene = Scene.from_any(scene)
    lib = _native.load()
    row = lib.hs_ply_row_bytes(scene.sh_degree, kind)
    out = torch.empty(len(scene) * row, dtype=torch.uint8, device=scene.device)
    st = device.scene_struct(scene)
    _native.check(lib.hs_ply_pack(ctypes.byref(st), ctypes.c_void_p(out.data_ptr()), kind,
                                  device._stream()), "hs_ply_pack")
    return scene, out.cpu().numpy()  # one D2H copy


def save_scene(scene, path):
    """Write a scene as a double-precision point file (scene_io.py:136-168)."""
    scene, payload = _pack(scene, 0)
    n, k = len(scene), (scene.sh_degree + 1) ** 2
    names = (["x", "y", "z", "nx", "ny", "nz", "f_dc_0", "f_dc_1", "f_dc_2"]
             + [f"f_rest_{i}" for i in range(3 * (k - 1))]
             + ["opacity", "opacity_2", "scale_0", "scale_1", "scale_2",
                "rot_0", "rot_1", "rot_2", "rot_3"])
    header = ["ply", "format binary_little_endian 1.0", f"comment sh_degree {scene.sh_degree}",
              "comment background " + " ".join(repr(float(v)) for v in scene.background_color),
              f"element vertex {n}"]
    header.extend(f"property double {name}" for name in names)
    header.append("end_header")
    with open(path, "wb") as fh:
        fh.write(("\n".join(header) + "\n").encode("ascii"))
        fh.write(payload.tobytes())


def export_3dgs(scene, path, opacity="mean"):
    """Write the alpha-collapsed scene in the float32 3D-GS layout (scene_io.py:242-269)."""
    if opacity not in ("mean", "first"):
        raise ValueError(f"unknown opacity mode {opacity!r}")
    scene, payload = _pack(scene, 1 if opacity == "mean" else 2)
    n, k = len(scene), (scene.sh_degree + 1) ** 2
    names = (["x", "y", "z", "nx", "ny", "nz", "f_dc_0", "f_dc_1", "f_dc_2"]
             + [f"f_rest_{i}" for i in range(3 * (k - 1))]
             + ["opacity", "scale_0", "scale_1", "scale_2", "rot_0", "rot_1", "rot_2", "rot_3"])
    header = ["ply", "format binary_little_endian 1.0", f"element vertex {n}"]
    header.extend(f"property float {name}" for name in names)
    header.append("end_header")
    with open(path, "wb") as fh:
        fh.write(("\n".join(header) + "\n").encode("ascii"))
        fh.write(payload.tobytes())
