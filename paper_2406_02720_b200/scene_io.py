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


class _Header:
    """What the header of a point file declares: the vertex count, the properties in
    payload order as (name, type), the `comment key value` pairs, and the offset of
    the first payload byte."""

    def __init__(self):
        self.count = None
        self.props = []
        self.comments = {}
        self.payload_offset = 0

    @property
    def stride(self):
        return sum(_PLY_TYPES[t][1] for _, t in self.props)


def _header_lines(blob):
    """Yields (line, end) for each newline-terminated line at the start of `blob`;
    `end` is the offset just past the line."""
    pos = 0
    while pos < len(blob):
        nl = blob.find(b"\n", pos)
        end = len(blob) if nl < 0 else nl + 1
        yield blob[pos:end], end
        pos = end


def _on_comment(h, words, line):
    key_value = line.decode("ascii", "replace").split(None, 2)[1:]
    if len(key_value) == 2:
        h.comments[key_value[0]] = key_value[1].strip()


def _on_element(h, words, line):
    if words[1] != b"vertex":
        raise MalformedHeader(f"unsupported element {words[1].decode()}")
    h.count = int(words[2])


def _on_property(h, words, line):
    if words[1] == b"list":
        raise MalformedHeader("list properties are not supported")
    type_name = words[1].decode()
    if type_name not in _PLY_TYPES:
        raise MalformedHeader(f"unsupported property type {type_name}")
    h.props.append((words[2].decode(), type_name))


_HEADER_KEYWORDS = {b"comment": _on_comment, b"element": _on_element, b"property": _on_property}


def _parse_header(blob):
    """The header grammar of scene_io.py:49-88 with the reference's exception types
    and messages: `ply`, `format binary_little_endian ...`, then comment / element
    vertex / scalar property lines up to `end_header`."""
    lines = _header_lines(blob)
    magic, _ = next(lines, (b"", 0))
    if magic.strip() != b"ply":
        raise MalformedHeader("not a PLY file")
    fmt, _ = next(lines, (b"", 0))
    if fmt.split()[:2] != [b"format", b"binary_little_endian"]:
        raise MalformedHeader("expected format binary_little_endian")
    h = _Header()
    for line, end in lines:
        words = line.split()
        if not words:
            continue
        if words[0] == b"end_header":
            h.payload_offset = end
            break
        handler = _HEADER_KEYWORDS.get(words[0])
        if handler is None:
            shown = line.decode(errors="replace").strip()
            raise MalformedHeader(f"unexpected header line {shown!r}")
        handler(h, words, line)
    else:
        raise MalformedHeader("unterminated header")
    if h.count is None:
        raise MalformedHeader("missing vertex element")
    return h


def _read_ply(path):
    """The header parsed on the host; the payload as one uint8 view of the file
    (scene_io.py:91-102), which crosses PCIe in one copy."""
    with open(path, "rb") as fh:
        blob = fh.read()
    h = _parse_header(blob)
    need = h.count * h.stride
    have = len(blob) - h.payload_offset
    if have < need:
        raise TruncatedPayload(f"expected {need} payload bytes, found {have}")
    if len(h.props) > 128:
        raise MalformedHeader("more than 128 properties")
    payload = np.frombuffer(blob, dtype=np.uint8, count=need, offset=h.payload_offset)
    return h.count, h.props, h.comments, payload, h.stride


def _require(columns, names):
    """MissingProperty for the first required name the file lacks (in `names` order)."""
    missing = [name for name in names if name not in columns]
    if missing:
        raise MissingProperty(f"point file is missing property {missing[0]!r}")


def _rest_names(columns):
    """The f_rest_<i> properties, which must be numbered 0..R-1 without gaps."""
    idx = sorted(int(c[len("f_rest_"):]) for c in columns
                 if c.startswith("f_rest_") and c[len("f_rest_"):].isdigit())
    if idx and (idx[0] != 0 or idx[-1] != len(idx) - 1 or len(set(idx)) != len(idx)):
        raise MissingProperty("f_rest_* properties are not contiguous")
    return [f"f_rest_{i}" for i in idx]


def _degree(rest_names):
    per_channel, ragged = divmod(len(rest_names), 3)
    degree = _SH_DEGREE_BY_REST.get(per_channel)
    if ragged or degree is None:
        raise MalformedHeader(f"unsupported f_rest count {len(rest_names)}")
    return degree


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
    declared = comments.get("sh_degree")
    if declared is not None and int(declared) != degree:
        raise MalformedHeader("sh_degree comment disagrees with f_rest count")
    background = tuple(map(float, comments.get("background", "0 0 0").split()))
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
