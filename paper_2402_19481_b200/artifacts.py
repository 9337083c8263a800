"""Run artifacts of the reference (proj/src/io.cpp), byte-compatible, on the host.

* TNSR tensors (io.cpp:47-88): magic "TNSR", version byte 1, ndim u32 LE (= 4), the four dims
  u32 LE, then the float32 payload little-endian row-major; round trips are bit-exact and the
  reader rejects bad magic / version / rank, short payloads and non-finite values with the
  reference's messages.
* PGM previews (io.cpp:90-108): P5, channel pages stacked vertically, min-max normalised over
  [lo, hi], round half up, a zero range writes mid-gray.
* psnr (tensor.cpp:336-347) and the flattened weight pool (dump_weights / load_weights,
  io.cpp:133-160) so the B200 runner can run on weights exchanged with the reference.

These are host-side file formats (no GPU work); the sampling itself runs on the B200 runner
(`patchsim.PatchRunner`)."""
from __future__ import annotations

import math
import re
import struct

import numpy as np

from . import patchsim as P


def write_tnsr(x, path: str) -> None:
    """write_tnsr (io.cpp:47-64)."""
    a = np.ascontiguousarray(x, dtype=np.float32)
    if a.ndim != 4:
        raise P.InvalidArgument("write_tnsr: expected an NCHW tensor")
    with open(path, "wb") as f:
        f.write(b"TNSR")
        f.write(bytes([1]))
        f.write(struct.pack("<5I", 4, *a.shape))
        f.write(a.astype("<f4", copy=False).tobytes())


def read_tnsr(path: str) -> np.ndarray:
    """read_tnsr (io.cpp:66-88), same checks and messages."""
    try:
        f = open(path, "rb")
    except OSError:
        raise P.RuntimeFailure(f"read_tnsr: cannot open {path}") from None
    with f:
        blob = f.read()
    if blob[:4] != b"TNSR":
        raise P.RuntimeFailure(f"read_tnsr: bad magic in {path}")
    if len(blob) < 5 or blob[4] != 1:
        raise P.RuntimeFailure(f"read_tnsr: unsupported version in {path}")
    if len(blob) < 9 or struct.unpack_from("<I", blob, 5)[0] != 4:
        raise P.RuntimeFailure(f"read_tnsr: expected 4 dims in {path}")
    if len(blob) < 25:
        raise P.RuntimeFailure(f"read_tnsr: payload shorter than dims in {path}")
    dims = struct.unpack_from("<4I", blob, 9)
    count = int(np.prod(dims, dtype=np.int64))
    if len(blob) < 25 + 4 * count:
        raise P.RuntimeFailure(f"read_tnsr: payload shorter than dims in {path}")
    out = np.frombuffer(blob, dtype="<f4", count=count, offset=25).astype(np.float32).reshape(dims)
    if not np.all(np.isfinite(out)):
        raise P.RuntimeFailure("read_tnsr: non-finite value in tensor")
    return out


def write_pgm(x, path: str, lo: float, hi: float) -> None:
    """write_pgm (io.cpp:90-108)."""
    a = np.asarray(x, dtype=np.float32)
    n, c, h, w = a.shape
    rng = float(hi) - float(lo)
    if rng > 0.0:
        t = (a.astype(np.float64) - float(lo)) / rng
        t = np.clip(t, 0.0, 1.0)
        px = np.floor(t * 255.0 + 0.5).astype(np.uint8)
    else:
        px = np.full(a.shape, 128, dtype=np.uint8)
    with open(path, "wb") as f:
        f.write(f"P5\n{w} {n * c * h}\n255\n".encode())
        f.write(px.reshape(-1).tobytes())


def _shape_str(shape):
    """Tensor::shape_str (tensor.cpp:30-34): '(1,4,8,8)'."""
    return "(" + ",".join(str(int(v)) for v in shape) + ")"


def psnr(a, b, peak: float) -> float:
    """psnr (tensor.cpp:336-347): 10 log10(peak^2 / mse), +inf when identical."""
    a = np.asarray(a, dtype=np.float32)
    b = np.asarray(b, dtype=np.float32)
    if a.shape != b.shape:
        raise P.InvalidArgument(f"psnr: shape mismatch {_shape_str(a.shape)} vs "
                                f"{_shape_str(b.shape)}")
    if not peak > 0.0:
        raise P.InvalidArgument("psnr: peak must be positive")
    se = float(np.sum((a.astype(np.float64) - b.astype(np.float64)) ** 2))
    if se == 0.0:
        return math.inf
    return 10.0 * math.log10(peak * peak / (se / a.size))


def dump_weights(model: "P.Model", path: str) -> None:
    """dump_weights (io.cpp:133-143): the pool flattened into one (1, 1, 1, total) TNSR."""
    pool = np.concatenate([w.reshape(-1) for w in model.weights()])
    write_tnsr(pool.reshape(1, 1, 1, -1), path)


def load_weights(cfg: "P.ModelConfig", path: str) -> "P.Model":
    """load_weights (io.cpp:145-160): a model of `cfg` on the file's pool; the element count
    must match ("load_weights: file holds X values, model expects Y")."""
    flat = read_tnsr(path).reshape(-1)
    try:
        return P.Model.from_pool(cfg, [flat])
    except P.InvalidArgument as e:
        m = re.search(r"has (\d+) floats, model expects (\d+)", str(e))
        if not m:
            raise
        raise P.InvalidArgument(f"load_weights: file holds {m.group(1)} values, model expects "
                                f"{m.group(2)}") from None


def similarity_report(trajectory):
    """input_similarity_report (proj/src/sampler.cpp:97-127): per consecutive pair of step
    inputs the mean |x_t - x_{t-1}| (fp64), their mean, the observed range over every state,
    and ratio = mean / range (0 when the range is 0).  trajectory: [steps, ...] array."""
    traj = np.asarray(trajectory)
    if traj.shape[0] == 0:
        return {"per_step_mean_abs_diff": [], "mean_abs_diff": 0.0, "range_min": 0.0,
                "range_max": 0.0, "ratio": 0.0}
    lo = float(np.min(traj).astype(np.float64))
    hi = float(np.max(traj).astype(np.float64))
    per = [float(np.mean(np.abs(traj[i].astype(np.float64) - traj[i - 1].astype(np.float64))))
           for i in range(1, traj.shape[0])]
    mean = float(np.mean(per)) if per else 0.0
    rng = hi - lo
    return {"per_step_mean_abs_diff": per, "mean_abs_diff": mean, "range_min": lo,
            "range_max": hi, "ratio": mean / rng if rng > 0.0 else 0.0}


COST_KEYS = ("compute_rate", "link_bandwidth", "link_latency", "comm_uses_compute_fraction")


def parse_cost_profile(path: str) -> dict:
    """parse_cost_profile (proj/src/io.cpp:110-131) + CostParams::validate
    (proj/src/costmodel.cpp:13-19): 'key = value' lines, '#' comments, unknown keys and bad
    values are InvalidArgument."""
    p = {"compute_rate": 1000.0, "link_bandwidth": 100.0, "link_latency": 5.0,
         "comm_uses_compute_fraction": 0.15}
    try:
        f = open(path)
    except OSError:
        raise P.InvalidArgument(f"cost profile: cannot open {path}") from None
    with f:
        for line in f:
            t = line.strip()
            if not t or t.startswith("#"):
                continue
            if "=" not in t:
                raise P.InvalidArgument(f"cost profile: expected 'key = value', got '{t}'")
            k, v = (s.strip() for s in t.split("=", 1))
            if k not in COST_KEYS:
                raise P.InvalidArgument(f"cost profile: unknown key '{k}'")
            try:
                p[k] = float(v)
            except ValueError:
                raise P.InvalidArgument(f"cost profile: bad value '{v}'") from None
    if p["compute_rate"] <= 0.0 or p["link_bandwidth"] <= 0.0:
        raise P.InvalidArgument("CostParams: rates must be positive")
    if p["link_latency"] < 0.0:
        raise P.InvalidArgument("CostParams: negative latency")
    if not (0.0 <= p["comm_uses_compute_fraction"] < 1.0):
        raise P.InvalidArgument("CostParams: comm_uses_compute_fraction must be in [0,1)")
    return p
