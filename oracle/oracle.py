"""TEST INFRASTRUCTURE ONLY -- ctypes loaders for the two CPU checkers.

* ``liborc``  : the C restatement of the reference hot path
  (oracle/fusechain_oracle.c, cites /root/reference/proj/src/simulator.cpp).
* ``libref``  : the reference's own sources compiled unmodified
  (oracle/_ref/libfuseplan_ref.so, built by oracle/Makefile).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
reference legs may import this module.  The product package
(paper_1509_04394_b200) never does.
"""
from __future__ import annotations

import ctypes
import json
import os
import subprocess
from typing import Optional, Sequence

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORC_SO = os.path.join(HERE, "_build", "liborc.so")
REF_SO = os.path.join(HERE, "_ref", "libfuseplan_ref.so")

# Op codes (fusechain_oracle.h)
OPS = {
    "rgba2gray": 0,
    "iir_temporal": 1,
    "gaussian": 2,
    "gradient": 3,
    "threshold": 4,
    "identity": 5,
    "scale_offset": 6,
    "box_mean": 7,
    "kalman_track": 8,
}

# Parameter defaults of apply_stencil_at (simulator.cpp:51-106)
DEFAULTS = {
    "rgba2gray": [("wr", 0.299), ("wg", 0.587), ("wb", 0.114)],
    "iir_temporal": [("alpha", 0.5)],
    "gaussian": [("radius", 2), ("sigma", 1.0)],
    "gradient": [],
    "threshold": [("th", 128.0), ("white", 255.0), ("black", 0.0)],
    "identity": [],
    "scale_offset": [("scale", 1.0), ("offset", 0.0)],
    "box_mean": [("radius_x", 1), ("radius_y", 1), ("radius_t", 0)],
    "kalman_track": [],
}


class OrcStage(ctypes.Structure):
    _fields_ = [("op", ctypes.c_int), ("p", ctypes.c_double * 4)]


def build(force: bool = False) -> None:
    """Build liborc (always possible) and _ref (only where /root/reference exists)."""
    targets = ["_build/liborc.so"]
    if os.path.isdir("/root/reference/proj"):
        targets.append("ref")
    if force or not os.path.exists(ORC_SO) or (
            len(targets) > 1 and not os.path.exists(REF_SO)):
        subprocess.run(["make", "-s", "-C", HERE] + targets, check=True)


_orc = None
_ref = None


def orc_lib():
    global _orc
    if _orc is None:
        if not os.path.exists(ORC_SO):
            build()
        lib = ctypes.CDLL(ORC_SO)
        lib.orc_gaussian_weights.argtypes = [ctypes.c_int, ctypes.c_double,
                                             ctypes.c_void_p]
        lib.orc_apply_stage.argtypes = [ctypes.POINTER(OrcStage), ctypes.c_void_p,
                                        ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                        ctypes.c_int, ctypes.c_void_p, ctypes.c_int]
        for fn in (lib.orc_chain_stream_u8, lib.orc_chain_stream_f32):
            fn.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                           ctypes.c_int, ctypes.POINTER(OrcStage), ctypes.c_int,
                           ctypes.c_int, ctypes.c_int, ctypes.c_void_p,
                           ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int]
        _orc = lib
    return _orc


def ref_available() -> bool:
    return os.path.exists(REF_SO)


def ref_lib():
    global _ref
    if _ref is None:
        if not os.path.exists(REF_SO):
            build()
        lib = ctypes.CDLL(REF_SO)
        c_p, c_i, c_s = ctypes.c_void_p, ctypes.c_int, ctypes.c_char_p
        lib.ref_plan_json.argtypes = [c_s, c_s, c_s, c_p, c_i, c_p, c_i]
        lib.ref_run_sequential.argtypes = [c_s, c_p, c_i, c_p, c_p, c_p, c_i]
        lib.ref_run_sequential_strips.argtypes = [c_s, c_p, c_i, c_p, c_i, c_p, c_i]
        lib.ref_run_tiled.argtypes = [c_s, c_s, c_s, c_p, c_i, c_p, c_p, c_p, c_i]
        lib.ref_synth_u8.argtypes = [c_s, c_p, c_p, c_i]
        lib.ref_codegen_manifest.argtypes = [c_s, c_s, c_s, c_s, c_p, c_i, c_p, c_i]
        _ref = lib
    return _ref


class RefError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"[{code}] {msg}")
        self.code = code


def _check(rc: int, err) -> None:
    if rc != 0:
        raise RefError(rc, err.value.decode(errors="replace"))


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


# ---------------------------------------------------------------- reference


def ref_plan_json(pipeline_json: str, device_json: str,
                  options: Optional[dict] = None) -> str:
    lib = ref_lib()
    err = ctypes.create_string_buffer(1024)
    cap = 1 << 20
    out = ctypes.create_string_buffer(cap)
    opts = json.dumps(options).encode() if options else b""
    rc = lib.ref_plan_json(pipeline_json.encode(), device_json.encode(), opts,
                           out, cap, err, 1024)
    _check(rc, err)
    return out.value.decode()


def ref_codegen_manifest(pipeline_json: str, device_json: str,
                         options: Optional[dict], name: str) -> dict:
    """The reference codegen's manifest (codegen.cpp:425-465) as a dict."""
    lib = ref_lib()
    err = ctypes.create_string_buffer(1024)
    cap = 1 << 20
    out = ctypes.create_string_buffer(cap)
    opts = json.dumps(options).encode() if options else b""
    rc = lib.ref_codegen_manifest(pipeline_json.encode(), device_json.encode(), opts,
                                  name.encode(), out, cap, err, 1024)
    _check(rc, err)
    return json.loads(out.value.decode())


def _pipe_dims(pipeline_json: str):
    v = json.loads(pipeline_json)["video"]
    return v["width"], v["height"], v["frames"], v.get("channels", 1)


def ref_run_sequential(pipeline_json: str, video: np.ndarray, stages: bool = False):
    """Returns (final [F,H,W] float32, stage outputs [n,F,H,W] or None)."""
    lib = ref_lib()
    W, H, F, C = _pipe_dims(pipeline_json)
    is_u8 = int(video.dtype == np.uint8)
    video = np.ascontiguousarray(video, dtype=np.uint8 if is_u8 else np.float32)
    final = np.empty((F, H, W), np.float32)
    n_exec = sum(1 for k in json.loads(pipeline_json)["kernels"]
                 if k["stencil_op"] != "kalman_track")
    st = np.empty((n_exec, F, H, W), np.float32) if stages else None
    err = ctypes.create_string_buffer(1024)
    rc = lib.ref_run_sequential(pipeline_json.encode(), _ptr(video), is_u8,
                                _ptr(final), _ptr(st) if stages else None, err, 1024)
    _check(rc, err)
    return final, st


def ref_run_sequential_strips(pipeline_json: str, video: np.ndarray,
                              nthreads: int) -> np.ndarray:
    lib = ref_lib()
    W, H, F, C = _pipe_dims(pipeline_json)
    is_u8 = int(video.dtype == np.uint8)
    video = np.ascontiguousarray(video)
    final = np.empty((F, H, W), np.float32)
    err = ctypes.create_string_buffer(1024)
    rc = lib.ref_run_sequential_strips(pipeline_json.encode(), _ptr(video), is_u8,
                                       _ptr(final), int(nthreads), err, 1024)
    _check(rc, err)
    return final


def ref_run_tiled(pipeline_json: str, device_json: str, video: np.ndarray,
                  options: Optional[dict] = None):
    lib = ref_lib()
    W, H, F, C = _pipe_dims(pipeline_json)
    is_u8 = int(video.dtype == np.uint8)
    video = np.ascontiguousarray(video)
    final = np.empty((F, H, W), np.float32)
    traffic = np.zeros(4, np.int64)
    err = ctypes.create_string_buffer(1024)
    opts = json.dumps(options).encode() if options else b""
    rc = lib.ref_run_tiled(pipeline_json.encode(), device_json.encode(), opts,
                           _ptr(video), is_u8, _ptr(final), _ptr(traffic), err, 1024)
    _check(rc, err)
    return final, traffic


def ref_synth_u8(spec: dict) -> np.ndarray:
    """synth_video + FPVD u8 round trip -> planar [F, C, H, W] uint8."""
    lib = ref_lib()
    F, C, H, W = (spec.get("frames", 32), spec.get("channels", 4),
                  spec.get("height", 64), spec.get("width", 64))
    out = np.empty((F, C, H, W), np.uint8)
    err = ctypes.create_string_buffer(1024)
    rc = lib.ref_synth_u8(json.dumps(spec).encode(), _ptr(out), err, 1024)
    _check(rc, err)
    return out


# ---------------------------------------------------------------- restatement


def stage_of(kernel: dict) -> OrcStage:
    op = kernel["stencil_op"]
    params = kernel.get("params", {})
    st = OrcStage()
    st.op = OPS[op]
    for i, (k, d) in enumerate(DEFAULTS[op]):
        st.p[i] = float(params.get(k, d))
    return st


def stages_of(pipeline: dict):
    ks = pipeline["kernels"]
    arr = (OrcStage * len(ks))()
    for i, k in enumerate(ks):
        arr[i] = stage_of(k)
    return arr, len(ks)


def gaussian_weights(radius: int, sigma: float) -> np.ndarray:
    d = 2 * radius + 1
    out = np.empty(d * d, np.float32)
    orc_lib().orc_gaussian_weights(radius, sigma, _ptr(out))
    return out.reshape(d, d)


def orc_chain(pipeline: dict, video: np.ndarray, t_begin: int = 0, t_out: int = 0,
              state_in: Optional[np.ndarray] = None, nthreads: int = 0,
              return_state: bool = False):
    """Streaming restatement of run_sequential.  video: planar [F, C, H, W]."""
    lib = orc_lib()
    F, C, H, W = video.shape
    arr, n = stages_of(pipeline)
    n_iir = sum(1 for k in pipeline["kernels"] if k["stencil_op"] == "iir_temporal")
    out = np.empty((F - t_out, H, W), np.float32)
    st_out = np.empty((max(n_iir, 1), H, W), np.float32)
    if nthreads <= 0:
        nthreads = os.cpu_count() or 1
    fn = lib.orc_chain_stream_u8 if video.dtype == np.uint8 else lib.orc_chain_stream_f32
    video = np.ascontiguousarray(video)
    sin = None
    if state_in is not None:
        state_in = np.ascontiguousarray(state_in, np.float32)
        sin = _ptr(state_in)
    rc = fn(_ptr(video), W, H, F, C, arr, n, t_begin, t_out, _ptr(out), sin,
            _ptr(st_out), nthreads)
    if rc != 0:
        raise ValueError("orc_chain: unsupported chain")
    return (out, st_out) if return_state else out


def orc_apply_stage(kernel: dict, vol: np.ndarray, nthreads: int = 0) -> np.ndarray:
    """apply_stencil on a planar [F, C, H, W] float volume -> [F, H, W]."""
    lib = orc_lib()
    F, C, H, W = vol.shape
    st = stage_of(kernel)
    out = np.empty((F, H, W), np.float32)
    vol = np.ascontiguousarray(vol, np.float32)
    rc = lib.orc_apply_stage(ctypes.byref(st), _ptr(vol), W, H, F, C, _ptr(out),
                             nthreads or (os.cpu_count() or 1))
    if rc != 0:
        raise ValueError("orc_apply_stage: unsupported")
    return out


def orc_run_sequential(pipeline: dict, video: np.ndarray, nthreads: int = 0):
    """Whole-volume stage-by-stage restatement; returns list of stage outputs."""
    cur = video.astype(np.float32)
    outs = []
    for k in pipeline["kernels"]:
        if k["stencil_op"] == "kalman_track":
            continue
        o = orc_apply_stage(k, cur, nthreads)
        outs.append(o)
        cur = o[:, None]
    return outs
