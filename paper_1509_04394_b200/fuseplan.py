"""Python binding of the fuseplan C ABI (include/fuseplan.h) -- the
reference-facing surface of this build, loaded from the in-tree
libfuseplan_b200.so.

Mirrors the reference's handles and status taxonomy
(/root/reference/proj/include/fuseplan.h:14-93): ``Pipeline`` / ``Device`` /
``Plan`` wrap the opaque handles, failures raise ``FuseplanError`` subclasses
carrying the fp_status code (Input -> 2, Infeasible -> 1, Internal -> 3) and
the thread-local fp_last_error() text.  ``Executor`` is the new device
executor (fp_exec_*): it takes torch CUDA tensors (zero-copy, asynchronous on
the current torch stream) or host numpy / torch CPU arrays (streamed through
the device, synchronous).

There is no CPU execution path: without the .so or without a CUDA device the
executor raises.
"""
from __future__ import annotations

import ctypes
import json
import os
from typing import Optional, Union

import numpy as np

PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("FUSEPLAN_LIB") or os.path.join(PKG, "libfuseplan_b200.so")
DATA_DIR = os.path.join(PKG, "data")

FP_OK, FP_ERR_INFEASIBLE, FP_ERR_INPUT, FP_ERR_INTERNAL = 0, 1, 2, 3
FP_ELEM_U8, FP_ELEM_F32 = 0, 1
FP_EXEC_HOST_PTRS, FP_EXEC_DEVICE_PTRS = 0, 1


class FuseplanError(RuntimeError):
    status = FP_ERR_INTERNAL

    def __init__(self, msg: str):
        super().__init__(msg)


class InfeasibleError(FuseplanError):
    status = FP_ERR_INFEASIBLE


class InputError(FuseplanError):
    status = FP_ERR_INPUT


class InternalError(FuseplanError):
    status = FP_ERR_INTERNAL


_ERRORS = {FP_ERR_INFEASIBLE: InfeasibleError, FP_ERR_INPUT: InputError,
           FP_ERR_INTERNAL: InternalError}

_lib = None


def lib() -> ctypes.CDLL:
    """The loaded C ABI.  Raises if the extension has not been built."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: run `python -m paper_1509_04394_b200.build` "
            "(there is no CPU fallback)")
    L = ctypes.CDLL(LIB_PATH)
    P, I, S, V = ctypes.c_void_p, ctypes.c_int, ctypes.c_char_p, None
    PP = ctypes.POINTER(ctypes.c_void_p)
    PS = ctypes.POINTER(ctypes.c_char_p)
    sig = {
        "fp_last_error": ([], ctypes.c_char_p),
        "fp_string_free": ([P], V),
        "fp_pipeline_parse": ([S, PP], I),
        "fp_pipeline_load": ([S, PP], I),
        "fp_pipeline_free": ([P], V),
        "fp_device_parse": ([S, PP], I),
        "fp_device_load": ([S, PP], I),
        "fp_device_free": ([P], V),
        "fp_plan_create": ([P, P, S, PP], I),
        "fp_plan_free": ([P], V),
        "fp_plan_render_json": ([P, PP], I),
        "fp_analyze_report": ([P, S, I, PP], I),
        "fp_plan_report": ([P, S, I, PP], I),
        "fp_tile_sweep": ([P, ctypes.POINTER(ctypes.c_int), I, I, S, PP], I),
        "fp_codegen": ([P, P, S, S, S, PP], I),
        "fp_simulate": ([P, P, S, S, S, S, S, I, PP], I),
        "fp_calibrate_csv": ([S, PP], I),
        "fp_device_render_with_cost": ([P, S, PP], I),
        "fp_exec_create": ([P, P, I, S, PP], I),
        "fp_exec_free": ([P], V),
        "fp_exec_output_type": ([P, ctypes.POINTER(ctypes.c_int)], I),
        "fp_exec_state_planes": ([P, ctypes.POINTER(ctypes.c_int)], I),
        "fp_exec_run": ([P, P, I, P, I, P], I),
        "fp_exec_run_range": ([P, P, I, P, I, I, P, P, P], I),
        "fp_exec_graph_create": ([P, P, I, P, P, PP], I),
        "fp_exec_graph_launch": ([P, P], I),
        "fp_exec_graph_free": ([P], V),
        "fp_exec_describe": ([P, PP], I),
        "fp_certified_params": ([P, PP], I),
        "fp_exec_run_file": ([P, S, S], I),
        "fp_synth_hash_u8": ([P, I, I, I, I, I, ctypes.c_uint64, P], I),
        "fp_exec_converge": ([P, P, I, I, P, P, ctypes.POINTER(ctypes.c_int), P], I),
        "fp_shard_exec_create": ([P, P, ctypes.POINTER(ctypes.c_int), I, S, PP], I),
        "fp_shard_exec_free": ([P], V),
        "fp_shard_exec_run": ([P, P, I, P], I),
        "fp_shard_exec_stats": ([P, PP], I),
        "fp_track_features": ([P, I, I, I, I, I, ctypes.POINTER(ctypes.c_int), I, S,
                               ctypes.POINTER(ctypes.c_double), PP, P], I),
    }
    for name, (args, res) in sig.items():
        fn = getattr(L, name)
        fn.argtypes = args
        fn.restype = res
    _lib = L
    return L


def _check(status: int) -> None:
    if status != FP_OK:
        msg = lib().fp_last_error().decode(errors="replace")
        raise _ERRORS.get(status, InternalError)(msg)


def _take_string(ptr: ctypes.c_void_p) -> str:
    s = ctypes.cast(ptr, ctypes.c_char_p).value.decode()
    lib().fp_string_free(ptr)
    return s


def _enc(s: Optional[str]):
    return None if s is None else s.encode()


def _opts(options: Union[None, str, dict]) -> Optional[bytes]:
    if options is None:
        return None
    return (options if isinstance(options, str) else json.dumps(options)).encode()


class _Handle:
    _free = ""

    def __init__(self, ptr):
        self._ptr = ptr

    def __del__(self):
        p = getattr(self, "_ptr", None)
        if p and _lib is not None:
            getattr(_lib, self._free)(p)
            self._ptr = None

    @property
    def ptr(self):
        return self._ptr


class Pipeline(_Handle):
    """fp_pipeline: a validated kernel chain (parse_pipeline, config.cpp:98-159)."""
    _free = "fp_pipeline_free"

    def __init__(self, json_text: str):
        out = ctypes.c_void_p()
        _check(lib().fp_pipeline_parse(json_text.encode(), ctypes.byref(out)))
        super().__init__(out)
        self.json = json_text
        self.spec = json.loads(json_text)

    @classmethod
    def load(cls, path: str) -> "Pipeline":
        with open(path) as fh:
            return cls(fh.read())

    @property
    def dims(self):
        v = self.spec["video"]
        return v["width"], v["height"], v["frames"], v.get("channels", 1)

    def analyze(self, fmt: str = "text", timestamp: bool = False) -> str:
        out = ctypes.c_void_p()
        _check(lib().fp_analyze_report(self.ptr, fmt.encode(), int(timestamp),
                                       ctypes.byref(out)))
        return _take_string(out)


    def certified_params(self) -> dict:
        """Certification parameters of the all-fused SPEC chain (host only):
        {g0, g1, mlo_n, band_n, S, mstar} (fp_certified_params)."""
        out = ctypes.c_void_p()
        _check(lib().fp_certified_params(self.ptr, ctypes.byref(out)))
        return json.loads(_take_string(out))


class Device(_Handle):
    """fp_device: a device profile (parse_device, config.cpp:161-190)."""
    _free = "fp_device_free"

    def __init__(self, json_text: str):
        out = ctypes.c_void_p()
        _check(lib().fp_device_parse(json_text.encode(), ctypes.byref(out)))
        super().__init__(out)
        self.json = json_text

    @classmethod
    def load(cls, path_or_name: str) -> "Device":
        path = path_or_name
        if not os.path.exists(path):
            bundled = os.path.join(DATA_DIR, path_or_name + ".json")
            if os.path.exists(bundled):
                path = bundled
        with open(path) as fh:
            return cls(fh.read())

    def tile_sweep(self, halo, max_x: int, max_t: int, fmt: str = "csv") -> str:
        arr = (ctypes.c_int * 6)(*halo)
        out = ctypes.c_void_p()
        _check(lib().fp_tile_sweep(self.ptr, arr, max_x, max_t, fmt.encode(),
                                   ctypes.byref(out)))
        return _take_string(out)


class Plan(_Handle):
    """fp_plan: the optimizer's fusion plan (plan(), planner.cpp:342-393)."""
    _free = "fp_plan_free"

    def __init__(self, pipeline: Pipeline, device: Device,
                 options: Union[None, str, dict] = None):
        out = ctypes.c_void_p()
        _check(lib().fp_plan_create(pipeline.ptr, device.ptr, _opts(options),
                                    ctypes.byref(out)))
        super().__init__(out)
        self.pipeline = pipeline

    def render_json(self) -> str:
        out = ctypes.c_void_p()
        _check(lib().fp_plan_render_json(self.ptr, ctypes.byref(out)))
        return _take_string(out)

    def report(self, fmt: str = "text", timestamp: bool = False) -> str:
        out = ctypes.c_void_p()
        _check(lib().fp_plan_report(self.ptr, fmt.encode(), int(timestamp),
                                    ctypes.byref(out)))
        return _take_string(out)

    @property
    def partition(self):
        return [(g["interval"]["first"], g["interval"]["last"])
                for g in json.loads(self.render_json())["groups"]]


def simulate(pipeline: Pipeline, device: Device, options=None, video_path=None,
             synth: Union[None, str, dict] = None, fmt: str = "text",
             timestamp: bool = False) -> str:
    out = ctypes.c_void_p()
    _check(lib().fp_simulate(pipeline.ptr, device.ptr, _opts(options),
                             _enc(video_path), _opts(synth), None, fmt.encode(),
                             int(timestamp), ctypes.byref(out)))
    return _take_string(out)


def _torch():
    import torch
    return torch


CUDA_STREAM_LEGACY = 0x1  # cudaStreamLegacy


def _stream_handle(stream) -> int:
    """cudaStream_t of a torch stream.  torch's default stream has handle 0,
    which the C ABI reads as "the executor's own stream"; map it to the legacy
    default stream so work stays ordered with torch's."""
    h = int(stream.cuda_stream) if hasattr(stream, "cuda_stream") else int(stream or 0)
    return h if h != 0 else CUDA_STREAM_LEGACY


class Executor(_Handle):
    """fp_exec: runs a plan's partitions as sm_100a kernels on one GPU."""
    _free = "fp_exec_free"

    def __init__(self, pipeline: Pipeline, plan: Plan, device: int = 0,
                 variant: str = "auto", host_chunk_frames: int = 0):
        out = ctypes.c_void_p()
        opts = json.dumps({"variant": variant, "host_chunk_frames": host_chunk_frames})
        _check(lib().fp_exec_create(pipeline.ptr, plan.ptr, device, opts.encode(),
                                    ctypes.byref(out)))
        super().__init__(out)
        self.pipeline = pipeline
        self.device = device
        t = ctypes.c_int()
        _check(lib().fp_exec_output_type(self.ptr, ctypes.byref(t)))
        self.out_elem = t.value
        _check(lib().fp_exec_state_planes(self.ptr, ctypes.byref(t)))
        self.state_planes = t.value

    def describe(self) -> dict:
        out = ctypes.c_void_p()
        _check(lib().fp_exec_describe(self.ptr, ctypes.byref(out)))
        return json.loads(_take_string(out))

    @property
    def out_dtype(self):
        return np.uint8 if self.out_elem == FP_ELEM_U8 else np.float32

    def _elem(self, dtype) -> int:
        if dtype in (np.uint8,) or str(dtype) in ("torch.uint8", "uint8"):
            return FP_ELEM_U8
        if dtype in (np.float32,) or str(dtype) in ("torch.float32", "float32"):
            return FP_ELEM_F32
        raise InputError(f"video dtype must be uint8 or float32, got {dtype}")

    # -- caller-buffer validation: the C side reads and writes with the
    # pipeline's dims, so a wrong shape / dtype / device here would become an
    # out-of-bounds device write or host heap corruption
    def _check_out(self, out, shape, on_cuda, device=None):
        out_dt = self.out_dtype
        if tuple(out.shape) != tuple(shape):
            raise InputError(f"out shape {tuple(out.shape)} != {tuple(shape)}")
        is_torch = type(out).__module__.startswith("torch")
        if on_cuda:
            if not (is_torch and out.is_cuda):
                raise InputError("out must be a CUDA tensor for a CUDA video")
            if device is not None and out.device != device:
                raise InputError(f"out is on {out.device}, the video on {device}")
            if not out.is_contiguous():
                raise InputError("out must be contiguous")
            want = "torch.uint8" if out_dt is np.uint8 else "torch.float32"
            if str(out.dtype) != want:
                raise InputError(f"out dtype {out.dtype} != {want}")
        else:
            if is_torch:
                if out.is_cuda:
                    raise InputError("out must be a host array for a host video")
                arr = out.numpy()
            else:
                arr = out
            if not isinstance(arr, np.ndarray) or arr.dtype != out_dt:
                raise InputError(f"out must be a {np.dtype(out_dt).name} array")
            if not arr.flags["C_CONTIGUOUS"]:
                raise InputError("out must be C-contiguous")

    def _check_state(self, st, name, device):
        W, H, _, _ = self.pipeline.dims
        n = max(self.state_planes, 1)
        if not (type(st).__module__.startswith("torch") and st.is_cuda):
            raise InputError(f"{name} must be a CUDA tensor")
        if st.device != device:
            raise InputError(f"{name} is on {st.device}, the video on {device}")
        if str(st.dtype) != "torch.float32" or not st.is_contiguous():
            raise InputError(f"{name} must be a contiguous float32 tensor")
        if st.numel() != n * H * W or (st.dim() == 3 and tuple(st.shape) != (n, H, W)):
            raise InputError(f"{name} shape {tuple(st.shape)} != {(n, H, W)}")

    def run(self, video, out=None, stream=None):
        """video: planar [F, C, H, W].  CUDA tensor -> CUDA tensor (async on the
        current torch stream); numpy / CPU tensor -> numpy (synchronous)."""
        W, H, F, C = self.pipeline.dims
        if tuple(video.shape) != (F, C, H, W):
            raise InputError(f"video shape {tuple(video.shape)} != {(F, C, H, W)}")
        self._elem(video.dtype)
        is_torch = type(video).__module__.startswith("torch")
        if is_torch and video.is_cuda:
            torch = _torch()
            video = video.contiguous()
            if out is None:
                out = torch.empty((F, H, W), device=video.device,
                                  dtype=torch.uint8 if self.out_elem == FP_ELEM_U8
                                  else torch.float32)
            else:
                self._check_out(out, (F, H, W), True, video.device)
            stream = _stream_handle(torch.cuda.current_stream(video.device)
                                    if stream is None else stream)
            _check(lib().fp_exec_run(self.ptr, video.data_ptr(), self._elem(video.dtype),
                                     out.data_ptr(), FP_EXEC_DEVICE_PTRS, stream))
            return out
        arr = video.numpy() if is_torch else np.asarray(video)
        arr = np.ascontiguousarray(arr)
        if out is None:
            out = np.empty((F, H, W), self.out_dtype)
        else:
            self._check_out(out, (F, H, W), False)
            if type(out).__module__.startswith("torch"):
                out = out.numpy()
        _check(lib().fp_exec_run(self.ptr, arr.ctypes.data, self._elem(arr.dtype),
                                 out.ctypes.data, FP_EXEC_HOST_PTRS, None))
        return out

    def capture(self, video, out=None, stream=None) -> "Graph":
        """fp_exec_graph_create: a CUDA graph of one whole run on these device
        buffers (runs once uncaptured, then captures).  Refill `video` in place
        and call Graph.launch() to re-run; the result lands in Graph.out."""
        torch = _torch()
        W, H, F, C = self.pipeline.dims
        if not (type(video).__module__.startswith("torch") and video.is_cuda):
            raise InputError("capture needs a CUDA video tensor")
        if tuple(video.shape) != (F, C, H, W) or not video.is_contiguous():
            raise InputError(f"video must be a contiguous {(F, C, H, W)} tensor")
        if out is None:
            out = torch.empty((F, H, W), device=video.device,
                              dtype=torch.uint8 if self.out_elem == FP_ELEM_U8
                              else torch.float32)
        else:
            self._check_out(out, (F, H, W), True, video.device)
        stream = _stream_handle(torch.cuda.current_stream(video.device)
                                if stream is None else stream)
        g = ctypes.c_void_p()
        _check(lib().fp_exec_graph_create(self.ptr, video.data_ptr(), self._elem(video.dtype),
                                          out.data_ptr(), stream, ctypes.byref(g)))
        return Graph(self, g, video, out)

    def converge(self, video, s_true, s_warm, stream=None) -> int:
        """fp_exec_converge: how many leading frames of a shard (CUDA video
        [n, C, H, W]) that ran from s_warm differ from a run from s_true."""
        torch = _torch()
        for st, name in ((s_true, "s_true"), (s_warm, "s_warm")):
            self._check_state(st, name, video.device)
        k = ctypes.c_int()
        stream = _stream_handle(torch.cuda.current_stream(video.device)
                                if stream is None else stream)
        video = video.contiguous()
        _check(lib().fp_exec_converge(self.ptr, video.data_ptr(), self._elem(video.dtype),
                                      int(video.shape[0]), s_true.data_ptr(),
                                      s_warm.data_ptr(), ctypes.byref(k), stream))
        return k.value

    def run_file(self, in_path: str, out_path: str) -> None:
        """FPVD file in -> FPVD file out, streamed through the GPU in chunks
        (fp_exec_run_file); the video never has to fit in host memory."""
        _check(lib().fp_exec_run_file(self.ptr, str(in_path).encode(), str(out_path).encode()))

    def run_range(self, video, n_warm: int = 0, state_in=None, state_out=None,
                  out=None, stream=None):
        """T-shard run on CUDA tensors: video [n, C, H, W] starting at the first
        processed frame; returns [n - n_warm, H, W]."""
        torch = _torch()
        W, H, _, C = self.pipeline.dims
        if not (type(video).__module__.startswith("torch") and video.is_cuda):
            raise InputError("run_range needs a CUDA tensor video")
        if video.dim() != 4 or tuple(video.shape[1:]) != (C, H, W):
            raise InputError(f"video shape {tuple(video.shape)} != (n, {C}, {H}, {W})")
        self._elem(video.dtype)
        n = int(video.shape[0])
        if not 0 <= n_warm <= n:
            raise InputError(f"n_warm {n_warm} outside [0, {n}]")
        video = video.contiguous()
        if out is None:
            out = torch.empty((n - n_warm, H, W), device=video.device,
                              dtype=torch.uint8 if self.out_elem == FP_ELEM_U8
                              else torch.float32)
        else:
            self._check_out(out, (n - n_warm, H, W), True, video.device)
        if state_in is not None:
            self._check_state(state_in, "state_in", video.device)
        if state_out is not None:
            self._check_state(state_out, "state_out", video.device)
        stream = _stream_handle(torch.cuda.current_stream(video.device)
                                if stream is None else stream)
        _check(lib().fp_exec_run_range(
            self.ptr, video.data_ptr(), self._elem(video.dtype), out.data_ptr(), n,
            n_warm, None if state_in is None else state_in.data_ptr(),
            None if state_out is None else state_out.data_ptr(), stream))
        return out


class ShardedExecutor(_Handle):
    """fp_shard_exec: one process drives several GPUs; the video is split along
    T, each shard's IIR restarts `warmup_frames` early, carries move device to
    device and a wrong warm start is repaired by re-running only the frames it
    reaches (exact for any warm-up).  Host numpy buffers in and out."""
    _free = "fp_shard_exec_free"

    def __init__(self, pipeline: Pipeline, plan: Plan, devices, variant: str = "auto",
                 warmup_frames: int = 48):
        out = ctypes.c_void_p()
        devs = (ctypes.c_int * len(devices))(*devices)
        opts = json.dumps({"variant": variant, "warmup_frames": warmup_frames})
        _check(lib().fp_shard_exec_create(pipeline.ptr, plan.ptr, devs, len(devices),
                                          opts.encode(), ctypes.byref(out)))
        super().__init__(out)
        self.pipeline = pipeline
        self._one = Executor(pipeline, plan, device=devices[0], variant=variant)

    def run(self, video, out=None):
        W, H, F, C = self.pipeline.dims
        arr = np.ascontiguousarray(video)
        if arr.shape != (F, C, H, W):
            raise InputError(f"video shape {arr.shape} != {(F, C, H, W)}")
        if out is None:
            out = np.empty((F, H, W), self._one.out_dtype)
        else:
            self._one._check_out(out, (F, H, W), False)
        _check(lib().fp_shard_exec_run(self.ptr, arr.ctypes.data, self._one._elem(arr.dtype),
                                       out.ctypes.data))
        return out

    def stats(self) -> dict:
        out = ctypes.c_void_p()
        _check(lib().fp_shard_exec_stats(self.ptr, ctypes.byref(out)))
        return json.loads(_take_string(out))


def synth_hash_u8(out, t0: int = 0, seed: int = 1234, stream=None):
    """Fill a CUDA uint8 tensor [F, C, H, W] with the counter-hash test video."""
    torch = _torch()
    F, C, H, W = out.shape
    stream = _stream_handle(torch.cuda.current_stream(out.device)
                            if stream is None else stream)
    _check(lib().fp_synth_hash_u8(out.data_ptr(), W, H, F, C, t0, seed, stream))
    return out


def hash_video_u8(frames: int, channels: int, height: int, width: int, seed: int,
                  t0: int = 0) -> np.ndarray:
    """Host copy of the counter-hash video (same values as synth_hash_u8)."""
    t = np.arange(t0, t0 + frames, dtype=np.uint64)[:, None, None, None]
    c = np.arange(channels, dtype=np.uint64)[None, :, None, None]
    y = np.arange(height, dtype=np.uint64)[None, None, :, None]
    x = np.arange(width, dtype=np.uint64)[None, None, None, :]
    with np.errstate(over="ignore"):
        idx = ((t * np.uint64(channels) + c) * np.uint64(height) + y) * np.uint64(width) + x
        z = idx + np.uint64((seed * 0x9E3779B97F4A7C15) & 0xFFFFFFFFFFFFFFFF)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        z = z ^ (z >> np.uint64(31))
    return (z >> np.uint64(56)).astype(np.uint8)


class Graph:
    """A captured run (Executor.capture): launch() replays it on the captured
    video / out buffers, asynchronously on `stream` (default: the current
    torch stream).  Holds the executor and the buffers alive."""

    def __init__(self, ex, handle, video, out):
        self.ex, self.ptr, self.video, self.out = ex, handle, video, out

    def launch(self, stream=None):
        torch = _torch()
        st = _stream_handle(torch.cuda.current_stream(self.video.device)
                            if stream is None else stream)
        _check(lib().fp_exec_graph_launch(self.ptr, st))
        return self.out

    def close(self):
        if getattr(self, "ptr", None):
            lib().fp_exec_graph_free(self.ptr)
            self.ptr = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def spec_chain(width: int, height: int, frames: int, alpha: float = 0.5,
               radius: int = 2, sigma: float = 1.0, th: float = 128.0,
               kalman: bool = False, channels: int = 4) -> dict:
    """The SPEC chain (proj/data/vision_pipeline.json:4-8) at a given size."""
    ks = []
    if channels == 4:
        ks.append({"name": "rgba_to_gray", "stencil_op": "rgba2gray"})
    ks += [{"name": "temporal_denoise", "stencil_op": "iir_temporal",
            "params": {"alpha": alpha}},
           {"name": "gaussian_smooth", "stencil_op": "gaussian",
            "params": {"radius": radius, "sigma": sigma}},
           {"name": "gradient_magnitude", "stencil_op": "gradient"},
           {"name": "binarize", "stencil_op": "threshold", "params": {"th": th}}]
    if kalman:
        ks.append({"name": "kalman_tracking", "stencil_op": "kalman_track"})
    return {"video": {"width": width, "height": height, "frames": frames, "fps": 1,
                      "channels": channels}, "kernels": ks}


TRACK_POINT_FIELDS = ("measured", "meas_x", "meas_y", "est_x", "est_y", "est_vx", "est_vy") + \
    tuple(f"cov{i}{j}" for i in range(4) for j in range(4))


def track_features(mask, rois, q: float = 0.01, r: float = 0.25, p0: float = 10.0,
                   stream=None, csv: bool = True):
    """K6 tracking on the GPU (fp_track_features; tracking.cpp:84-128).

    mask: [F, H, W] uint8 / float32, numpy (host) or a torch CUDA tensor;
    rois: [(x, y, w, h)] initial ROI per marker.  Returns (points, csv):
    points [n, F, 23] float64 (TRACK_POINT_FIELDS), csv the reference's
    trajectory CSV text (None when csv=False)."""
    F, H, W = (int(v) for v in mask.shape)
    rois = np.ascontiguousarray(np.asarray(rois, np.int32).reshape(-1, 4))
    n = rois.shape[0]
    pts = np.zeros((n, F, 23), np.float64)
    out = ctypes.c_void_p()
    kal = json.dumps({"q": q, "r": r, "p0": p0}).encode()
    is_torch = type(mask).__module__.startswith("torch")
    if is_torch and mask.is_cuda:
        torch = _torch()
        mask = mask.contiguous()
        elem = FP_ELEM_U8 if mask.dtype == torch.uint8 else FP_ELEM_F32
        st = _stream_handle(torch.cuda.current_stream(mask.device) if stream is None else stream)
        ptr, on_dev = mask.data_ptr(), 1
    else:
        arr = np.ascontiguousarray(mask.numpy() if is_torch else np.asarray(mask))
        elem = FP_ELEM_U8 if arr.dtype == np.uint8 else FP_ELEM_F32
        if elem == FP_ELEM_F32:
            arr = arr.astype(np.float32, copy=False)
        mask, ptr, on_dev, st = arr, arr.ctypes.data, 0, None
    _check(lib().fp_track_features(
        ptr, elem, on_dev, W, H, F, rois.ctypes.data_as(ctypes.POINTER(ctypes.c_int)), n, kal,
        pts.ctypes.data_as(ctypes.POINTER(ctypes.c_double)),
        ctypes.byref(out) if csv else None, st))
    return pts, (_take_string(out) if csv else None)


def write_fpvd(path: str, video: np.ndarray) -> None:
    """FPVD writer (video.cpp:46-62): planar [F, C, H, W] (or [F, H, W]) u8/f32."""
    import struct
    v = np.asarray(video)
    if v.ndim == 3:
        v = v[:, None]
    F, C, H, W = v.shape
    et = 0 if v.dtype == np.uint8 else 1
    with open(path, "wb") as fh:
        fh.write(b"FPVD" + struct.pack("<6I", 1, W, H, F, C, et))
        fh.write(np.ascontiguousarray(v if et == 0 else v.astype(np.float32)).tobytes())


def read_fpvd(path: str) -> np.ndarray:
    """FPVD reader (video.cpp:64-94) -> planar [F, C, H, W] u8 / f32."""
    import struct
    with open(path, "rb") as fh:
        hdr = fh.read(28)
        if hdr[:4] != b"FPVD":
            raise InputError("not an FPVD video file")
        ver, W, H, F, C, et = struct.unpack("<6I", hdr[4:])
        if ver != 1:
            raise InputError("unsupported FPVD version")
        dt = np.uint8 if et == 0 else np.float32
        data = np.fromfile(fh, dtype=dt)
    if data.size != F * C * H * W:
        raise InputError("video payload size mismatch")
    return data.reshape(F, C, H, W)
