"""The C-ABI library loads and exports every entry point include/fuseplan.h
declares; handle / status / ownership conventions match the reference's
tests/test_capi.cpp (no GPU needed for these)."""
import ctypes
import json
import os
import re

import pytest

from conftest import ROOT

HEADER = os.path.join(ROOT, "include", "fuseplan.h")


def declared_functions():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(fp_[a-z0-9_]+)\s*\(", text)))


def test_header_declares_reference_abi():
    names = declared_functions()
    reference = ["fp_last_error", "fp_string_free", "fp_pipeline_parse",
                 "fp_pipeline_load", "fp_pipeline_free", "fp_device_parse",
                 "fp_device_load", "fp_device_free", "fp_plan_create", "fp_plan_free",
                 "fp_plan_render_json", "fp_analyze_report", "fp_plan_report",
                 "fp_tile_sweep", "fp_codegen", "fp_simulate", "fp_calibrate_csv",
                 "fp_device_render_with_cost"]
    for n in reference:
        assert n in names, n


def test_library_exports_every_declared_symbol(fp):
    L = fp.lib()
    for name in declared_functions():
        assert hasattr(L, name), f"{name} not exported"


def test_null_arguments_are_input_errors(fp):
    L = fp.lib()
    out = ctypes.c_void_p()
    assert L.fp_plan_create(None, None, None, ctypes.byref(out)) == fp.FP_ERR_INPUT
    assert b"null" in L.fp_last_error()
    assert L.fp_pipeline_parse(None, ctypes.byref(out)) == fp.FP_ERR_INPUT


def test_device_load_errors(fp):
    L = fp.lib()
    out = ctypes.c_void_p()
    assert L.fp_device_load(b"/nonexistent/device.json", ctypes.byref(out)) == \
        fp.FP_ERR_INPUT
    os.environ["FUSEPLAN_DEVICE_DIR"] = fp.DATA_DIR
    assert L.fp_device_load(b"k20_like", ctypes.byref(out)) == fp.FP_OK
    L.fp_device_free(out)


def test_render_json_owned_string(fp):
    p = fp.Pipeline.load(os.path.join(fp.DATA_DIR, "vision_pipeline.json"))
    plan = fp.Plan(p, fp.Device.load("k20_like"))
    js = plan.render_json()
    assert '"schema_version": 1' in js


def test_pipeline_validation_errors(fp):
    bad = [
        '{"video": {"width": 8, "height": 8, "frames": 2, "channels": 1},'
        ' "kernels": [{"stencil_op": "rgba2gray"}]}',                       # channels
        '{"video": {"width": 8, "height": 8, "frames": 2, "channels": 1},'
        ' "kernels": [{"stencil_op": "warp"}]}',                            # unknown op
        '{"video": {"width": 8, "height": 8, "frames": 2, "channels": 1},'
        ' "kernels": [{"stencil_op": "gaussian", "halo": {"x_lo": -1}}]}',  # negative
        '{"video": {"width": 0, "height": 8, "frames": 2},'
        ' "kernels": [{"stencil_op": "identity"}]}',                        # width
        '{"video": {"width": 8, "height": 8}, "kernels": []}',             # frames
    ]
    for text in bad:
        with pytest.raises(fp.InputError):
            fp.Pipeline(text)


def test_executor_without_gpu_fails_loudly(fp):
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    p = fp.Pipeline.load(os.path.join(fp.DATA_DIR, "vision_pipeline.json"))
    plan = fp.Plan(p, fp.Device.load("k20_like"))
    with pytest.raises(fp.InternalError):
        fp.Executor(p, plan)


def test_malformed_calibration_csv_is_an_input_error(fp):
    L = fp.lib()
    out = ctypes.c_void_p()
    assert L.fp_calibrate_csv(b"n_kernels\n", ctypes.byref(out)) == fp.FP_ERR_INPUT


def test_certified_params_of_the_spec_chain(fp):
    """fp_certified_params (host only): the SPEC chain's normalised taps,
    threshold and band; FP_ERR_INPUT for other chains."""
    import json
    c = fp.Pipeline(json.dumps(fp.spec_chain(64, 32, 4))).certified_params()
    assert c["mstar"] == 16384.0 and abs(c["g1"] - 0.6065306663513184) < 1e-7
    assert 0 < c["band_n"] < 1e-3 * c["mlo_n"]  # a band of ~1e-4 relative
    spec = fp.spec_chain(64, 32, 4)
    spec["kernels"] = spec["kernels"][:3]
    with pytest.raises(fp.InputError):
        fp.Pipeline(json.dumps(spec)).certified_params()


CODEGEN_CASES = [
    ("vision_pipeline.json", "k20_like", None),
    ("vision_pipeline.json", "b200", None),
    ("vision_pipeline.json", "c1060_like", {"halo_mode": "paper-max"}),
    ("vision_pipeline.json", "k20_like", {"force_partition": "1,2,3-5,6"}),
]


@pytest.mark.parametrize("pipe_file,device,opts", CODEGEN_CASES)
def test_codegen_manifest_matches_reference_schema(fp, oracle, tmp_path, pipe_file, device,
                                                   opts):
    """fp_codegen's manifest carries the reference's schema and values
    (codegen.cpp:425-465: pipeline, device, halo_mode, kernels[group, file,
    tile, smem_bytes, staged_arrays, sync_points]), plus the sm_100a kernel
    that executes each group."""
    if not oracle.ref_available():
        pytest.skip("oracle/_ref not built")
    pj = open(os.path.join(fp.DATA_DIR, pipe_file)).read()
    dj = open(os.path.join(fp.DATA_DIR, device + ".json")).read()
    want = oracle.ref_codegen_manifest(pj, dj, opts, "vp")
    L = fp.lib()
    p, d = fp.Pipeline(pj), fp.Device(dj)
    out = ctypes.c_void_p()
    ours = dict(opts or {}, cost_model="reference") if device == "b200" else opts
    st = L.fp_codegen(p.ptr, d.ptr, json.dumps(ours).encode() if ours else None, b"vp",
                      str(tmp_path).encode(), ctypes.byref(out))
    assert st == fp.FP_OK, L.fp_last_error()
    got = json.loads(fp._take_string(out))
    for key in ("pipeline", "device", "halo_mode"):
        assert got[key] == want[key]
    assert len(got["kernels"]) == len(want["kernels"])
    for g, w in zip(got["kernels"], want["kernels"]):
        for key in ("group", "file", "tile", "smem_bytes", "staged_arrays", "sync_points"):
            assert g[key] == w[key], key
        assert "sm_100a" in g["source"] or g["source"].startswith("paper_1509_04394_b200/")
        assert (tmp_path / g["file"]).exists()
