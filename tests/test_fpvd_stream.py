"""FPVD file ingest / egress streamed through the GPU:
fp_exec_run_file reads the reference's raw planar format (video.cpp:46-109)
in chunks, carries the IIR between chunks and writes the output file."""
import json
import struct

import numpy as np
import pytest

from conftest import GOLDEN


def test_python_fpvd_roundtrip(tmp_path):
    from paper_1509_04394_b200.fuseplan import read_fpvd, write_fpvd
    v = np.arange(2 * 3 * 4 * 5, dtype=np.uint8).reshape(2, 3, 4, 5)
    p = tmp_path / "v.fpvd"
    write_fpvd(str(p), v)
    raw = p.read_bytes()
    assert raw[:4] == b"FPVD" and struct.unpack("<6I", raw[4:28]) == (1, 5, 4, 2, 3, 0)
    np.testing.assert_array_equal(read_fpvd(str(p)), v)
    f = (v.astype(np.float32) / 3.0)
    write_fpvd(str(p), f)
    assert struct.unpack("<I", p.read_bytes()[24:28])[0] == 1
    np.testing.assert_array_equal(read_fpvd(str(p)), f)


@pytest.mark.gpu
@pytest.mark.parametrize("chunk", [0, 1, 5, 40])
def test_run_file_spec_chain(fp, cuda, oracle, tmp_path, chunk):
    from paper_1509_04394_b200.fuseplan import hash_video_u8, read_fpvd, spec_chain, write_fpvd
    W, H, F = 160, 96, 23
    pipe = spec_chain(W, H, F, th=24.0)
    v = hash_video_u8(F, 4, H, W, 8)
    src, dst = tmp_path / "in.fpvd", tmp_path / "out.fpvd"
    write_fpvd(str(src), v)
    p = fp.Pipeline(json.dumps(pipe))
    ex = fp.Executor(p, fp.Plan(p, fp.Device.load("b200")), host_chunk_frames=chunk)
    ex.run_file(str(src), str(dst))
    raw = dst.read_bytes()
    assert struct.unpack("<6I", raw[4:28]) == (1, W, H, F, 1, 0)
    got = read_fpvd(str(dst))[:, 0].astype(np.float32)
    np.testing.assert_array_equal(got, oracle.orc_chain(pipe, v))


@pytest.mark.gpu
def test_run_file_f32_planes(fp, cuda, oracle, tmp_path):
    """f32 video in, the F12 group's f32 IIR planes out, chunked."""
    from paper_1509_04394_b200.fuseplan import hash_video_u8, read_fpvd, spec_chain, write_fpvd
    W, H, F = 48, 40, 17
    pipe = spec_chain(W, H, F, alpha=0.3)
    pipe12 = dict(pipe, kernels=pipe["kernels"][:2])
    v = hash_video_u8(F, 4, H, W, 3).astype(np.float32) * 0.5
    src, dst = tmp_path / "in.fpvd", tmp_path / "out.fpvd"
    write_fpvd(str(src), v)
    p = fp.Pipeline(json.dumps(pipe12))
    ex = fp.Executor(p, fp.Plan(p, fp.Device.load("b200")), host_chunk_frames=4)
    ex.run_file(str(src), str(dst))
    got = read_fpvd(str(dst))[:, 0]
    want = oracle.orc_run_sequential(pipe12, v)[-1]
    np.testing.assert_array_equal(got, want)


@pytest.mark.gpu
def test_run_file_errors(fp, cuda, tmp_path):
    from paper_1509_04394_b200.fuseplan import InputError, spec_chain, write_fpvd
    pipe = spec_chain(32, 16, 4)
    p = fp.Pipeline(json.dumps(pipe))
    ex = fp.Executor(p, fp.Plan(p, fp.Device.load("b200")))
    bad = tmp_path / "bad.fpvd"
    bad.write_bytes(b"NOPE" + bytes(24))
    with pytest.raises(InputError):
        ex.run_file(str(bad), str(tmp_path / "o.fpvd"))
    write_fpvd(str(bad), np.zeros((4, 4, 16, 33), np.uint8))  # wrong width
    with pytest.raises(InputError):
        ex.run_file(str(bad), str(tmp_path / "o.fpvd"))
    write_fpvd(str(bad), np.zeros((4, 4, 16, 32), np.uint8))
    bad.write_bytes(bad.read_bytes()[:-10])  # truncated payload
    with pytest.raises(InputError):
        ex.run_file(str(bad), str(tmp_path / "o.fpvd"))
    with pytest.raises(InputError):
        ex.run_file(str(tmp_path / "missing.fpvd"), str(tmp_path / "o.fpvd"))
