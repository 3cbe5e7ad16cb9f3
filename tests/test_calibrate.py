"""fp_calibrate_csv: the reference's cost-model calibration (calibrate.cpp)
restated without Eigen; mirrors proj/tests/test_calibrate.cpp and
test_capi.cpp:187-200."""
import ctypes
import json

import numpy as np
import pytest


def features(n, blocks, tile, halo):
    """calibrate.cpp:10-24 (input box = tile + halo per side)."""
    out = blocks * tile[0] * tile[1] * tile[2]
    inb = blocks * (tile[0] + halo[0] + halo[1]) * (tile[1] + halo[2] + halo[3]) * \
        (tile[2] + halo[4] + halo[5])
    win = (halo[0] + halo[1] + 1) * (halo[2] + halo[3] + 1) * (halo[4] + halo[5] + 1)
    return [inb + out, n * out * (win + 1.0), n * out, 1.0]


def varied_rows(seed=77, count=24):
    rng = np.random.default_rng(seed)
    rows = []
    for _ in range(count):
        n = int(rng.integers(1, 7))
        blocks = int(rng.integers(1, 65))
        tile = [int(v) for v in rng.integers(1, 17, 3)]
        r = [int(v) for v in rng.integers(0, 4, 3)]
        rows.append((n, blocks, tile, [r[0], r[0], r[1], r[1], r[2], r[2]]))
    return rows


def csv_of(rows, times):
    lines = ["n_kernels,blocks,tile_x,tile_y,tile_t,halo_x_lo,halo_x_hi,halo_y_lo,halo_y_hi,"
             "halo_t_lo,halo_t_hi,measured_time"]
    for (n, b, t, h), y in zip(rows, times):
        lines.append(",".join(str(v) for v in [n, b, *t, *h]) + f",{y!r}")
    return "\n".join(lines) + "\n"


def calibrate(fp, text):
    out = ctypes.c_void_p()
    st = fp.lib().fp_calibrate_csv(text.encode(), ctypes.byref(out))
    if st != 0:
        return st, fp.lib().fp_last_error().decode()
    s = ctypes.cast(out, ctypes.c_char_p).value.decode()
    fp.lib().fp_string_free(out)
    return st, json.loads(s)


def test_recovers_exact_parameters(fp):
    truth = [73.5, 2.25, 0.4, 12345.0]
    rows = varied_rows()
    times = [float(np.dot(features(*r), truth)) for r in rows]
    st, j = calibrate(fp, csv_of(rows, times))
    assert st == 0, j
    got = [j["params"][k] for k in ("gmem_cost_per_elem", "smem_cost_per_elem",
                                     "compute_cost_unit", "launch_overhead")]
    np.testing.assert_allclose(got, truth, rtol=1e-9)
    assert j["residual_rms"] < 1e-6


def test_noisy_timings(fp):
    truth = [100.0, 1.0, 1.0, 10000.0]
    rows = varied_rows()
    rng = np.random.default_rng(5)
    times = [float(np.dot(features(*r), truth)) * (1 + rng.normal(0, 0.01)) for r in rows]
    st, j = calibrate(fp, csv_of(rows, times))
    assert st == 0
    assert abs(j["params"]["gmem_cost_per_elem"] - 100.0) < 10.0
    assert j["residual_rms"] > 0.0
    # matches a numpy least-squares fit of the same system to rounding
    a = np.array([features(*r) for r in rows])
    x = np.linalg.lstsq(a, np.array(times), rcond=None)[0]
    np.testing.assert_allclose([j["params"][k] for k in ("gmem_cost_per_elem",
                                                          "smem_cost_per_elem",
                                                          "compute_cost_unit",
                                                          "launch_overhead")], x, rtol=1e-6)


def test_validation(fp):
    rows = varied_rows()[:3]
    st, msg = calibrate(fp, csv_of(rows, [1.0, 2.0, 3.0]))
    assert st == 2 and ">= 4 measurements" in msg
    dup = [(2, 8, [8, 8, 2], [1, 1, 1, 1, 0, 0])] * 24
    st, msg = calibrate(fp, csv_of(dup, [123.0] * 24))
    assert st == 2 and "rank deficient" in msg
    st, msg = calibrate(fp, "1,2,3\n")
    assert st == 2 and "expected 12 columns" in msg
    st, msg = calibrate(fp, "1,2,3,4,5,6,7,8,9,10,11,abc\n")
    assert st == 2 and "bad number" in msg
    st, msg = calibrate(fp, "# only a comment\n")
    assert st == 2 and "no measurement rows" in msg


def test_capi_round_trip(fp):
    """test_capi.cpp:187-200."""
    csv = ("2,16,4,4,2,1,1,1,1,0,1,51234.5\n"
           "1,1,32,32,1,0,0,0,0,0,0,220000\n"
           "3,8,8,8,4,2,2,2,2,1,1,990000\n"
           "1,64,2,2,2,0,0,0,0,0,0,170000\n"
           "4,4,16,16,2,1,1,0,0,0,0,880000\n")
    st, j = calibrate(fp, csv)
    assert st == 0
    assert "residual_rms" in j and "gmem_cost_per_elem" in j["params"]
