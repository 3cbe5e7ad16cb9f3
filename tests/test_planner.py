"""Partition optimizer parity: this build's planner (C ABI fp_plan_create /
fp_plan_render_json) against the reference planner's output on 146 cases
(tests/golden/plans.json, made by the reference itself: planner.cpp:342-442),
byte for byte, plus the reference's planner known answers
(test_planner.cpp:161-189, acceptance.cpp:255-262, test_capi.cpp:71-94)."""
import json
import os

import pytest

from conftest import GOLDEN, ROOT

DATA = os.path.join(ROOT, "paper_1509_04394_b200", "data")
CASES = json.load(open(os.path.join(GOLDEN, "plans.json")))


def _device_json(name):
    return open(os.path.join(DATA, name + ".json")).read()


def _capi_options(opts, device=None):
    # the golden plans are the reference planner's: the b200 profile's
    # streaming cost model (a B200 extension) is switched off for them
    if device == "b200":
        opts = dict(opts or {}, cost_model="reference")
    if not opts:
        return None
    o = dict(opts)
    if "force_partition" in o:
        o["force_partition"] = ",".join(
            f"{a}-{b}" if a != b else f"{a}" for a, b in o["force_partition"])
    return o


@pytest.mark.parametrize("i", range(len(CASES)))
def test_plan_json_matches_reference(fp, i):
    c = CASES[i]
    p = fp.Pipeline(c["pipeline"])
    d = fp.Device(_device_json(c["device"]))
    if c["status"] != 0:
        with pytest.raises(fp.FuseplanError) as e:
            fp.Plan(p, d, _capi_options(c["options"], c["device"]))
        assert e.value.status == c["status"]
        return
    plan = fp.Plan(p, d, _capi_options(c["options"], c["device"]))
    assert plan.render_json() == c["plan"]


def bundled(fp):
    return fp.Pipeline.load(os.path.join(DATA, "vision_pipeline.json"))


def test_default_plan_bundled_k20(fp):
    """test_planner.cpp:161-175: {1-5},{6}, tile.t == F, halo 3/3/0."""
    plan = fp.Plan(bundled(fp), fp.Device.load("k20_like"))
    doc = json.loads(plan.render_json())
    assert plan.partition == [(1, 5), (6, 6)]
    g = doc["groups"][0]
    assert g["tiled"] and not g["global_aggregation"]
    assert doc["groups"][1]["global_aggregation"]
    assert g["halo"] == {"x_lo": 3, "x_hi": 3, "y_lo": 3, "y_hi": 3, "t_lo": 0, "t_hi": 0}
    assert g["tile"]["t"] == 32
    assert doc["gmem_buffers"]["count"] == 3


def test_traffic_known_answer(fp):
    """acceptance.cpp:255-262: serial 1310720 vs fused 315904 elements."""
    plan = fp.Plan(bundled(fp), fp.Device.load("k20_like"),
                   {"force_partition": "1-5,6", "tile": {"x": 32, "y": 32, "t": 8}})
    doc = json.loads(plan.render_json())
    fused = sum(g["transfer_exact"] for g in doc["groups"])
    assert fused == 315904
    assert 2 * 5 * 64 * 64 * 32 == 1310720


def test_status_taxonomy(fp):
    """test_capi.cpp:71-94."""
    p, d = bundled(fp), fp.Device.load("k20_like")
    with pytest.raises(fp.InputError):
        fp.Plan(p, d, {"force_partition": "2-1"})
    with pytest.raises(fp.InfeasibleError):
        fp.Plan(p, d, {"force_partition": "1-4,5-6"})
    with pytest.raises(fp.InputError):
        fp.Plan(p, d, {"halo_mode": "sideways"})
    plan = fp.Plan(p, d, {"force_partition": "1-5,6"})
    assert "1-5,6" in plan.report()
    with pytest.raises(fp.InputError) as e:
        fp.Pipeline("{bad json")
    assert "JSON" in str(e.value)


def test_large_video_partitions(fp):
    """SURVEY finding 2/3: the reference's Eq-2 model plans >=600 frames as
    1-2,3-5,6 and reports 16000 frames infeasible on k20_like; the b200
    profile under the reference model agrees."""
    from paper_1509_04394_b200.fuseplan import spec_chain
    ref = {"cost_model": "reference"}
    for dev in ("k20_like", "b200"):
        p = fp.Pipeline(json.dumps(spec_chain(800, 600, 1000, kalman=True)))
        assert fp.Plan(p, fp.Device.load(dev), ref).partition == [(1, 2), (3, 5), (6, 6)]
    p = fp.Pipeline(json.dumps(spec_chain(800, 600, 16000, kalman=True)))
    with pytest.raises(fp.InfeasibleError):
        fp.Plan(p, fp.Device.load("k20_like"))
    assert fp.Plan(p, fp.Device.load("b200"), ref).partition == [(1, 2), (3, 5), (6, 6)]


@pytest.mark.parametrize("shape", [(192, 432, 600), (800, 600, 1000), (800, 600, 16000),
                                   (2048, 2048, 1000)])
def test_b200_streaming_cost_picks_the_fastest_partition(fp, shape):
    """The b200 profile's streaming cost model (calibrated on a B200,
    scripts/calibrate_streaming.py) prices each group as the executor runs
    it, so the optimizer returns the all-fused 1-5 -- the measured fastest
    partition on every BASELINE shape (profiles/r02_configs.jsonl) -- where
    the reference's model returned 1-2,3-5."""
    W, H, F = shape
    p = fp.Pipeline(json.dumps(fp.spec_chain(W, H, F, kalman=True)))
    plan = fp.Plan(p, fp.Device.load("b200"))
    assert plan.partition == [(1, 5), (6, 6)]
    doc = json.loads(plan.render_json())
    assert doc["cost_model"].startswith("streaming")
    # predicted cost ranks the partitions like the measurements: all-fused <
    # optimizer-of-the-reference < unfused
    costs = {}
    for part in ("1-5,6", "1-2,3-5,6", "1,2,3,4,5,6"):
        d = json.loads(fp.Plan(p, fp.Device.load("b200"),
                               {"force_partition": part}).render_json())
        costs[part] = d["total_cost"]
    assert costs["1-5,6"] < costs["1-2,3-5,6"] < costs["1,2,3,4,5,6"]
    # the k20_like / c1060_like profiles keep the reference's model
    assert "cost_model" not in json.loads(
        fp.Plan(p, fp.Device.load("k20_like"), None).render_json() if F <= 1000 else "{}")


def test_streaming_cost_model_option(fp):
    p = fp.Pipeline(json.dumps(fp.spec_chain(800, 600, 1000, kalman=True)))
    with pytest.raises(fp.InputError):
        fp.Plan(p, fp.Device.load("k20_like"), {"cost_model": "streaming"})
    with pytest.raises(fp.InputError):
        fp.Plan(p, fp.Device.load("b200"), {"cost_model": "fastest"})
    # an uncertifiable chain (alpha != 0.5): priced with the exact kernels
    q = fp.Pipeline(json.dumps(fp.spec_chain(800, 600, 1000, alpha=0.3, kalman=True)))
    plan = fp.Plan(q, fp.Device.load("b200"))
    assert plan.partition[-1] == (6, 6)


def test_reports_render(fp):
    p = bundled(fp)
    txt = p.analyze()
    assert "TT" in txt and "KK" in txt
    sweep = fp.Device.load("k20_like").tile_sweep([1, 1, 1, 1, 0, 0], 8, 4)
    assert sweep.startswith("x,y,t,du,v,feasible")


def test_iir_streaming_option(fp):
    """B200 extension: by default the planner keeps the reference's rule that
    an IIR group holds the whole time extent (800x600x16000 -> infeasible,
    SURVEY P1); with iir_streaming the streaming executor's plan is feasible
    and the partition / tiles of groups without the IIR are unchanged."""
    spec = fp.spec_chain(800, 600, 16000, kalman=True)
    p = fp.Pipeline(json.dumps(spec))
    dev = fp.Device.load("b200")
    ref = {"cost_model": "reference"}
    with pytest.raises(fp.InfeasibleError):
        fp.Plan(p, dev, dict(ref, force_partition="1-5,6"))
    plan = fp.Plan(p, dev, dict(ref, force_partition="1-5,6", iir_streaming=True))
    assert plan.partition == [(1, 5), (6, 6)]
    # short videos: the option does not change a plan whose t already fits
    q = fp.Pipeline(json.dumps(fp.spec_chain(800, 600, 1000, kalman=True)))
    a = json.loads(fp.Plan(q, dev, dict(ref, force_partition="1-2,3-5,6")).render_json())
    b = json.loads(fp.Plan(q, dev, dict(ref, force_partition="1-2,3-5,6",
                                        iir_streaming=False)).render_json())
    assert a == b
