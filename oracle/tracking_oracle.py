"""TEST INFRASTRUCTURE ONLY -- CPU restatement of the reference's K6 tracking
stage (proj/src/tracking.cpp:40-146), the checker for the device kernel
(paper_1509_04394_b200/csrc/kernels/fc_track.cu).  Never imported by the
product path.

The reference implements the Kalman algebra with Eigen, which is not
available in this container (the reference's tracking.cpp cannot be built
here), so this restatement is pinned to the reference's own behavioural
tests instead (tests/test_tracking.py: static-marker convergence,
test_tracking.cpp:103-117; the 2-marker RMSE <= 1.5 px acceptance criterion,
acceptance.cpp:440-480; the CSV format, tracking.cpp:130-146) -- parity with
the reference's exact FP64 rounding of the Kalman update is unpinned.  The
device kernel is checked bit for bit against THIS restatement: both use the
textbook product order (sum over k ascending from the k = 0 product) and the
closed-form 2x2 inverse, plain IEEE double operations, no contraction.
"""
from __future__ import annotations

import math

import numpy as np

PTS = 23  # measured, meas_x, meas_y, est_x, est_y, est_vx, est_vy, cov[16]


def _matmul(a, b, m, k, n):
    """row-major lists: C[m x n] = A[m x k] B[k x n]."""
    c = [0.0] * (m * n)
    for i in range(m):
        for j in range(n):
            acc = a[i * k] * b[j]
            for kk in range(1, k):
                acc = acc + a[i * k + kk] * b[kk * n + j]
            c[i * n + j] = acc
    return c


def _lround(v: float) -> int:
    """std::lround: nearest, halves away from zero (x - floor(x) is exact)."""
    f = math.floor(v)
    d = v - f
    r = f + 1 if d >= 0.5 else f
    if v < 0 and d == 0.5:
        r = f
    return int(r)


def _centroid(mask_t: np.ndarray, roi, W: int, H: int):
    """tracking.cpp:54-70: pixels > 127 inside the clipped ROI."""
    x0, y0 = max(roi[0], 0), max(roi[1], 0)
    x1, y1 = min(roi[0] + roi[2], W), min(roi[1] + roi[3], H)
    if x1 <= x0 or y1 <= y0:
        return None
    ys, xs = np.nonzero(mask_t[y0:y1, x0:x1] > 127)
    n = len(xs)
    if n == 0:
        return None
    sx = int(xs.sum()) + n * x0
    sy = int(ys.sum()) + n * y0
    return float(sx) / float(n), float(sy) / float(n)


def track_features(mask: np.ndarray, rois, q: float = 0.01, r: float = 0.25,
                   p0: float = 10.0) -> np.ndarray:
    """mask [F, H, W] (u8 or f32); rois [(x, y, w, h)]; returns [n, F, 23]."""
    F, H, W = mask.shape
    f = [1.0 if i % 5 == 0 else 0.0 for i in range(16)]
    f[0 * 4 + 2] = 1.0
    f[1 * 4 + 3] = 1.0
    ft = [f[j * 4 + i] for i in range(4) for j in range(4)]
    qm = [0.0] * 16
    for axis in range(2):  # tracking.cpp:28-38
        p, v = axis, axis + 2
        qm[p * 4 + p] = 0.25 * q
        qm[p * 4 + v] = 0.5 * q
        qm[v * 4 + p] = 0.5 * q
        qm[v * 4 + v] = q
    out = np.zeros((len(rois), F, PTS), np.float64)
    for m, roi0 in enumerate(rois):
        roi = list(roi0)
        state = [float(roi[0]) + float(roi[2]) / 2.0, float(roi[1]) + float(roi[3]) / 2.0,
                 0.0, 0.0]
        cov = [p0 if i % 5 == 0 else 0.0 for i in range(16)]
        for t in range(F):
            if t > 0:
                state = _matmul(f, state, 4, 4, 1)
                fc = _matmul(f, cov, 4, 4, 4)
                fcf = _matmul(fc, ft, 4, 4, 4)
                cov = [fcf[i] + qm[i] for i in range(16)]
            roi[0] = _lround(state[0]) - roi[2] // 2
            roi[1] = _lround(state[1]) - roi[3] // 2
            z = _centroid(mask[t], roi, W, H)
            pt = out[m, t]
            if z is not None:
                zx, zy = z
                if t == 0:
                    state[0], state[1] = zx, zy
                else:
                    s = [cov[0] + r, cov[1] + 0.0, cov[4] + 0.0, cov[5] + r]
                    det = s[0] * s[3] - s[2] * s[1]
                    inv = 1.0 / det
                    si = [s[3] * inv, -s[1] * inv, -s[2] * inv, s[0] * inv]
                    ch = []
                    for i in range(4):
                        ch += [cov[4 * i], cov[4 * i + 1]]
                    k = _matmul(ch, si, 4, 2, 2)
                    y = [zx - state[0], zy - state[1]]
                    ky = _matmul(k, y, 4, 2, 1)
                    state = [state[i] + ky[i] for i in range(4)]
                    ikh = []
                    for i in range(4):
                        for j in range(4):
                            kh = k[2 * i + j] if j < 2 else 0.0
                            ikh.append((1.0 if i == j else 0.0) - kh)
                    cov = _matmul(ikh, cov, 4, 4, 4)
                pt[0], pt[1], pt[2] = 1.0, zx, zy
            pt[3:7] = state
            pt[7:] = cov
    return out


def _g9(v: float) -> str:
    """std::ostream << double with setprecision(9) (%.9g without padding)."""
    return "%.9g" % v


def trajectories_csv(points: np.ndarray) -> str:
    """trajectories_to_csv (tracking.cpp:130-146)."""
    lines = ["frame,marker_id,meas_x,meas_y,est_x,est_y,est_vx,est_vy"]
    n, F, _ = points.shape
    for m in range(n):
        for t in range(F):
            p = points[m, t]
            meas = f"{_g9(p[1])},{_g9(p[2])}" if p[0] != 0.0 else ","
            lines.append(f"{t},{m + 1},{meas},{_g9(p[3])},{_g9(p[4])},{_g9(p[5])},"
                         f"{_g9(p[6])}")
    return "\n".join(lines) + "\n"


def marker_rois(markers):
    """capi.cpp:371-377: a square ROI of side 2 ceil(radius) + 9 at each start."""
    rois = []
    for mk in markers:
        side = 2 * int(math.ceil(mk.get("radius", 3.0))) + 9
        rois.append((_lround(mk.get("x", 0.0)) - side // 2, _lround(mk.get("y", 0.0)) - side // 2,
                     side, side))
    return rois


def truth_centers(spec: dict):
    """synth.cpp:12-18, 55-58: reflected linear marker motion -> [n][F] (x, y)."""
    W, H, F = spec.get("width", 64), spec.get("height", 64), spec.get("frames", 32)

    def reflect(u, limit):
        if limit <= 0.0:
            return 0.0
        period = 2.0 * limit
        m = math.fmod(u, period)
        if m < 0.0:
            m += period
        return m if m <= limit else period - m

    out = []
    for mk in spec.get("markers", []):
        out.append([(reflect(mk.get("x", 0.0) + mk.get("vx", 0.0) * t, W - 1.0),
                     reflect(mk.get("y", 0.0) + mk.get("vy", 0.0) * t, H - 1.0))
                    for t in range(F)])
    return out
