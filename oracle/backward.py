"""CPU oracle of N4's projection backward -- TEST INFRASTRUCTURE (see
oracle/__init__.py for who may import it).  numpy, float64.

Chains the per-record 2D gradients of `oracle.radiance_backward`
(dL/d{u, v, e_a, e_b, e_c, z}) through the forward projection O1-O7 to the
Gaussian's 3D mean (Alg. 1 l.10-14; the EWA Jacobian of O5 with
the off-screen clamp of reading Q6; the conic of O6; the exponent
coefficients e = k * conic of reading Q29):

  p = R mu + t;  u = fx px/pz + cx,  v = fy py/pz + cy;  z = pz
  J = [[fx/pz, 0, -fx xc/pz^2], [0, fy/pz, -fy yc/pz^2]],  xc = clamp(px/pz) pz
  Sigma' = (J R) Sigma (J R)^T + dilation I = [[a, b], [b, c]]
  conic = (c, -b, a) / (a c - b^2);  (e_a, e_b, e_c) = (k c_a, 2k c_b, k c_c)

dL/dmu = R^T dL/dp + (I - d d^T)/|mu - c| dL/dd, the second term the SH view
direction of O10: rgb_c = max(sum_k b_k(d) f_kc + 0.5, 0), d = (mu - c)/|mu - c|,
c = -R^T t, so dL/dd = sum_c dL/drgb_c [rgb_c > 0] sum_k f_kc grad b_k(d) with the
basis polynomials of O10 differentiated term by term (zero for degree 0).
Alg. 1's literal render-gradient test is ||dL/dmu|| > 0 for L = the
sum of the rendered colour.

`param_backward` continues the same chain to the Gaussian's other parameters
(Theta_i of P:134: opacity, colour, scale, rotation): with G = dL/dSigma' =
[[ga, gb/2], [gb/2, gc]] (a, b, c the entries of Sigma'), dL/dSigma =
T^T G T (T = J R, rows T0, T1); Sigma = M M^T gives dL/dM = 2 dL/dSigma M;
M = R(q) diag(s) gives dL/ds_i = sum_r dL/dM_ri R_ri and dL/dR = dL/dM diag(s);
R(q) of the normalised quaternion (O4) is differentiated entry by entry and
projected, dL/dq = (I - q^ q^T)/|q| dL/dq^; the SH coefficients get
dL/df_kc = b_k(d) dL/drgb_c [rgb_c > 0]; the opacity gets dL/do directly (the
record's o is the scene's linear opacity).
"""
from __future__ import annotations

import numpy as np

K = float(np.float32(-0.72134752044448170368))   # reading Q29 (fp32 constant)


def _sigma3(scale, quat):
    w, x, y, z = (float(q) for q in quat)
    n = np.sqrt(w * w + x * x + y * y + z * z)
    w, x, y, z = w / n, x / n, y / n, z / n
    Rq = np.array([[1 - 2 * (y * y + z * z), 2 * (x * y - w * z), 2 * (x * z + w * y)],
                   [2 * (x * y + w * z), 1 - 2 * (x * x + z * z), 2 * (y * z - w * x)],
                   [2 * (x * z - w * y), 2 * (y * z + w * x), 1 - 2 * (x * x + y * y)]])
    M = Rq @ np.diag(np.asarray(scale, np.float64))
    return M @ M.T


SH_C1 = 0.4886025119029199
SH_C2 = (1.0925484305920792, -1.0925484305920792, 0.31539156525252005, -1.0925484305920792, 0.5462742152960396)
SH_C3 = (-0.5900435899266435, 2.890611442640554, -0.4570457994644658, 0.3731763325901154,
         -0.4570457994644658, 1.445305721320277, -0.5900435899266435)


def sh_basis_grad(deg: int, d) -> np.ndarray:
    """[(deg+1)^2][3]: d b_k / d(x, y, z) of the O10 basis polynomials at d
    (x, y, z treated as independent; the projection onto the sphere is applied
    by the caller)."""
    x, y, z = (float(a) for a in d)
    g = np.zeros(((deg + 1) ** 2, 3))
    if deg < 1:
        return g
    g[1] = (0.0, -SH_C1, 0.0)
    g[2] = (0.0, 0.0, SH_C1)
    g[3] = (-SH_C1, 0.0, 0.0)
    if deg < 2:
        return g
    c = SH_C2
    g[4] = (c[0] * y, c[0] * x, 0.0)
    g[5] = (0.0, c[1] * z, c[1] * y)
    g[6] = (-2 * c[2] * x, -2 * c[2] * y, 4 * c[2] * z)
    g[7] = (c[3] * z, 0.0, c[3] * x)
    g[8] = (2 * c[4] * x, -2 * c[4] * y, 0.0)
    if deg < 3:
        return g
    c = SH_C3
    xx, yy, zz = x * x, y * y, z * z
    g[9] = (6 * c[0] * x * y, c[0] * (3 * xx - 3 * yy), 0.0)
    g[10] = (c[1] * y * z, c[1] * x * z, c[1] * x * y)
    g[11] = (-2 * c[2] * x * y, c[2] * (4 * zz - xx - 3 * yy), 8 * c[2] * y * z)
    g[12] = (-6 * c[3] * x * z, -6 * c[3] * y * z, c[3] * (6 * zz - 3 * xx - 3 * yy))
    g[13] = (c[4] * (4 * zz - 3 * xx - yy), -2 * c[4] * x * y, 8 * c[4] * x * z)
    g[14] = (2 * c[5] * x * z, -2 * c[5] * y * z, c[5] * (xx - yy))
    g[15] = (c[6] * (3 * xx - 3 * yy), -6 * c[6] * x * y, 0.0)
    return g


SH_C0 = 0.28209479177387814


def sh_basis(deg: int, d) -> np.ndarray:
    """O10's real SH basis b_k(d), k < (deg+1)^2 (the polynomials of gs_oracle.cpp)."""
    x, y, z = (float(a) for a in d)
    b = np.zeros((deg + 1) ** 2)
    b[0] = SH_C0
    if deg >= 1:
        b[1], b[2], b[3] = -SH_C1 * y, SH_C1 * z, -SH_C1 * x
    if deg >= 2:
        c = SH_C2
        b[4], b[5] = c[0] * x * y, c[1] * y * z
        b[6] = c[2] * (2 * z * z - x * x - y * y)
        b[7], b[8] = c[3] * x * z, c[4] * (x * x - y * y)
    if deg >= 3:
        c = SH_C3
        xx, yy, zz = x * x, y * y, z * z
        b[9] = c[0] * y * (3 * xx - yy)
        b[10] = c[1] * x * y * z
        b[11] = c[2] * y * (4 * zz - xx - yy)
        b[12] = c[3] * z * (2 * zz - 3 * xx - 3 * yy)
        b[13] = c[4] * x * (4 * zz - xx - yy)
        b[14] = c[5] * z * (xx - yy)
        b[15] = c[6] * x * (xx - 3 * yy)
    return b


def rotation_grads(q):
    """dR/dw, dR/dx, dR/dy, dR/dz of O4's rotation matrix at the unit quaternion q."""
    w, x, y, z = (float(a) for a in q)
    return [np.array([[0, -2 * z, 2 * y], [2 * z, 0, -2 * x], [-2 * y, 2 * x, 0]]),
            np.array([[0, 2 * y, 2 * z], [2 * y, -4 * x, -2 * w], [2 * z, 2 * w, -4 * x]]),
            np.array([[-4 * y, 2 * x, 2 * w], [2 * x, 0, 2 * z], [-2 * w, 2 * z, -4 * y]]),
            np.array([[-4 * z, -2 * w, 2 * x], [2 * w, -4 * z, 2 * y], [2 * x, 2 * y, 0]])]


def param_backward(scene, view, rec, grec, params) -> dict:
    """Per record: dL/d{scale [3], quat [4], opacity, sh [(deg+1)^2 * 3]} (fp64)."""
    R = np.asarray(view.R, np.float64).reshape(3, 3)
    t = np.asarray(view.t, np.float64).reshape(3)
    fx, fy, cx, cy = float(view.fx), float(view.fy), float(view.cx), float(view.cy)
    W, H = view.width, view.height
    m = float(params.clamp_margin)
    lox, hix = (-(m * W) - cx) / fx, ((1.0 + m) * W - cx) / fx
    loy, hiy = (-(m * H) - cy) / fy, ((1.0 + m) * H - cy) / fy
    dil = float(params.dilation)
    cam = -R.T @ t
    deg = int(scene.sh_degree)
    nk = (deg + 1) ** 2
    cnt = len(rec["gid"])
    out = {"scale": np.zeros((cnt, 3)), "quat": np.zeros((cnt, 4)), "opacity": np.zeros(cnt),
           "sh": np.zeros((cnt, nk * 3))}
    for r, g in enumerate(rec["gid"]):
        mu = scene.pos[:, g].astype(np.float64)
        px, py, pz = R @ mu + t
        qraw = scene.quat[:, g].astype(np.float64)
        qn = float(np.linalg.norm(qraw))
        qh = qraw / qn
        w, x, y, z = qh
        Rq = np.array([[1 - 2 * (y * y + z * z), 2 * (x * y - w * z), 2 * (x * z + w * y)],
                       [2 * (x * y + w * z), 1 - 2 * (x * x + z * z), 2 * (y * z - w * x)],
                       [2 * (x * z - w * y), 2 * (y * z + w * x), 1 - 2 * (x * x + y * y)]])
        sc = scene.scale[:, g].astype(np.float64)
        M = Rq @ np.diag(sc)
        Sg = M @ M.T
        xcl = min(max(px / pz, lox), hix)
        ycl = min(max(py / pz, loy), hiy)
        T0 = (fx / pz) * R[0] + (-fx * xcl / pz) * R[2]
        T1 = (fy / pz) * R[1] + (-fy * ycl / pz) * R[2]
        a = T0 @ Sg @ T0 + dil
        b = T0 @ Sg @ T1
        c = T1 @ Sg @ T1 + dil
        det = a * c - b * b
        gu, gv, gea, geb, gec, gop, gr, gg, gb_, gz = grec[r]
        gca, gcb, gcc = K * gea, 2.0 * K * geb, K * gec
        d2 = det * det
        ga = gca * (-c * c / d2) + gcb * (b * c / d2) + gcc * (1.0 / det - a * c / d2)
        gb = gca * (2.0 * b * c / d2) + gcb * (-1.0 / det - 2.0 * b * b / d2) + gcc * (2.0 * a * b / d2)
        gc = gca * (1.0 / det - c * a / d2) + gcb * (b * a / d2) + gcc * (-a * a / d2)
        GS = ga * np.outer(T0, T0) + 0.5 * gb * (np.outer(T0, T1) + np.outer(T1, T0)) + gc * np.outer(T1, T1)
        dM = 2.0 * GS @ M
        out["scale"][r] = (dM * Rq).sum(axis=0)
        dR = dM * sc[None, :]
        dqh = np.array([(dR * G).sum() for G in rotation_grads(qh)])
        out["quat"][r] = (dqh - qh * (qh @ dqh)) / qn
        out["opacity"][r] = gop
        grgb = np.array([gr, gg, gb_]) * (np.asarray(rec["rgb"][r], np.float64) > 0)
        dv = mu - cam
        bk = sh_basis(deg, dv / np.linalg.norm(dv))
        out["sh"][r] = np.outer(bk, grgb).reshape(-1)
    return out


def mean_backward(scene, view, rec, grec, params) -> np.ndarray:
    """dL/dmu [cnt][3] (fp64) for each record; grec [cnt][10] from radiance_backward."""
    R = np.asarray(view.R, np.float64).reshape(3, 3)
    t = np.asarray(view.t, np.float64).reshape(3)
    fx, fy, cx, cy = float(view.fx), float(view.fy), float(view.cx), float(view.cy)
    W, H = view.width, view.height
    m = float(params.clamp_margin)
    lox, hix = (-(m * W) - cx) / fx, ((1.0 + m) * W - cx) / fx
    loy, hiy = (-(m * H) - cy) / fy, ((1.0 + m) * H - cy) / fy
    dil = float(params.dilation)
    cam = -R.T @ t
    out = np.zeros((len(rec["gid"]), 3))
    for r, g in enumerate(rec["gid"]):
        mu = scene.pos[:, g].astype(np.float64)
        p = R @ mu + t
        px, py, pz = p
        Sg = _sigma3(scene.scale[:, g], scene.quat[:, g])
        xn, yn = px / pz, py / pz
        xcl, ycl = min(max(xn, lox), hix), min(max(yn, loy), hiy)
        j00, j11 = fx / pz, fy / pz
        j02, j12 = -fx * xcl / pz, -fy * ycl / pz          # = -fx xc / pz^2 with xc = xcl pz
        T0 = j00 * R[0] + j02 * R[2]
        T1 = j11 * R[1] + j12 * R[2]
        a = T0 @ Sg @ T0 + dil
        b = T0 @ Sg @ T1
        c = T1 @ Sg @ T1 + dil
        det = a * c - b * b
        gu, gv, gea, geb, gec, _, _, _, _, gz = grec[r]
        gca, gcb, gcc = K * gea, 2.0 * K * geb, K * gec
        # conic = (c, -b, a) / det
        d2 = det * det
        ga = gca * (-c * c / d2) + gcb * (b * c / d2) + gcc * (1.0 / det - a * c / d2)
        gb = gca * (2.0 * b * c / d2) + gcb * (-1.0 / det - 2.0 * b * b / d2) + gcc * (2.0 * a * b / d2)
        gc = gca * (1.0 / det - c * a / d2) + gcb * (b * a / d2) + gcc * (-a * a / d2)
        dT0 = 2.0 * ga * (Sg @ T0) + gb * (Sg @ T1)
        dT1 = gb * (Sg @ T0) + 2.0 * gc * (Sg @ T1)
        gj00, gj02 = dT0 @ R[0], dT0 @ R[2]
        gj11, gj12 = dT1 @ R[1], dT1 @ R[2]
        gp = np.zeros(3)
        # u, v, z
        gp[0] += gu * fx / pz
        gp[1] += gv * fy / pz
        gp[2] += -gu * fx * px / (pz * pz) - gv * fy * py / (pz * pz) + gz
        # J entries
        gp[2] += gj00 * (-fx / (pz * pz)) + gj11 * (-fy / (pz * pz))
        if lox < xn < hix:          # j02 = -fx px / pz^2
            gp[0] += gj02 * (-fx / (pz * pz))
            gp[2] += gj02 * (2.0 * fx * px / pz ** 3)
        else:                       # j02 = -fx L / pz (L the clamp bound)
            gp[2] += gj02 * (fx * xcl / (pz * pz))
        if loy < yn < hiy:
            gp[1] += gj12 * (-fy / (pz * pz))
            gp[2] += gj12 * (2.0 * fy * py / pz ** 3)
        else:
            gp[2] += gj12 * (fy * ycl / (pz * pz))
        out[r] = R.T @ gp
        # SH view direction (O10)
        deg = int(scene.sh_degree)
        grgb = np.asarray(grec[r][6:9], np.float64) * (np.asarray(rec["rgb"][r], np.float64) > 0)
        if deg >= 1 and grgb.any():
            dv = mu - cam
            dn = float(np.linalg.norm(dv))
            d = dv / dn
            nk = (deg + 1) ** 2
            coeff = scene.sh[:nk * 3, g].astype(np.float64).reshape(nk, 3)
            gd = sh_basis_grad(deg, d).T @ (coeff @ grgb)
            out[r] += (gd - d * (d @ gd)) / dn
    return out
