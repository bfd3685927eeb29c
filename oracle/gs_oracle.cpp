// ============================================================================
// gs_oracle.cpp -- plain, slow, single-threaded CPU oracle of the Hi^2-GSLoc
// 3DGS forward rasterizer hot path (TEST INFRASTRUCTURE ONLY).
//
// Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may
// load this library.  It shares no code, header, table or constant generator
// with the CUDA path under paper_2507_15683_b200/csrc/.
//
// What it computes (PAPER.md = P:<line>, SPEC.md = S:<line>, readings Q<n> are
// listed in DESIGN.md §2 and SURVEY.md §8(c)):
//   O1-O9  projection, cull, EWA covariance, conic, radius, tile rectangle,
//          depth key                 -- Alg. 1 l.9-12
//   O10    SH colour                 -- colour c_i of Theta_i, [3DGS] basis
//   O11    tile binning: (tile, depth_bits, gid) keys sorted with std::sort,
//          lower-bound ranges        -- "tile-based rasterization"
//   O12    front-to-back alpha compositing of colour, depth, opacity and
//          features                  -- P:136 "alpha blending", "identical
//                                       rasterization"
//   O13    depth back-projection     -- P:278 "fully leverage the depth
//                                       information ... for 3D constraints"
//   O14    threshold-ambiguity flags -- reading Q20
//   brute force: per pixel, all Gaussians whose tile rectangle covers the
//   pixel's tile, sorted by (depth_bits, gid) -- the plain definition that
//   O11+O12 reach faster.
//
// Precision (task rule 3 + reading Q25): every quantity that decides an
// integer (cull, tile rectangle, depth key, the alpha >= 1/255 skip, the
// T < 1e-4 stop, the A >= a_min mask) is computed in IEEE fp32 in the pinned
// operation order written below -- the kernel's precision -- so both sides
// take the same decision.  Build with -ffp-contract=off -fno-fast-math (no FMA
// contraction; x86-64 SSE has FLT_EVAL_METHOD 0).  Values that decide nothing
// (SH colour, the accumulated colour / depth / feature sums, back-projected
// points) are computed in fp64.
//
// Parity status of each function: see the "pins" table in DESIGN.md §5.
// Conventions with no pin but the cited 3DGS convention ("parity unpinned"):
// the Jacobian off-screen clamp margin (Q6), the 0.3 px^2 dilation (Q7),
// the SH signs (O10), the pyramid intrinsics (Q21).
// ============================================================================
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <vector>

extern "C" {

struct or_view {                 // pose maps world -> camera (Q1)
    float R[9];                  // row-major
    float t[3];
    float fx, fy, cx, cy;
    int32_t width, height;
};

struct or_params {
    float z_near;        // Q5   0.2
    float dilation;      // Q7   0.3 px^2
    float clamp_margin;  // Q6   0.15
    float alpha_min;     // Q14  1/255
    float alpha_max;     // Q14  0.99
    float t_min;         // Q15  1e-4
};

// counters layout for oracle_project
enum { OR_NEAR = 0, OR_TRANSPARENT = 1, OR_DEGENERATE = 2, OR_OFFSCREEN = 3 };

}  // extern "C"

namespace {

// ---------------------------------------------------------------------------
// O10: real spherical harmonics up to degree 3 ([3DGS] constants and signs;
// signs are a convention -> parity unpinned; magnitudes pinned by the
// orthonormality quadrature test).  fp64.
// ---------------------------------------------------------------------------
const double SH_C0 = 0.28209479177387814;
const double SH_C1 = 0.4886025119029199;
const double SH_C2[5] = {1.0925484305920792, -1.0925484305920792, 0.31539156525252005,
                         -1.0925484305920792, 0.5462742152960396};
const double SH_C3[7] = {-0.5900435899266435, 2.890611442640554, -0.4570457994644658,
                         0.3731763325901154, -0.4570457994644658, 1.445305721320277,
                         -0.5900435899266435};

// basis[k] for k < (deg+1)^2 at unit direction (x, y, z)
void sh_basis(int deg, double x, double y, double z, double* b) {
    b[0] = SH_C0;
    if (deg < 1) return;
    b[1] = -SH_C1 * y;
    b[2] = SH_C1 * z;
    b[3] = -SH_C1 * x;
    if (deg < 2) return;
    double xx = x * x, yy = y * y, zz = z * z, xy = x * y, yz = y * z, xz = x * z;
    b[4] = SH_C2[0] * xy;
    b[5] = SH_C2[1] * yz;
    b[6] = SH_C2[2] * (2.0 * zz - xx - yy);
    b[7] = SH_C2[3] * xz;
    b[8] = SH_C2[4] * (xx - yy);
    if (deg < 3) return;
    b[9] = SH_C3[0] * y * (3.0 * xx - yy);
    b[10] = SH_C3[1] * xy * z;
    b[11] = SH_C3[2] * y * (4.0 * zz - xx - yy);
    b[12] = SH_C3[3] * z * (2.0 * zz - 3.0 * xx - 3.0 * yy);
    b[13] = SH_C3[4] * x * (4.0 * zz - xx - yy);
    b[14] = SH_C3[5] * z * (xx - yy);
    b[15] = SH_C3[6] * x * (xx - 3.0 * yy);
}

// rgb = max(sum_k basis_k(d) * coeff_k + 0.5, 0)  (colour clamp at 0, Q17)
void sh_color(int deg, const double* coeff /*[nk][3]*/, double dx, double dy, double dz,
              double* rgb) {
    double b[16];
    sh_basis(deg, dx, dy, dz, b);
    int nk = (deg + 1) * (deg + 1);
    for (int c = 0; c < 3; ++c) {
        double s = 0.0;
        for (int k = 0; k < nk; ++k) s += b[k] * coeff[k * 3 + c];
        s += 0.5;
        rgb[c] = s > 0.0 ? s : 0.0;
    }
}

// Q29: the Gaussian exponent is evaluated in log2 units with the fp32 constant
// k = -log2(e)/2 (the literal rounds to the nearest fp32)
const float K_EXP2 = -0.72134752044448170368f;

inline uint32_t float_bits(float f) {
    uint32_t u;
    std::memcpy(&u, &f, 4);
    return u;
}

inline bool finite3(float a, float b, float c) {
    return std::isfinite(a) && std::isfinite(b) && std::isfinite(c);
}

}  // namespace

extern "C" {

// ---------------------------------------------------------------------------
// O10 exported for the SH pins (orthonormality quadrature, degree-0 identity).
// ---------------------------------------------------------------------------
void oracle_sh_color(int32_t deg, const double* coeff, const double* dir, double* rgb) {
    sh_color(deg, coeff, dir[0], dir[1], dir[2], rgb);
}

// ---------------------------------------------------------------------------
// Reading Q30: the alpha >= alpha_min cut in log2 units, from operations that
// round identically everywhere.  alpha = o 2^p >= alpha_min <=> p >= -log2(x),
// x = o / alpha_min >= 1.  For x = m 2^k, m in [1, 2): log2(m) lies below its
// tangent at m0 = 1/ln 2, m - 0.913929 (log2 is concave), so
// log2(x) <= k + (m - 0.9135) (0.0004 slack covers the fp32 rounding; the
// bound is at most 0.0865 loose); inflated by 5% + 0.0075:
// e_cut = -((k + (m - 0.9135)) 1.05 + 0.0075) <= -1.05 log2(x) - 0.0075.
// ---------------------------------------------------------------------------
static float e_cut_of(float op, float alpha_min) {
    const float x = op / alpha_min;
    const uint32_t b = float_bits(x);
    const int32_t k = (int32_t)((b >> 23) & 0xffu) - 127;
    const uint32_t mb = (b & 0x7fffffu) | 0x3f800000u;
    float m;
    std::memcpy(&m, &mb, 4);
    const float lub = (float)k + (m - 0.9135f);
    return -(lub * 1.05f + 0.0075f);
}

// Reading Q30 (N3 tight binning): does the alpha >= alpha_min ellipse
// {d : p(d) >= e_cut}, p(d) = ea dx^2 + eb dx dy + ec dy^2 (ea, ec < 0), reach
// the pixel centres [16tx, 16tx+15] x [16ty, 16ty+15] of tile (tx, ty)?  p is
// concave, so if the mean is outside the rectangle its maximum lies on a
// facing edge, at the edge point nearest the 1-D stationary point.  fp32, this
// exact operation order (the GPU's is identical, so key lists are bit-exact).
static float p_at(float ea, float eb, float ec, float dx, float dy) {
    return ((ea * dx) * dx + (eb * dx) * dy) + (ec * dy) * dy;
}
static bool tile_hit(float u, float v, float ea, float eb, float ec, float ecut, int32_t tx, int32_t ty) {
    const float X0 = (float)(tx * 16), X1 = (float)(tx * 16 + 15);
    const float Y0 = (float)(ty * 16), Y1 = (float)(ty * 16 + 15);
    const bool inx = X0 <= u && u <= X1, iny = Y0 <= v && v <= Y1;
    if (inx && iny) return true;
    float pmax = -INFINITY;
    // stationary-point slopes, one rounded division each: dy*(dx) = sy dx, dx*(dy) = sx dy
    const float sy = -eb / (2.0f * ec), sx = -eb / (2.0f * ea);
    if (!inx) {   // facing vertical edge
        const float dx = (u < X0 ? X0 : X1) - u;
        const float dy = std::fmin(std::fmax(sy * dx, Y0 - v), Y1 - v);
        pmax = std::fmax(pmax, p_at(ea, eb, ec, dx, dy));
    }
    if (!iny) {   // facing horizontal edge
        const float dy = (v < Y0 ? Y0 : Y1) - v;
        const float dx = std::fmin(std::fmax(sx * dy, X0 - u), X1 - u);
        pmax = std::fmax(pmax, p_at(ea, eb, ec, dx, dy));
    }
    return pmax >= ecut;
}

// ---------------------------------------------------------------------------
// O1-O10 for one view.  Scene planes are SoA: pos[3][n], quat[4][n] (w,x,y,z),
// scale[3][n], opacity[n], sh[(deg+1)^2*3][n].  Visible Gaussians are written
// in ascending gid order; returns their count.  diag[4] += cull counters.
// ---------------------------------------------------------------------------
int64_t oracle_project(int64_t n, const float* pos, const float* quat, const float* scale,
                       const float* opacity, const float* sh, int32_t sh_degree,
                       const or_view* V, const or_params* P,
                       int32_t* out_gid, float* out_u, float* out_v, float* out_z,
                       float* out_conic /*[cnt][3]*/, float* out_radius,
                       int32_t* out_rect /*[cnt][4] = x0,x1,y0,y1 inclusive*/,
                       float* out_rgb /*[cnt][3]*/, float* out_opacity,
                       float* out_cov /*[cnt][3] = a,b,c incl. dilation (diagnostic)*/,
                       float* out_ecut /*[cnt] reading Q30*/, int64_t* diag) {
    const float* R = V->R;
    const float W = (float)V->width, H = (float)V->height;
    const int32_t TX = (V->width + 15) / 16, TY = (V->height + 15) / 16;
    const float TXf = (float)TX, TYf = (float)TY;
    // camera centre in world (fp64, SH view direction only): c = -R^T t
    double cc[3];
    for (int k = 0; k < 3; ++k)
        cc[k] = -((double)R[0 * 3 + k] * V->t[0] + (double)R[1 * 3 + k] * V->t[1] +
                  (double)R[2 * 3 + k] * V->t[2]);
    const int nk = (sh_degree + 1) * (sh_degree + 1);
    int64_t cnt = 0;
    for (int64_t i = 0; i < n; ++i) {
        const float mx = pos[0 * n + i], my = pos[1 * n + i], mz = pos[2 * n + i];
        // O1: camera transform, p_k = ((R_k0 mx + R_k1 my) + R_k2 mz) + t_k
        const float px = ((R[0] * mx + R[1] * my) + R[2] * mz) + V->t[0];
        const float py = ((R[3] * mx + R[4] * my) + R[5] * mz) + V->t[1];
        const float pz = ((R[6] * mx + R[7] * my) + R[8] * mz) + V->t[2];
        // O2: near cull (NaN z is culled here too)
        if (!(pz > P->z_near)) { diag[OR_NEAR]++; continue; }
        const float op = opacity[i];
        if (!(op >= P->alpha_min)) { diag[OR_TRANSPARENT]++; continue; }
        const float s0 = scale[0 * n + i], s1 = scale[1 * n + i], s2 = scale[2 * n + i];
        const float qw = quat[0 * n + i], qx = quat[1 * n + i], qy = quat[2 * n + i],
                    qz = quat[3 * n + i];
        if (!(s0 > 0.0f) || !(s1 > 0.0f) || !(s2 > 0.0f) || !finite3(s0, s1, s2) ||
            !finite3(px, py, pz) || !finite3(qw, qx, qy) || !std::isfinite(qz)) {
            diag[OR_DEGENERATE]++; continue;
        }
        // O3: mean, Alg. 1 order: divide by depth first, then apply K
        const float xn = px / pz, yn = py / pz;
        const float u = V->fx * xn + V->cx;
        const float v = V->fy * yn + V->cy;
        // O4: 3D covariance Sigma = M M^T, M = R(q) diag(s), q normalised (Q2)
        const float qn2 = ((qw * qw + qx * qx) + qy * qy) + qz * qz;
        if (!(qn2 > 0.0f)) { diag[OR_DEGENERATE]++; continue; }
        const float qn = std::sqrt(qn2);
        const float w = qw / qn, x = qx / qn, y = qy / qn, z = qz / qn;
        const float xx = x * x, yy = y * y, zz = z * z;
        const float xy = x * y, xz = x * z, yz = y * z;
        const float wx = w * x, wy = w * y, wz = w * z;
        const float Rq[9] = {1.0f - 2.0f * (yy + zz), 2.0f * (xy - wz), 2.0f * (xz + wy),
                             2.0f * (xy + wz), 1.0f - 2.0f * (xx + zz), 2.0f * (yz - wx),
                             2.0f * (xz - wy), 2.0f * (yz + wx), 1.0f - 2.0f * (xx + yy)};
        float M[9];
        for (int r = 0; r < 3; ++r) {
            M[r * 3 + 0] = Rq[r * 3 + 0] * s0;
            M[r * 3 + 1] = Rq[r * 3 + 1] * s1;
            M[r * 3 + 2] = Rq[r * 3 + 2] * s2;
        }
        float S[9];  // Sigma_ij = (M_i0 M_j0 + M_i1 M_j1) + M_i2 M_j2
        for (int r = 0; r < 3; ++r)
            for (int c = 0; c < 3; ++c)
                S[r * 3 + c] = (M[r * 3 + 0] * M[c * 3 + 0] + M[r * 3 + 1] * M[c * 3 + 1]) +
                               M[r * 3 + 2] * M[c * 3 + 2];
        // O5: EWA.  Off-screen guard (Q6): clamp x/z to [(-m W - cx)/fx, ((1+m) W - cx)/fx]
        const float m = P->clamp_margin;
        const float lox = (-(m * W) - V->cx) / V->fx, hix = ((1.0f + m) * W - V->cx) / V->fx;
        const float loy = (-(m * H) - V->cy) / V->fy, hiy = ((1.0f + m) * H - V->cy) / V->fy;
        const float xc = std::min(std::max(xn, lox), hix) * pz;
        const float yc = std::min(std::max(yn, loy), hiy) * pz;
        // J = [[fx/z, 0, -fx x~/z^2], [0, fy/z, -fy y~/z^2]]
        const float z2 = pz * pz;
        const float j00 = V->fx / pz, j02 = -((V->fx * xc) / z2);
        const float j11 = V->fy / pz, j12 = -((V->fy * yc) / z2);
        // T = J R (2x3)
        float T[6];
        for (int k = 0; k < 3; ++k) {
            T[0 * 3 + k] = j00 * R[0 * 3 + k] + j02 * R[2 * 3 + k];
            T[1 * 3 + k] = j11 * R[1 * 3 + k] + j12 * R[2 * 3 + k];
        }
        // Sigma' = T Sigma T^T : first Vt = T Sigma (2x3), then Vt T^T
        float Vt[6];
        for (int r = 0; r < 2; ++r)
            for (int k = 0; k < 3; ++k)
                Vt[r * 3 + k] = (T[r * 3 + 0] * S[0 * 3 + k] + T[r * 3 + 1] * S[1 * 3 + k]) +
                                T[r * 3 + 2] * S[2 * 3 + k];
        const float s00 = (Vt[0] * T[0] + Vt[1] * T[1]) + Vt[2] * T[2];
        const float s01 = (Vt[0] * T[3] + Vt[1] * T[4]) + Vt[2] * T[5];
        const float s11 = (Vt[3] * T[3] + Vt[4] * T[4]) + Vt[5] * T[5];
        const float a = s00 + P->dilation, b = s01, c = s11 + P->dilation;
        // O6: conic = inverse of [[a, b], [b, c]]
        const float det = a * c - b * b;
        if (!(det > 0.0f)) { diag[OR_DEGENERATE]++; continue; }
        const float ca = c / det, cb = -(b / det), ccn = a / det;
        // O7: radius r = ceil(3 sqrt(lambda_max)), lambda_max = mid + sqrt(max(mid^2 - det, 0)) (Q8, Q9)
        const float mid = 0.5f * (a + c);
        const float lam = mid + std::sqrt(std::max(mid * mid - det, 0.0f));
        const float r = std::ceil(3.0f * std::sqrt(lam));
        // O8: tile rectangle, inclusive floor((u -+ r)/16) (Q10), cull if off-grid
        if (!std::isfinite(u) || !std::isfinite(v) || !std::isfinite(r)) { diag[OR_DEGENERATE]++; continue; }
        const float fx0 = std::floor((u - r) * 0.0625f), fx1 = std::floor((u + r) * 0.0625f);
        const float fy0 = std::floor((v - r) * 0.0625f), fy1 = std::floor((v + r) * 0.0625f);
        if (fx1 < 0.0f || fx0 >= TXf || fy1 < 0.0f || fy0 >= TYf) { diag[OR_OFFSCREEN]++; continue; }
        const int32_t x0 = (int32_t)std::max(fx0, 0.0f), x1 = (int32_t)std::min(fx1, TXf - 1.0f);
        const int32_t y0 = (int32_t)std::max(fy0, 0.0f), y1 = (int32_t)std::min(fy1, TYf - 1.0f);
        // O10: SH colour at view direction d = (mu - c_cam)/|mu - c_cam| (fp64)
        double d[3] = {(double)mx - cc[0], (double)my - cc[1], (double)mz - cc[2]};
        const double dn = std::sqrt(d[0] * d[0] + d[1] * d[1] + d[2] * d[2]);
        double coeff[48], rgb[3];
        for (int k = 0; k < nk * 3; ++k) coeff[k] = sh[(int64_t)k * n + i];
        sh_color(sh_degree, coeff, d[0] / dn, d[1] / dn, d[2] / dn, rgb);

        out_gid[cnt] = (int32_t)i;
        out_u[cnt] = u;
        out_v[cnt] = v;
        out_z[cnt] = pz;
        out_conic[cnt * 3 + 0] = ca;
        out_conic[cnt * 3 + 1] = cb;
        out_conic[cnt * 3 + 2] = ccn;
        out_radius[cnt] = r;
        out_rect[cnt * 4 + 0] = x0;
        out_rect[cnt * 4 + 1] = x1;
        out_rect[cnt * 4 + 2] = y0;
        out_rect[cnt * 4 + 3] = y1;
        for (int k = 0; k < 3; ++k) out_rgb[cnt * 3 + k] = (float)rgb[k];
        out_opacity[cnt] = op;
        out_cov[cnt * 3 + 0] = a;
        out_cov[cnt * 3 + 1] = b;
        out_cov[cnt * 3 + 2] = c;
        out_ecut[cnt] = e_cut_of(op, P->alpha_min);
        ++cnt;
    }
    return cnt;
}

// ---------------------------------------------------------------------------
// O11: number of (tile, Gaussian) pairs = sum of rectangle areas.
// ---------------------------------------------------------------------------
// Binning mode (N3, reading Q30): tight == NULL -> every tile of the 3-sigma
// rectangle (O8); else only the rectangle's tiles with tile_hit, from the
// record fields u, v, conic and e_cut (exponent coefficients as in Q29).
struct Tight {
    const float *u, *v, *conic, *ecut;
};
static bool keep_tile(const Tight* tight, int64_t i, int32_t tx, int32_t ty) {
    if (!tight) return true;
    const float* c = tight->conic + i * 3;
    const float ea = K_EXP2 * c[0], eb = (2.0f * K_EXP2) * c[1], ec = K_EXP2 * c[2];
    return tile_hit(tight->u[i], tight->v[i], ea, eb, ec, tight->ecut[i], tx, ty);
}

int64_t oracle_count_pairs(int64_t cnt, const int32_t* rect, const Tight* tight) {
    int64_t p = 0;
    for (int64_t i = 0; i < cnt; ++i)
        for (int32_t ty = rect[i * 4 + 2]; ty <= rect[i * 4 + 3]; ++ty)
            for (int32_t tx = rect[i * 4 + 0]; tx <= rect[i * 4 + 1]; ++tx) p += keep_tile(tight, i, tx, ty);
    return p;
}

// ---------------------------------------------------------------------------
// O11: emit one key (tile = ty*TX + tx, depth_bits = bits(z), gid) per tile of
// each rectangle; sort lexicographically (Q12: equal depth -> ascending gid);
// ranges[t] = [#keys with smaller tile, that + count[t])  (lower bound, Q13).
// key_rec[j] is the record index of key j (into the oracle_project arrays).
// ---------------------------------------------------------------------------
struct Key {
    uint32_t tile, depth, gid, rec;
};

void oracle_bin(int64_t cnt, const int32_t* gid, const float* zv, const int32_t* rect, const Tight* tight,
                int32_t tiles_x, int32_t tiles_y, uint32_t* key_tile, uint32_t* key_depth,
                uint32_t* key_gid, uint32_t* key_rec, uint32_t* ranges /*[T][2]*/) {
    std::vector<Key> keys;
    for (int64_t i = 0; i < cnt; ++i)
        for (int32_t ty = rect[i * 4 + 2]; ty <= rect[i * 4 + 3]; ++ty)
            for (int32_t tx = rect[i * 4 + 0]; tx <= rect[i * 4 + 1]; ++tx)
                if (keep_tile(tight, i, tx, ty))
                    keys.push_back({(uint32_t)(ty * tiles_x + tx), float_bits(zv[i]), (uint32_t)gid[i],
                                    (uint32_t)i});
    std::sort(keys.begin(), keys.end(), [](const Key& a, const Key& b) {
        if (a.tile != b.tile) return a.tile < b.tile;
        if (a.depth != b.depth) return a.depth < b.depth;
        return a.gid < b.gid;
    });
    for (size_t j = 0; j < keys.size(); ++j) {
        key_tile[j] = keys[j].tile;
        key_depth[j] = keys[j].depth;
        key_gid[j] = keys[j].gid;
        key_rec[j] = keys[j].rec;
    }
    const int64_t T = (int64_t)tiles_x * tiles_y;
    size_t j = 0;
    for (int64_t t = 0; t < T; ++t) {
        while (j < keys.size() && keys[j].tile < (uint32_t)t) ++j;
        ranges[t * 2 + 0] = (uint32_t)j;
        size_t e = j;
        while (e < keys.size() && keys[e].tile == (uint32_t)t) ++e;
        ranges[t * 2 + 1] = (uint32_t)e;
    }
}

// ---------------------------------------------------------------------------
// O12 + O14: composite one pixel given its ordered list of record indices.
// ---------------------------------------------------------------------------
struct Records {
    const float *u, *v, *conic, *opacity, *rgb, *z;
    const int32_t* gid;
    const float* feat;  // [n_gauss][D]
    int32_t D;
};

struct PixelOut {
    double C[3], Dz;
    std::vector<double> F;
    float T;
    uint8_t flags;
    int64_t evals, blends;
    double a_err;   // O14: bound on |A_kernel - A_oracle| (absolute), for the a_min band
};

// O14 flag bands (reading Q20, derived in DESIGN.md §2 "Q20 bands"): the only
// decision input the kernel evaluates differently is 2^p (ex2.approx.ftz.f32 vs
// the oracle's fp64 2^p).  EX2_REL bounds |ex2.approx(p) / 2^p - 1| over every
// fp32 p <= 0 (measured exhaustively on the B200: tools/ex2_probe.cu,
// profiles/r02_ex2_probe.json, times a margin of 2); both sides then round
// o * 2^p once, so alpha_raw deviates by at most ALPHA_REL relative.  The
// deviation of T is propagated step by step: 1 - alpha (absolute alpha
// deviation, both sides' rounding), T (1 - alpha) (both sides' rounding).  A
// decision is flagged when the oracle's value lies within BAND_SAFETY times the
// propagated bound of its threshold.
const double U24 = 1.0 / 16777216.0;          // 2^-24, unit roundoff of fp32
const double EX2_REL = 1.0 / 2097152.0;       // 2^-21
const double ALPHA_REL = EX2_REL + 2.0 * U24;
const double BAND_SAFETY = 2.0;

// N4 (feature-field backward, Eq. 2 with the geometry frozen): when gF is set,
// fgrad[gid][c] += w * gF[c][pix] for every blended entry -- dL/df of a loss
// whose gradient w.r.t. the rendered feature map is gF, since F = sum_k w_k f_k.
struct FeatGrad {
    const float* gF;   // [D][H][W] upstream gradient of this view
    int64_t HW, pix;
    double* fgrad;     // [n_gauss][D]
};

void composite_pixel(const Records& rc, const or_params* P, int32_t pxi, int32_t pyi,
                     const uint32_t* list, int64_t len, PixelOut& o, double* contrib,
                     const FeatGrad* fg = nullptr) {
    const float pxf = (float)pxi, pyf = (float)pyi;
    float T = 1.0f;
    o.C[0] = o.C[1] = o.C[2] = 0.0;
    o.Dz = 0.0;
    o.F.assign(rc.D, 0.0);
    o.flags = 0;
    o.evals = 0;
    o.blends = 0;
    double eps_T = 0.0;   // O14: bound on |T_kernel / T_oracle - 1|
    for (int64_t k = 0; k < len; ++k) {
        const uint32_t i = list[k];
        o.evals++;
        // 1. offset of the mean from the pixel centre (integer centres, Q4)
        const float dx = rc.u[i] - pxf, dy = rc.v[i] - pyf;
        // 2. power = -0.5 (ca dx dx + cc dy dy) - cb dx dy, evaluated in log2 units (reading
        //    Q29): p = power log2(e) = dx (ea dx + eb dy) + ec dy dy with ea = k ca, eb = 2k cb,
        //    ec = k cc, k = fp32(-log2(e) / 2), fp32 fused multiply-adds in this order
        const float ca = rc.conic[i * 3 + 0], cb = rc.conic[i * 3 + 1], cc = rc.conic[i * 3 + 2];
        const float ea = K_EXP2 * ca, eb = (2.0f * K_EXP2) * cb, ec = K_EXP2 * cc;
        const float p = std::fmaf(dx, std::fmaf(ea, dx, eb * dy), (ec * dy) * dy);
        // 3. skip if power > 0
        if (p > 0.0f) continue;
        // 4. alpha = min(alpha_max, o exp(power)) = min(alpha_max, o 2^p); 2^p in fp64 rounded
        //    once to fp32
        const float araw = (float)((double)rc.opacity[i] * std::exp2((double)p));
        // O14 (a): the alpha >= alpha_min decision is ambiguous within ALPHA_REL
        if (std::fabs((double)araw - (double)P->alpha_min) <= BAND_SAFETY * ALPHA_REL * (double)araw)
            o.flags |= 1;
        const float alpha = std::min(P->alpha_max, araw);
        // 5. skip if alpha < alpha_min (1/255)
        if (alpha < P->alpha_min) continue;
        // 6. Tn = T (1 - alpha); stop WITHOUT blending if Tn < t_min (Q15)
        const float om = 1.0f - alpha;
        const float Tn = T * om;
        // O14 (b): deviation bound of Tn.  alpha deviates by <= ALPHA_REL alpha_raw
        // unless both sides clamp to alpha_max (then it is identical)
        const double d_alpha = ((double)araw > (double)P->alpha_max * (1.0 + ALPHA_REL)) ? 0.0
                                                                                      : ALPHA_REL * (double)araw;
        const double eps_Tn = eps_T + (d_alpha / (double)om + 2.0 * U24) + 2.0 * U24;
        if (std::fabs((double)Tn - (double)P->t_min) <= BAND_SAFETY * eps_Tn * (double)Tn) o.flags |= 2;
        if (Tn < P->t_min) break;
        // 7. w = alpha T; accumulate colour, depth (camera z, Q16) and features (Q18)
        const float w = alpha * T;
        for (int c = 0; c < 3; ++c) o.C[c] += (double)w * rc.rgb[i * 3 + c];
        o.Dz += (double)w * rc.z[i];
        if (rc.D > 0) {
            const float* f = rc.feat + (int64_t)rc.gid[i] * rc.D;
            for (int c = 0; c < rc.D; ++c) o.F[c] += (double)w * f[c];
        }
        o.blends++;
        if (contrib) contrib[i] += (double)w;   // N1: per-Gaussian accumulated blend weight
        if (fg)
            for (int c = 0; c < rc.D; ++c)
                fg->fgrad[(int64_t)rc.gid[i] * rc.D + c] += (double)w * fg->gF[c * fg->HW + fg->pix];
        // 8. T = Tn
        T = Tn;
        eps_T = eps_Tn;
    }
    o.T = T;
    // O14 (c): A = 1 - T deviates by <= T eps_T plus both sides' rounding of 1 - T
    o.a_err = BAND_SAFETY * ((double)T * eps_T + 2.0 * U24);
}

void store_pixel(const PixelOut& o, int64_t HW, int64_t pix, float* out_rgb, float* out_depth,
                 float* out_alpha, float* out_feat, uint8_t* flags, int32_t D, float* a_err) {
    if (a_err) a_err[pix] = (float)o.a_err;
    for (int c = 0; c < 3; ++c) out_rgb[c * HW + pix] = (float)o.C[c];
    out_depth[pix] = (float)o.Dz;
    out_alpha[pix] = 1.0f - o.T;  // A = 1 - T
    for (int c = 0; c < D; ++c) out_feat[(int64_t)c * HW + pix] = (float)o.F[c];
    flags[pix] = o.flags;
}

// O12 over the binned lists: outputs planar [3][H][W], [H][W], [H][W], [D][H][W]
void oracle_composite(const or_view* V, const or_params* P, const float* u, const float* v,
                      const float* conic, const float* opac, const float* rgb, const float* z,
                      const int32_t* gid, const float* feat, int32_t D, const uint32_t* key_rec,
                      const uint32_t* ranges, float* out_rgb, float* out_depth, float* out_alpha,
                      float* out_feat, uint8_t* flags, int64_t* counters /*[2] E, B*/,
                      double* contrib /*[cnt] or NULL*/, float* a_err /*[H][W] or NULL*/) {
    Records rc{u, v, conic, opac, rgb, z, gid, feat, D};
    const int32_t W = V->width, H = V->height, TX = (W + 15) / 16;
    const int64_t HW = (int64_t)W * H;
    PixelOut o;
    for (int32_t py = 0; py < H; ++py)
        for (int32_t px = 0; px < W; ++px) {
            const int64_t t = (int64_t)(py / 16) * TX + px / 16;
            const uint32_t s = ranges[t * 2], e = ranges[t * 2 + 1];
            composite_pixel(rc, P, px, py, key_rec + s, (int64_t)e - s, o, contrib);
            const int64_t pix = (int64_t)py * W + px;
            store_pixel(o, HW, pix, out_rgb, out_depth, out_alpha, out_feat, flags, D, a_err);
            counters[0] += o.evals;
            counters[1] += o.blends;
        }
}

// N4: dL/df accumulated over this view (fgrad [n_gauss][D], added to).
void oracle_feature_grad(const or_view* V, const or_params* P, const float* u, const float* v,
                         const float* conic, const float* opac, const float* rgb, const float* z,
                         const int32_t* gid, const float* feat, int32_t D, const uint32_t* key_rec,
                         const uint32_t* ranges, const float* gF, double* fgrad) {
    Records rc{u, v, conic, opac, rgb, z, gid, feat, D};
    const int32_t W = V->width, H = V->height, TX = (W + 15) / 16;
    const int64_t HW = (int64_t)W * H;
    PixelOut o;
    for (int32_t py = 0; py < H; ++py)
        for (int32_t px = 0; px < W; ++px) {
            const int64_t t = (int64_t)(py / 16) * TX + px / 16;
            const uint32_t s = ranges[t * 2], e = ranges[t * 2 + 1];
            const FeatGrad fg{gF, HW, (int64_t)py * W + px, fgrad};
            composite_pixel(rc, P, px, py, key_rec + s, (int64_t)e - s, o, nullptr, &fg);
        }
}

// N4 (radiance backward): for the linear loss L = sum_px gC . C + gD Dz + gA A
// (any loss's first-order term), per record the gradient w.r.t.
// g[10] = {u, v, ea, eb, ec, opacity, r, g, b, z}, fp64, front to back:
//   dC/dalpha_k = T_k c_k - (C_f - C_{<=k}) / (1 - alpha_k),   dA/dalpha_k = T_f / (1 - alpha_k),
//   alpha = o 2^p (unclamped): dalpha/do = 2^p, dalpha/dp = alpha ln 2,
//   p = ea dx^2 + eb dx dy + ec dy^2 with dx = u - px, dy = v - py.
// The skip and stop decisions are taken exactly as in composite_pixel (their
// gradient is zero); a clamped alpha (0.99) has no opacity / exponent gradient.
// Also returns the loss itself in fp64 (for finite-difference pins).
// N4 joint step (Eq. 1 with Eq. 2's feature term through the geometry):
// gF (may be NULL) is this pixel's upstream gradient of the rendered feature
// vector F = sum_k w_k f_k; it enters exactly like a colour channel,
//   dF_c/dalpha_k = T_k f_kc - (F_c - F_c,<=k) / (1 - alpha_k),
// and the returned loss includes sum_c gF_c F_c.
double backward_pixel(const Records& rc, const or_params* P, int32_t pxi, int32_t pyi, const uint32_t* list,
                      int64_t len, const double gC[3], double gD, double gA, double* grec /*[cnt][10]*/,
                      const double* gF = nullptr) {
    PixelOut f;
    composite_pixel(rc, P, pxi, pyi, list, len, f, nullptr);
    const int32_t DF = gF ? rc.D : 0;
    std::vector<double> Facc(DF, 0.0);
    const double Tf = f.T;
    const float pxf = (float)pxi, pyf = (float)pyi;
    float T = 1.0f;
    double Cacc[3] = {0, 0, 0}, Dacc = 0;
    for (int64_t k = 0; k < len; ++k) {
        const uint32_t i = list[k];
        const float dx = rc.u[i] - pxf, dy = rc.v[i] - pyf;
        const float ca = rc.conic[i * 3 + 0], cb = rc.conic[i * 3 + 1], cc = rc.conic[i * 3 + 2];
        const float ea = K_EXP2 * ca, eb = (2.0f * K_EXP2) * cb, ec = K_EXP2 * cc;
        const float p = std::fmaf(dx, std::fmaf(ea, dx, eb * dy), (ec * dy) * dy);
        if (p > 0.0f) continue;
        const double e2p = std::exp2((double)p);
        const float araw = (float)((double)rc.opacity[i] * e2p);
        const float alpha = std::min(P->alpha_max, araw);
        if (alpha < P->alpha_min) continue;
        const float Tn = T * (1.0f - alpha);
        if (Tn < P->t_min) break;
        const float w = alpha * T;
        const double* c = nullptr;
        double cd[3] = {rc.rgb[i * 3], rc.rgb[i * 3 + 1], rc.rgb[i * 3 + 2]};
        c = cd;
        for (int q = 0; q < 3; ++q) Cacc[q] += (double)w * c[q];
        Dacc += (double)w * rc.z[i];
        const double om = 1.0 - (double)alpha;
        double dLda = 0.0;
        for (int q = 0; q < 3; ++q) dLda += gC[q] * ((double)T * c[q] - (f.C[q] - Cacc[q]) / om);
        dLda += gD * ((double)T * rc.z[i] - (f.Dz - Dacc) / om);
        dLda += gA * (Tf / om);
        if (DF) {
            const float* fk = rc.feat + (int64_t)rc.gid[i] * rc.D;
            for (int q = 0; q < DF; ++q) {
                Facc[q] += (double)w * fk[q];
                dLda += gF[q] * ((double)T * fk[q] - (f.F[q] - Facc[q]) / om);
            }
        }
        double* g = grec + (int64_t)i * 10;
        for (int q = 0; q < 3; ++q) g[6 + q] += (double)w * gC[q];
        g[9] += (double)w * gD;
        if (araw <= P->alpha_max) {   // unclamped: alpha = o 2^p
            g[5] += dLda * e2p;
            const double dLdp = dLda * (double)araw * 0.69314718055994530942;
            const double ddx = dx, ddy = dy;
            g[2] += dLdp * ddx * ddx;
            g[3] += dLdp * ddx * ddy;
            g[4] += dLdp * ddy * ddy;
            g[0] += dLdp * (2.0 * ea * ddx + eb * ddy);
            g[1] += dLdp * (eb * ddx + 2.0 * ec * ddy);
        }
        T = Tn;
    }
    double loss = gC[0] * f.C[0] + gC[1] * f.C[1] + gC[2] * f.C[2] + gD * f.Dz + gA * (1.0 - Tf);
    for (int q = 0; q < DF; ++q) loss += gF[q] * f.F[q];
    return loss;
}

double oracle_radiance_backward(const or_view* V, const or_params* P, const float* u, const float* v,
                                const float* conic, const float* opac, const float* rgb, const float* z,
                                const int32_t* gid, const uint32_t* key_rec, const uint32_t* ranges,
                                const float* gC /*[3][H][W]*/, const float* gD, const float* gA, double* grec,
                                const float* feat /*[n_gauss][D] or NULL*/, int32_t D,
                                const float* gF /*[D][H][W] or NULL*/) {
    Records rc{u, v, conic, opac, rgb, z, gid, feat, gF ? D : 0};
    const int32_t W = V->width, H = V->height, TX = (W + 15) / 16;
    const int64_t HW = (int64_t)W * H;
    double loss = 0.0;
    std::vector<double> gpx(gF ? D : 0);
    for (int32_t py = 0; py < H; ++py)
        for (int32_t px = 0; px < W; ++px) {
            const int64_t t = (int64_t)(py / 16) * TX + px / 16, pix = (int64_t)py * W + px;
            const uint32_t s = ranges[t * 2], e = ranges[t * 2 + 1];
            const double g3[3] = {gC[pix], gC[HW + pix], gC[2 * HW + pix]};
            if (gF)
                for (int32_t q = 0; q < D; ++q) gpx[q] = gF[(int64_t)q * HW + pix];
            loss += backward_pixel(rc, P, px, py, key_rec + s, (int64_t)e - s, g3, gD[pix], gA[pix], grec,
                                   gF ? gpx.data() : nullptr);
        }
    return loss;
}

// Brute force (the plain definition): per pixel, scan ALL projected records,
// keep those whose tile rectangle contains the pixel's tile, order them by
// (depth_bits, gid) with a plain comparator, composite.
void oracle_brute_force(const or_view* V, const or_params* P, int64_t cnt, const float* u,
                        const float* v, const float* conic, const float* opac, const float* rgb,
                        const float* z, const int32_t* gid, const int32_t* rect, const float* feat,
                        int32_t D, float* out_rgb, float* out_depth, float* out_alpha,
                        float* out_feat, uint8_t* flags, double* contrib /*[cnt] or NULL*/,
                        float* a_err /*[H][W] or NULL*/) {
    Records rc{u, v, conic, opac, rgb, z, gid, feat, D};
    const int32_t W = V->width, H = V->height;
    const int64_t HW = (int64_t)W * H;
    PixelOut o;
    std::vector<uint32_t> list;
    for (int32_t py = 0; py < H; ++py)
        for (int32_t px = 0; px < W; ++px) {
            const int32_t tx = px / 16, ty = py / 16;
            list.clear();
            for (int64_t i = 0; i < cnt; ++i)
                if (rect[i * 4 + 0] <= tx && tx <= rect[i * 4 + 1] && rect[i * 4 + 2] <= ty &&
                    ty <= rect[i * 4 + 3])
                    list.push_back((uint32_t)i);
            std::sort(list.begin(), list.end(), [&](uint32_t a, uint32_t b) {
                const uint32_t da = float_bits(z[a]), db = float_bits(z[b]);
                if (da != db) return da < db;
                return gid[a] < gid[b];
            });
            composite_pixel(rc, P, px, py, list.data(), (int64_t)list.size(), o, contrib);
            store_pixel(o, HW, (int64_t)py * W + px, out_rgb, out_depth, out_alpha, out_feat, flags, D, a_err);
        }
}

// ---------------------------------------------------------------------------
// N1: render-visibility check with projection filtering and
// significance scoring, for one view.
//   Alg. 1: M^r[j] = render-gradient visibility, read
//     as the forward criterion contrib[j] > eps, contrib[j] = sum over pixels of
//     the blend weight w of Gaussian j (O12); M^i = 0 <= U < W and 0 <= V < H
//     (Alg. 1 l.17); M = M^i and M^r; (U', V') = (U, V)[:, M].
//   Eq. 4: S(G_i) = cos(F_G, F^t(U', V')), the target map sampled at
//     the nearest feature cell (reading Q27: cell = floor((U+0.5)/s)).
//   Eq. 5: S(G) = sum over views; Eq. 6: S(g_j) = S(G_j)/M,
//     M = number of views in which g_j is visible (formed by the caller).
// cos of a zero vector is 0 (reading Q28).  fp64.
// ---------------------------------------------------------------------------
void oracle_visibility_score(const or_view* V, int64_t cnt, const float* u, const float* v,
                             const int32_t* gid, const double* contrib, double eps, const float* feat,
                             int32_t D, const float* fmap /*[D][H'][W'] or NULL*/, int32_t stride,
                             uint8_t* visible /*[cnt]*/, double* score_sum /*[N]*/,
                             int64_t* count /*[N]*/) {
    const int32_t Wf = (V->width + stride - 1) / stride, Hf = (V->height + stride - 1) / stride;
    for (int64_t i = 0; i < cnt; ++i) {
        const bool mi = u[i] >= 0.0f && u[i] < (float)V->width && v[i] >= 0.0f && v[i] < (float)V->height;
        const bool mr = contrib[i] > eps;
        visible[i] = (uint8_t)(mi && mr);
        if (!visible[i]) continue;
        count[gid[i]] += 1;
        if (fmap == nullptr || D == 0) continue;
        int32_t cx = (int32_t)std::floor(((double)u[i] + 0.5) / stride);
        int32_t cy = (int32_t)std::floor(((double)v[i] + 0.5) / stride);
        cx = std::min(std::max(cx, 0), Wf - 1);
        cy = std::min(std::max(cy, 0), Hf - 1);
        const float* f = feat + (int64_t)gid[i] * D;
        double dot = 0.0, nf = 0.0, nt = 0.0;
        for (int32_t c = 0; c < D; ++c) {
            const double t = fmap[((int64_t)c * Hf + cy) * Wf + cx];
            dot += (double)f[c] * t;
            nf += (double)f[c] * f[c];
            nt += t * t;
        }
        const double cs = (nf > 0.0 && nt > 0.0) ? dot / (std::sqrt(nf) * std::sqrt(nt)) : 0.0;
        score_sum[gid[i]] += cs;
    }
}

// ---------------------------------------------------------------------------
// O13: back-projection.  valid iff A >= a_min (fp32 compare) and Dz/A > 0;
// zbar = Dz/A; X = R^T(((px - cx)/fx zbar, (py - cy)/fy zbar, zbar) - t)  (fp64).
// flags bit 2 (value 4) marks |A - a_min| <= a_err[p], the O14 (c) bound on the
// kernel's deviation of A (Q20); a_err = NULL means the kernel back-projects the
// very same A (no band).
// ---------------------------------------------------------------------------
void oracle_backproject(const or_view* V, const float* depth, const float* alpha, float a_min,
                        float* xyz /*[3][H][W]*/, uint8_t* valid, uint8_t* flags, const float* a_err) {
    const int32_t W = V->width, H = V->height;
    const int64_t HW = (int64_t)W * H;
    const float* R = V->R;
    for (int32_t py = 0; py < H; ++py)
        for (int32_t px = 0; px < W; ++px) {
            const int64_t p = (int64_t)py * W + px;
            const float A = alpha[p];
            if (a_err && std::fabs((double)A - (double)a_min) <= (double)a_err[p]) flags[p] |= 4;
            const double zbar = (double)depth[p] / (double)A;
            if (!(A >= a_min) || !(zbar > 0.0)) {
                xyz[p] = xyz[HW + p] = xyz[2 * HW + p] = 0.0f;
                valid[p] = 0;
                continue;
            }
            const double c0 = ((double)px - V->cx) / V->fx * zbar - V->t[0];
            const double c1 = ((double)py - V->cy) / V->fy * zbar - V->t[1];
            const double c2 = zbar - V->t[2];
            for (int k = 0; k < 3; ++k)
                xyz[k * HW + p] = (float)((double)R[0 * 3 + k] * c0 + (double)R[1 * 3 + k] * c1 +
                                          (double)R[2 * 3 + k] * c2);
            valid[p] = 1;
        }
}

}  // extern "C"
