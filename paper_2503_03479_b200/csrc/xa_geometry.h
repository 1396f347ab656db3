// xa_geometry.h — host-side view geometry, bit-identical to the reference's
// double arithmetic (compiled with -ffp-contract=off, source evaluation order).
//
// Reference: proj/src/geometry.cpp:9-112 (matrices, affine_from_params,
// simulation_from_params, invert, map_point, build_param_grid) and
// proj/src/warp.cpp:13-42 (center_adjusted, framing).
#pragma once

#include <cmath>
#include <string>
#include <vector>

namespace xa {

struct Mat3 {
    double m[9] = {1, 0, 0, 0, 1, 0, 0, 0, 1};
};

inline Mat3 mat_shift(double tx, double ty) {
    Mat3 r;
    r.m[2] = tx;
    r.m[5] = ty;
    return r;
}

inline Mat3 mat_rot(double a) {  // geometry.cpp:18-26
    Mat3 r;
    const double c = std::cos(a), s = std::sin(a);
    r.m[0] = c;
    r.m[1] = -s;
    r.m[3] = s;
    r.m[4] = c;
    return r;
}

inline Mat3 mat_scale(double s) {
    Mat3 r;
    r.m[0] = s;
    r.m[4] = s;
    return r;
}

inline Mat3 operator*(const Mat3& a, const Mat3& b) {  // geometry.cpp:35-44
    Mat3 r;
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) {
            double acc = 0;
            for (int k = 0; k < 3; ++k) acc += a.m[i * 3 + k] * b.m[k * 3 + j];
            r.m[i * 3 + j] = acc;
        }
    return r;
}

// T(tx,ty) * R(psi) * S(s) * diag(tilt_factor, 1) * R(phi) (geometry.cpp:42-58)
inline Mat3 compose_params(const double* p /* psi,t,phi,s,tx,ty */, bool simulate) {
    Mat3 tau;
    tau.m[0] = simulate ? 1.0 / p[1] : p[1];
    return mat_shift(p[4], p[5]) * mat_rot(p[0]) * mat_scale(p[3]) * tau * mat_rot(p[2]);
}

// Cofactor inverse (geometry.cpp:65-78); returns false when singular.
inline bool mat_inv(const Mat3& a, Mat3& r) {
    const double* m = a.m;
    const double det = m[0] * (m[4] * m[8] - m[5] * m[7]) - m[1] * (m[3] * m[8] - m[5] * m[6]) +
                       m[2] * (m[3] * m[7] - m[4] * m[6]);
    if (std::abs(det) < 1e-14) return false;
    r.m[0] = (m[4] * m[8] - m[5] * m[7]) / det;
    r.m[1] = (m[2] * m[7] - m[1] * m[8]) / det;
    r.m[2] = (m[1] * m[5] - m[2] * m[4]) / det;
    r.m[3] = (m[5] * m[6] - m[3] * m[8]) / det;
    r.m[4] = (m[0] * m[8] - m[2] * m[6]) / det;
    r.m[5] = (m[2] * m[3] - m[0] * m[5]) / det;
    r.m[6] = (m[3] * m[7] - m[4] * m[6]) / det;
    r.m[7] = (m[1] * m[6] - m[0] * m[7]) / det;
    r.m[8] = (m[0] * m[4] - m[1] * m[3]) / det;
    return true;
}

inline void map_pt_h(const Mat3& m, double x, double y, double& ox, double& oy) {
    ox = m.m[0] * x + m.m[1] * y + m.m[2];
    oy = m.m[3] * x + m.m[4] * y + m.m[5];
}

// Warp frame (warp.cpp:13-42, :92-95).
struct Frame {
    int W = 0, H = 0;
    double tx = 0, ty = 0;
    Mat3 forward, back;
};

// Returns 0, or -2 when a required inverse is singular.
inline int warp_frame(const Mat3& m, int w, int h, bool check_adj, Frame& f) {
    const Mat3 adj = mat_shift(-0.5, -0.5) * m * mat_shift(0.5, 0.5);
    Mat3 tmp;
    if (check_adj && !mat_inv(adj, tmp)) return -2;
    const double cx[4] = {0.0, double(w - 1), 0.0, double(w - 1)};
    const double cy[4] = {0.0, 0.0, double(h - 1), double(h - 1)};
    double minx = 1e30, miny = 1e30, maxx = -1e30, maxy = -1e30;
    for (int i = 0; i < 4; ++i) {
        double x, y;
        map_pt_h(adj, cx[i], cy[i], x, y);
        if (x < minx) minx = x;
        if (maxx < x) maxx = x;
        if (y < miny) miny = y;
        if (maxy < y) maxy = y;
    }
    f.tx = -std::floor(minx + 1e-9);
    f.ty = -std::floor(miny + 1e-9);
    f.W = static_cast<int>(std::ceil(maxx - 1e-9) + f.tx) + 1;
    f.H = static_cast<int>(std::ceil(maxy - 1e-9) + f.ty) + 1;
    f.forward = mat_shift(f.tx, f.ty) * adj;
    if (!mat_inv(f.forward, f.back)) return -2;
    return 0;
}

// map_point_projective (geometry.cpp:84-88)
inline void map_pt_proj(const Mat3& m, double x, double y, double& ox, double& oy) {
    const double w = m.m[6] * x + m.m[7] * y + m.m[8];
    ox = (m.m[0] * x + m.m[1] * y + m.m[2]) / w;
    oy = (m.m[3] * x + m.m[4] * y + m.m[5]) / w;
}

// synth_warp_case framing (eval.cpp:104-131). Returns 0, or the EvalError
// cases: 1 = a corner maps to w ~ 0, 2 = unbounded target, 3 = not invertible.
inline int synth_frame(const Mat3& h, int w, int hgt, Frame& f) {
    const Mat3 adj = mat_shift(-0.5, -0.5) * h * mat_shift(0.5, 0.5);
    const double cx[4] = {0.0, double(w - 1), 0.0, double(w - 1)};
    const double cy[4] = {0.0, 0.0, double(hgt - 1), double(hgt - 1)};
    double minx = 1e30, miny = 1e30, maxx = -1e30, maxy = -1e30;
    for (int i = 0; i < 4; ++i) {
        const double wq = adj.m[6] * cx[i] + adj.m[7] * cy[i] + adj.m[8];
        if (std::abs(wq) < 1e-9) return 1;
        double x, y;
        map_pt_proj(adj, cx[i], cy[i], x, y);
        minx = x < minx ? x : minx;  // std::min / std::max argument order
        maxx = maxx < x ? x : maxx;
        miny = y < miny ? y : miny;
        maxy = maxy < y ? y : maxy;
    }
    if (maxx - minx > 20000 || maxy - miny > 20000) return 2;
    f.tx = -std::floor(minx + 1e-9);
    f.ty = -std::floor(miny + 1e-9);
    f.W = static_cast<int>(std::ceil(maxx - 1e-9) + f.tx) + 1;
    f.H = static_cast<int>(std::ceil(maxy - 1e-9) + f.ty) + 1;
    f.forward = mat_shift(f.tx, f.ty) * adj;
    if (!mat_inv(f.forward, f.back)) return 3;
    return 0;
}

// build_param_grid (geometry.cpp:90-112): rows of (psi, t, phi, s, tx, ty).
inline std::vector<double> param_grid(double a, int n, double b_deg, double delta_s) {
    std::vector<double> out;
    for (int k = 0; k <= n; ++k) {
        const double t = std::pow(a, k);
        const double s = 1.0 + k * delta_s;
        if (k == 0) {
            out.insert(out.end(), {0.0, t, 0.0, s, 0.0, 0.0});
            continue;
        }
        const double step = b_deg / t;
        for (int j = 0; j * step < 180.0 - 1e-9; ++j)
            out.insert(out.end(), {0.0, t, j * step * M_PI / 180.0, s, 0.0, 0.0});
    }
    return out;
}

}  // namespace xa
