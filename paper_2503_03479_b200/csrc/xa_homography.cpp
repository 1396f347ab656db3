// xa_homography.cpp — geometric verification of the fine stage and the
// evaluation harness: normalised-DLT homography
// and 4-point RANSAC (proj/include/xaffine/homography.hpp:27-39,
// proj/src/homography.cpp). Host code: RANSAC is sequential and seeded and
// stays outside the timed hot path.
//
// Same algorithm, order of operations and random stream as the reference:
// Hartley normalisation (centroid, mean distance -> sqrt 2), the 2n x 9 DLT
// system, its right singular vector of the smallest singular value, the
// denormalised model scaled to h22 = 1; RANSAC draws samples with
// std::mt19937_64(seed) + std::uniform_int_distribution<int>(0, n-1)
// (rejecting duplicates), skips samples with three collinear points on either
// side, keeps the largest symmetric-transfer consensus, shrinks the iteration
// bound adaptively and refits on all inliers. The reference takes the SVD from
// Eigen (absent in this image); here a one-sided Jacobi SVD in double gives
// the same null vector up to rounding, so models agree to ~1e-12 and inlier
// sets agree except for points within rounding of the threshold.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <random>
#include <string>
#include <vector>

#include "../../include/xaffine_b200.h"
#include "xa_geometry.h"

namespace xa {
int host_error(int code, const std::string& msg);
}

namespace {

using xa::Mat3;

struct Pt {
    double x1, y1, x2, y2;
};

struct HomFail {
    int code;
    std::string msg;
};

Mat3 mat_translation(double tx, double ty) { return xa::mat_shift(tx, ty); }

void normalizing_transforms(const std::vector<Pt>& pts, Mat3& t1, Mat3& t2) {  // homography.cpp:17-44
    double cx1 = 0, cy1 = 0, cx2 = 0, cy2 = 0;
    for (const Pt& p : pts) {
        cx1 += p.x1;
        cy1 += p.y1;
        cx2 += p.x2;
        cy2 += p.y2;
    }
    const double n = static_cast<double>(pts.size());
    cx1 /= n;
    cy1 /= n;
    cx2 /= n;
    cy2 /= n;
    double d1 = 0, d2 = 0;
    for (const Pt& p : pts) {
        d1 += std::hypot(p.x1 - cx1, p.y1 - cy1);
        d2 += std::hypot(p.x2 - cx2, p.y2 - cy2);
    }
    d1 /= n;
    d2 /= n;
    const double s1 = (d1 > 1e-12) ? std::sqrt(2.0) / d1 : 1.0;
    const double s2 = (d2 > 1e-12) ? std::sqrt(2.0) / d2 : 1.0;
    t1 = xa::mat_scale(s1) * mat_translation(-cx1, -cy1);
    t2 = xa::mat_scale(s2) * mat_translation(-cx2, -cy2);
}

// Right singular vector of the smallest singular value of A (rows x 9,
// row-major), by one-sided (Hestenes) Jacobi orthogonalisation of A's columns.
void smallest_right_singular_vector(std::vector<double> a, int rows, double out[9]) {
    double v[81] = {0};
    for (int i = 0; i < 9; ++i) v[i * 9 + i] = 1.0;
    for (int sweep = 0; sweep < 80; ++sweep) {
        bool rotated = false;
        for (int p = 0; p < 8; ++p)
            for (int q = p + 1; q < 9; ++q) {
                double al = 0, be = 0, ga = 0;
                for (int r = 0; r < rows; ++r) {
                    const double x = a[r * 9 + p], y = a[r * 9 + q];
                    al += x * x;
                    be += y * y;
                    ga += x * y;
                }
                if (ga == 0.0 || std::abs(ga) <= 1e-15 * std::sqrt(al * be)) continue;
                rotated = true;
                const double zeta = (be - al) / (2.0 * ga);
                const double t = (zeta >= 0 ? 1.0 : -1.0) / (std::abs(zeta) + std::sqrt(1.0 + zeta * zeta));
                const double c = 1.0 / std::sqrt(1.0 + t * t), s = c * t;
                for (int r = 0; r < rows; ++r) {
                    const double x = a[r * 9 + p], y = a[r * 9 + q];
                    a[r * 9 + p] = c * x - s * y;
                    a[r * 9 + q] = s * x + c * y;
                }
                for (int r = 0; r < 9; ++r) {
                    const double x = v[r * 9 + p], y = v[r * 9 + q];
                    v[r * 9 + p] = c * x - s * y;
                    v[r * 9 + q] = s * x + c * y;
                }
            }
        if (!rotated) break;
    }
    int best = 0;
    double bn = INFINITY;
    for (int j = 0; j < 9; ++j) {
        double nn = 0;
        for (int r = 0; r < rows; ++r) nn += a[r * 9 + j] * a[r * 9 + j];
        if (nn < bn) {
            bn = nn;
            best = j;
        }
    }
    for (int i = 0; i < 9; ++i) out[i] = v[i * 9 + best];
}

Mat3 fit_dlt(const std::vector<Pt>& pts) {  // homography.cpp:79-101
    if (pts.size() < 4) throw HomFail{XA_EHOMOGRAPHY, "homography fit needs at least 4 points"};
    Mat3 t1, t2;
    normalizing_transforms(pts, t1, t2);
    const int rows = 2 * (int)pts.size();
    std::vector<double> a((size_t)rows * 9);
    for (size_t i = 0; i < pts.size(); ++i) {
        double x1, y1, x2, y2;
        xa::map_pt_h(t1, pts[i].x1, pts[i].y1, x1, y1);
        xa::map_pt_h(t2, pts[i].x2, pts[i].y2, x2, y2);
        const double r0[9] = {-x1, -y1, -1, 0, 0, 0, x2 * x1, x2 * y1, x2};
        const double r1[9] = {0, 0, 0, -x1, -y1, -1, y2 * x1, y2 * y1, y2};
        std::copy(r0, r0 + 9, &a[(2 * i) * 9]);
        std::copy(r1, r1 + 9, &a[(2 * i + 1) * 9]);
    }
    Mat3 hn;
    smallest_right_singular_vector(std::move(a), rows, hn.m);
    Mat3 t2i;
    if (!xa::mat_inv(t2, t2i)) throw HomFail{XA_ESINGULAR, "invert: singular matrix"};
    Mat3 h = t2i * hn * t1;
    if (std::abs(h.m[8]) > 1e-12) {
        const double w = h.m[8];
        for (double& v : h.m) v /= w;
    }
    return h;
}

double transfer_error(const Mat3& h, const Mat3& hi, const Pt& p) {  // homography.cpp:46-51
    double fx, fy, bx, by;
    xa::map_pt_proj(h, p.x1, p.y1, fx, fy);
    xa::map_pt_proj(hi, p.x2, p.y2, bx, by);
    return std::max(std::hypot(fx - p.x2, fy - p.y2), std::hypot(bx - p.x1, by - p.y1));
}

bool three_collinear(const Pt* s[4], bool second) {  // homography.cpp:53-74
    for (int a = 0; a < 2; ++a)
        for (int b = a + 1; b < 3; ++b)
            for (int c = b + 1; c < 4; ++c) {
                const double x1 = second ? s[a]->x2 : s[a]->x1, y1 = second ? s[a]->y2 : s[a]->y1;
                const double x2 = second ? s[b]->x2 : s[b]->x1, y2 = second ? s[b]->y2 : s[b]->y1;
                const double x3 = second ? s[c]->x2 : s[c]->x1, y3 = second ? s[c]->y2 : s[c]->y1;
                const double cross = (x2 - x1) * (y3 - y1) - (y2 - y1) * (x3 - x1);
                const double len = std::hypot(x2 - x1, y2 - y1) * std::hypot(x3 - x1, y3 - y1);
                if (std::abs(cross) < 1e-6 * std::max(len, 1.0)) return true;
            }
    return false;
}

std::vector<Pt> as_points(const double* pts, int n) {
    std::vector<Pt> v((size_t)std::max(n, 0));
    for (int i = 0; i < n; ++i) v[i] = {pts[4 * i], pts[4 * i + 1], pts[4 * i + 2], pts[4 * i + 3]};
    return v;
}

}  // namespace

extern "C" {

int xa_fit_homography_dlt(const double* pts, int n, double h[9]) {
    try {
        const Mat3 r = fit_dlt(as_points(pts, n));
        std::copy(r.m, r.m + 9, h);
        return XA_OK;
    } catch (const HomFail& e) {
        return xa::host_error(e.code, e.msg);
    }
}

int xa_estimate_homography_ransac(const double* pts_in, int n, double threshold, int max_iters,
                                  double confidence, uint64_t seed, double h[9], int32_t* inliers,
                                  int cap, int* n_inliers) {
    *n_inliers = 0;
    try {
        if (n < 4) throw HomFail{XA_EHOMOGRAPHY, "RANSAC needs at least 4 correspondences"};
        const std::vector<Pt> pts = as_points(pts_in, n);
        std::mt19937_64 rng(seed);
        std::uniform_int_distribution<int> pick(0, n - 1);
        std::vector<int> best;
        int iters = max_iters;
        for (int it = 0; it < iters; ++it) {  // homography.cpp:108-147
            int idx[4];
            idx[0] = pick(rng);
            for (int k = 1; k < 4; ++k) {
                bool dup;
                do {
                    idx[k] = pick(rng);
                    dup = false;
                    for (int j = 0; j < k; ++j) dup |= (idx[j] == idx[k]);
                } while (dup);
            }
            const Pt* s[4] = {&pts[idx[0]], &pts[idx[1]], &pts[idx[2]], &pts[idx[3]]};
            if (three_collinear(s, false) || three_collinear(s, true)) continue;
            Mat3 m, mi;
            try {
                m = fit_dlt({*s[0], *s[1], *s[2], *s[3]});
            } catch (const HomFail& e) {
                if (e.code == XA_ESINGULAR) continue;  // the reference skips GeometryError
                throw;
            }
            if (!xa::mat_inv(m, mi)) continue;
            std::vector<int> cur;
            for (int i = 0; i < n; ++i)
                if (transfer_error(m, mi, pts[i]) < threshold) cur.push_back(i);
            if (cur.size() > best.size()) {
                best = std::move(cur);
                const double w = static_cast<double>(best.size()) / n;
                const double p_out = 1.0 - w * w * w * w;
                if (p_out < 1e-12) {
                    iters = it + 1;
                } else if (p_out < 1.0) {
                    const double need = std::log(1.0 - confidence) / std::log(p_out);
                    iters = std::min(iters, static_cast<int>(std::ceil(need)));
                }
            }
        }
        if (best.size() < 4) throw HomFail{XA_EHOMOGRAPHY, "no consensus"};
        std::vector<Pt> support;
        support.reserve(best.size());
        for (int i : best) support.push_back(pts[i]);
        const Mat3 r = fit_dlt(support);
        Mat3 ri;
        if (!xa::mat_inv(r, ri)) throw HomFail{XA_ESINGULAR, "invert: singular matrix"};
        std::vector<int> fin;
        for (int i = 0; i < n; ++i)
            if (transfer_error(r, ri, pts[i]) < threshold) fin.push_back(i);
        if (fin.size() < 4) fin = best;
        std::copy(r.m, r.m + 9, h);
        *n_inliers = (int)fin.size();
        if ((int)fin.size() > cap) return xa::host_error(XA_ECAPACITY, "RANSAC: inlier capacity");
        std::copy(fin.begin(), fin.end(), inliers);
        return XA_OK;
    } catch (const HomFail& e) {
        return xa::host_error(e.code, e.msg);
    }
}

}  // extern "C"
