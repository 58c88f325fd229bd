// mapman.cpp — NEXT-4 of SURVEY §8(f), on the host: the map merge gate
// (Eqs. 4-5) and the scalar vertical-drift Kalman filter (Eqs.
// 6-10), applied to the plane table of the hot path (one plane
// per region stands in for the paper's polygon, Q30-Q34).  The
// work is sequential, a few dozen flops per plane and pose-dependent: it
// stays on the CPU (SURVEY: "adds no GPU value").
#include <math.h>
#include <stdint.h>

#include "../../include/pmap.h"

namespace {

double angle_between(const double a[3], const double b[3]) {
    const double d = a[0] * b[0] + a[1] * b[1] + a[2] * b[2];
    const double na = sqrt(a[0] * a[0] + a[1] * a[1] + a[2] * a[2]);
    const double nb = sqrt(b[0] * b[0] + b[1] * b[1] + b[2] * b[2]);
    double c = fabs(d) / (na * nb);
    if (c > 1.0) c = 1.0;
    return acos(c);
}

}  // namespace

extern "C" {

PM_API double pm_drift_kalman_step(pm_drift_filter* f, double z, double sigma_p, double sigma_m) {
    if (!f) return NAN;
    const double x_pred = f->x;                       // Eq. 6
    const double P_pred = f->P + sigma_p;             // Eq. 7
    const double K = P_pred / (P_pred + sigma_m);     // Eq. 8
    f->x = x_pred + K * (z - x_pred);                 // Eq. 9
    f->P = (1.0 - K) * P_pred;                        // Eq. 10
    return K;
}

PM_API int32_t pm_merge_gate(double z_new, double z_map, double drift_tol, double* dz_out) {
    const double dz = fabs(z_new - z_map);            // Eq. 4
    if (dz_out) *dz_out = dz;
    return dz <= drift_tol ? 1 : 0;                   // Eq. 5
}

PM_API pm_status pm_plane_map_merge_frame(pm_map_plane* map, int32_t* map_count, int32_t map_capacity,
                                          const pm_plane* frame, int32_t n_planes, const double pose[16],
                                          pm_drift_filter* filter, const pm_map_params* prm, int32_t* match_out,
                                          double* z_k_out) {
    if (!map_count || !pose || !filter || !prm || n_planes < 0 || (n_planes > 0 && !frame) || *map_count < 0 ||
        *map_count > map_capacity || (*map_count > 0 && !map))
        return PM_ERR_INVALID_ARGUMENT;
    if (!(prm->drift_tol >= 0.0) || !(prm->normal_tol >= 0.0) || !(prm->xy_radius >= 0.0) ||
        !(prm->sigma_p >= 0.0) || !(prm->sigma_m >= 0.0))
        return PM_ERR_INVALID_ARGUMENT;
    const int32_t m0 = *map_count;
    // (1)-(2): OK planes to the world frame, minus the current drift estimate
    struct Inc { double n[3], c[3], w; int ok; int match; };
    Inc stack_buf[256];
    Inc* inc = n_planes <= 256 ? stack_buf : new Inc[n_planes];
    int32_t inserts = 0;
    for (int32_t i = 0; i < n_planes; ++i) {
        Inc& p = inc[i];
        p.ok = frame[i].status == PM_PLANE_OK;
        p.match = -1;
        if (!p.ok) continue;
        for (int r = 0; r < 3; ++r) {
            p.n[r] = pose[4 * r] * frame[i].n[0] + pose[4 * r + 1] * frame[i].n[1] + pose[4 * r + 2] * frame[i].n[2];
            p.c[r] = pose[4 * r] * frame[i].centroid[0] + pose[4 * r + 1] * frame[i].centroid[1] +
                     pose[4 * r + 2] * frame[i].centroid[2] + pose[4 * r + 3];
        }
        p.c[2] -= filter->x;
        p.w = (double)frame[i].inliers;
        // (3): gate against the map as it was before this frame
        int best = -1;
        double bd = 0.0;
        for (int32_t j = 0; j < m0; ++j) {
            const pm_map_plane& m = map[j];
            if (angle_between(p.n, m.n) > prm->normal_tol) continue;
            const double dxy = hypot(p.c[0] - m.c[0], p.c[1] - m.c[1]);
            if (dxy > prm->xy_radius) continue;
            if (!pm_merge_gate(p.c[2], m.c[2], prm->drift_tol, nullptr)) continue;
            if (best < 0 || dxy < bd) { best = j; bd = dxy; }
        }
        p.match = best;
        if (best < 0) ++inserts;
    }
    if (m0 + inserts > map_capacity) {
        if (inc != stack_buf) delete[] inc;
        return PM_ERR_WORKSPACE;
    }
    // (4): drift measurement z_k = mean signed residual + x, Eqs. 6-10
    double sum = 0.0;
    int32_t nres = 0;
    for (int32_t i = 0; i < n_planes; ++i)
        if (inc[i].ok && inc[i].match >= 0) { sum += inc[i].c[2] - map[inc[i].match].c[2]; ++nres; }
    double zk = NAN;
    if (nres > 0) {
        zk = sum / nres + filter->x;
        const double x_old = filter->x;
        pm_drift_kalman_step(filter, zk, prm->sigma_p, prm->sigma_m);
        for (int32_t i = 0; i < n_planes; ++i)
            if (inc[i].ok) inc[i].c[2] -= (filter->x - x_old);
    }
    // (5): merge matched pairs (inlier-weighted), insert the rest in frame order
    int32_t cnt = m0;
    for (int32_t i = 0; i < n_planes; ++i) {
        Inc& p = inc[i];
        if (match_out) match_out[i] = p.ok ? p.match : -1;
        if (!p.ok) continue;
        if (p.match < 0) {
            pm_map_plane& q = map[cnt++];
            for (int r = 0; r < 3; ++r) { q.n[r] = p.n[r]; q.c[r] = p.c[r]; }
            q.w = p.w;
            q.n_obs = 1;
            q.pad = 0;
            continue;
        }
        pm_map_plane& m = map[p.match];
        const double s = (p.n[0] * m.n[0] + p.n[1] * m.n[1] + p.n[2] * m.n[2]) >= 0.0 ? 1.0 : -1.0;
        const double wa = m.w, wb = p.w;
        double nn[3];
        for (int r = 0; r < 3; ++r) nn[r] = wa * m.n[r] + wb * s * p.n[r];
        const double L = sqrt(nn[0] * nn[0] + nn[1] * nn[1] + nn[2] * nn[2]);
        for (int r = 0; r < 3; ++r) {
            m.n[r] = nn[r] / L;
            m.c[r] = (wa * m.c[r] + wb * p.c[r]) / (wa + wb);
        }
        m.w = wa + wb;
        m.n_obs += 1;
    }
    *map_count = cnt;
    if (z_k_out) *z_k_out = zk;
    if (inc != stack_buf) delete[] inc;
    return PM_OK;
}

}  // extern "C"
