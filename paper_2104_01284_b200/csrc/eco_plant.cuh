// eco_plant.cuh — device restatement of the P0 mild-hybrid plant and the
// grid primitives of the reference (_kernels.py:60-414, cited K:line).
//
// Everything here is IEEE double.  The library is compiled with -fmad=false,
// so every a*b+c below rounds twice exactly like numba's LLVM output (the
// reference jits without fastmath, K:1-7); sqrt and '/' are IEEE-rounded in
// CUDA double.  cos/sin(grade) come from the host (libm), because CUDA's
// cos/sin are not correctly rounded.
#pragma once

#include <cstdint>
#include "../../include/eco_b200.h"

namespace eco {

constexpr double kGravity = 9.81;
constexpr double kWeightSnap = 1e-12;   // K:281

enum Feas : int { kFeasOk = 0, kFeasTorque = 1, kFeasAccel = 2, kFeasNoMotion = 3, kFeasBattery = 6 };

// np.searchsorted(a, x, 'left'): number of entries strictly below x.
__device__ __forceinline__ int searchsorted_left(const double* a, int n, double x) {
    int c = 0;
    for (int i = 0; i < n; ++i) c += (a[i] < x);
    return c;
}

// K:60-70
__device__ __forceinline__ double interp1_clamped(const double* xa, const double* y, int n, double x) {
    if (x <= xa[0]) return y[0];
    if (x >= xa[n - 1]) return y[n - 1];
    const int i = searchsorted_left(xa, n, x) - 1;
    const double w = (x - xa[i]) / (xa[i + 1] - xa[i]);
    return y[i] + w * (y[i + 1] - y[i]);
}

// K:73-102 (row-major (x, y) map; y-blend inside, then x)
__device__ __forceinline__ double interp2_clamped(const double* xa, int nx, const double* ya, int ny,
                                                  const double* vals, double x, double y) {
    int ix, iy;
    double wx, wy;
    if (x <= xa[0]) { ix = 0; wx = 0.0; }
    else if (x >= xa[nx - 1]) { ix = nx - 2; wx = 1.0; }
    else { ix = searchsorted_left(xa, nx, x) - 1; wx = (x - xa[ix]) / (xa[ix + 1] - xa[ix]); }
    if (y <= ya[0]) { iy = 0; wy = 0.0; }
    else if (y >= ya[ny - 1]) { iy = ny - 2; wy = 1.0; }
    else { iy = searchsorted_left(ya, ny, y) - 1; wy = (y - ya[iy]) / (ya[iy + 1] - ya[iy]); }
    const double v00 = vals[ix * ny + iy], v01 = vals[ix * ny + iy + 1];
    const double v10 = vals[(ix + 1) * ny + iy], v11 = vals[(ix + 1) * ny + iy + 1];
    const double lo = v00 + wy * (v01 - v00);
    const double hi = v10 + wy * (v11 - v10);
    return lo + wx * (hi - lo);
}

// K:109-131: gear, engine and BSG shaft speeds
struct Drive { int gear; double w_eng, w_bsg; };

__device__ __forceinline__ Drive drivetrain(const EcoPlant& p, double v) {
    Drive d;
    int g = 0;
    for (int i = 0; i < p.n_gears - 1; ++i)
        if (v > p.shift_v[i]) g = i + 1;
    double w = v / p.wheel_radius * p.final_drive * p.gear_ratios[g];
    if (w < p.idle_speed) w = p.idle_speed;
    d.gear = g;
    d.w_eng = w;
    d.w_bsg = w * p.belt_ratio;
    return d;
}

// K:134-142 (sum left to right)
__device__ __forceinline__ double road_load(const EcoPlant& p, double v, double cos_g, double sin_g) {
    return p.c0 * cos_g + p.c1 * v + p.c2 * v * v + p.mass * kGravity * sin_g;
}

// K:145-158
__device__ __forceinline__ double tractive_force(const EcoPlant& p, int gear, double te, double tb) {
    const double crank = te + tb * p.belt_ratio;
    const double ratio = p.gear_ratios[gear] * p.final_drive;
    const double eff = p.gear_eff[gear];
    const double axle = crank * ratio;
    if (axle >= 0.0) return axle * eff / p.wheel_radius;
    return axle / eff / p.wheel_radius;
}

// K:161-166
__device__ __forceinline__ double fuel_rate(const EcoPlant& p, double w_eng, double te) {
    if (te <= 0.0) return 0.0;
    return interp2_clamped(p.fuel_w, p.n_fuel_w, p.fuel_t, p.n_fuel_t, p.fuel_vals, w_eng, te);
}

// K:169-180
__device__ __forceinline__ double bsg_power(const EcoPlant& p, double w_bsg, double tb) {
    if (tb == 0.0) return 0.0;
    const double mech = tb * w_bsg;
    const double eff = interp2_clamped(p.eff_w, p.n_eff_w, p.eff_t, p.n_eff_t, p.eff_vals, w_bsg, fabs(tb));
    if (tb > 0.0) return mech / eff;
    return mech * eff;
}

// K:183-196: returns ok, current in *cur
__device__ __forceinline__ bool battery_current(const EcoPlant& p, double p_bat, double soc, double* cur) {
    if (p_bat == 0.0) { *cur = 0.0; return true; }
    const double voc = interp1_clamped(p.voc_soc, p.voc_v, p.n_voc, soc);
    const double disc = voc * voc - 4.0 * p.r0 * p_bat;
    if (disc < 0.0) { *cur = 0.0; return false; }
    *cur = (voc - sqrt(disc)) / (2.0 * p.r0);
    return true;
}

// K:210-222: speed-only quantities of a step
struct StepPre { Drive d; double te_lo, te_hi, tb_lo, tb_hi, f_road; };

__device__ __forceinline__ StepPre step_pre(const EcoPlant& p, double v, double cos_g, double sin_g) {
    StepPre q;
    q.d = drivetrain(p, v);
    q.te_lo = interp1_clamped(p.eng_w, p.eng_tmin, p.n_eng, q.d.w_eng);
    q.te_hi = interp1_clamped(p.eng_w, p.eng_tmax, p.n_eng, q.d.w_eng);
    q.tb_lo = interp1_clamped(p.bsg_w, p.bsg_tmin, p.n_bsg, q.d.w_bsg);
    q.tb_hi = interp1_clamped(p.bsg_w, p.bsg_tmax, p.n_bsg, q.d.w_bsg);
    q.f_road = road_load(p, v, cos_g, sin_g);
    return q;
}

// K:225-251: action-dependent remainder of a step
struct StepOut { int feas; bool clamped; double v_next, v_bar, dt_move, accel, mf, p_bat; };

__device__ __forceinline__ StepOut step_eval_pre(const EcoPlant& p, double v, double te, double tb,
                                                 double dd, double a_min, double a_max, double brake,
                                                 const StepPre& q) {
    StepOut o{};
    if (te < q.te_lo || te > q.te_hi || tb < q.tb_lo || tb > q.tb_hi) { o.feas = kFeasTorque; return o; }
    const double f_tr = tractive_force(p, q.d.gear, te, tb);
    const double rad = v * v + 2.0 * dd * (f_tr - q.f_road - brake) / p.mass;
    o.clamped = rad < 0.0;
    o.v_next = o.clamped ? 0.0 : sqrt(rad);
    o.v_bar = 0.5 * (v + o.v_next);
    if (o.v_bar <= 0.0) { o.feas = kFeasNoMotion; return o; }
    o.accel = (o.v_next * o.v_next - v * v) / (2.0 * dd);
    if (o.accel < a_min || o.accel > a_max) { o.feas = kFeasAccel; return o; }
    o.dt_move = dd / o.v_bar;
    o.mf = fuel_rate(p, q.d.w_eng, te);
    o.p_bat = bsg_power(p, q.d.w_bsg, tb);
    o.feas = (o.p_bat > p.p_bat_max) ? kFeasBattery : kFeasOk;
    return o;
}

// K:284-306: uniform-axis cell (lo, hi, w); returns ok.  int64 floor like numba.
__device__ __forceinline__ bool locate_uniform(double x, double x0, double dx, int n, int* lo, int* hi, double* w) {
    const double f = (x - x0) / dx;
    const double fl = floor(f);
    *lo = 0; *hi = 0; *w = 0.0;
    if (!(fl > -4.0e18 && fl < 4.0e18)) return false;
    long long i = (long long)fl;
    double ww = f - (double)i;
    if (ww < kWeightSnap) ww = 0.0;
    else if (ww > 1.0 - kWeightSnap) { i += 1; ww = 0.0; }
    if (i < 0 || i > n - 1) return false;
    if (ww == 0.0) { *lo = (int)i; *hi = (int)i; return true; }
    if (i == n - 1) return false;
    *lo = (int)i; *hi = (int)i + 1; *w = ww;
    return true;
}

// K:309-322 (shift saturates: any offset past the ladder is infeasible anyway)
__device__ __forceinline__ void tcell_shift(double dt_move, double dtg, int* zoff, double* wz) {
    const double d = dt_move / dtg;
    const double fl = floor(d);
    long long z = fl < 1.0e18 ? (long long)fl : (long long)1e18;
    double w = d - (double)z;
    if (w < kWeightSnap) w = 0.0;
    else if (w > 1.0 - kWeightSnap) { z += 1; w = 0.0; }
    *zoff = z > (1 << 30) ? (1 << 30) : (int)z;
    *wz = w;
}

// K:364-367
__device__ __forceinline__ double stage_cost(double mf, double dt, double gamma) {
    return (gamma * mf + (1.0 - gamma)) * dt;
}

// Python float % (Objects/floatobject.c float_rem): result carries the
// divisor's sign; route.py:69-70 relies on it for negative clocks.
__device__ __forceinline__ double py_mod(double a, double b) {
    double m = fmod(a, b);
    if (m != 0.0) {
        if ((b < 0.0) != (m < 0.0)) m += b;
    } else {
        m = copysign(0.0, b);
    }
    return m;
}

// SignalTiming.is_green / next_green_from (route.py:72-86)
__device__ __forceinline__ bool sig_is_green(double cycle, double offset, const double* win, int nwin, double t) {
    const double tau = py_mod(t - offset, cycle);
    for (int i = 0; i < nwin; ++i)
        if (win[2 * i] <= tau && tau < win[2 * i + 1]) return true;
    return false;
}

__device__ __forceinline__ double sig_next_green(double cycle, double offset, const double* win, int nwin, double t) {
    const double tau = py_mod(t - offset, cycle);
    double best = 0.0;
    for (int i = 0; i < nwin; ++i) {
        const double d = py_mod(win[2 * i] - tau, cycle);
        if (i == 0 || d < best) best = d;
    }
    return t + best;
}

}  // namespace eco
