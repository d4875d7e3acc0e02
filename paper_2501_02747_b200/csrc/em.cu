// EM consumer of the path sets: ray_gains and
// channel_stats (src/em.cpp:194-277), one thread per path / per snapshot.
//
// Free-space amplitude over the unfolded length (or spherical spreading to
// the edge + the UTD spreading factor for a final diffraction), one Fresnel
// coefficient per reflection (incidence angle against the face normal,
// complex permittivity eps_r - j sigma / (2 pi f eps0)), and the
// Kouyoumjian-Pathak UTD wedge coefficient with transition-function smoothing
// (Fresnel-integral series / asymptotics, src/em.cpp:21-87) for a diffraction.
// The operation order follows the reference; transcendental functions are
// CUDA's (not glibc's), so parity is tolerance-based (relative 1e-9 in the
// tests), as SURVEY.md §8(f) anticipates.
#include <cmath>

#include "capi_internal.h"

namespace visrt {
namespace {

constexpr double kPi = 3.14159265358979323846;
constexpr double kEps0 = 8.8541878128e-12;
constexpr double kC = 299792458.0;

struct Cx {
    double re, im;
};
__device__ __forceinline__ Cx cx(double r, double i = 0.0) { return {r, i}; }
__device__ __forceinline__ Cx operator+(Cx a, Cx b) { return {a.re + b.re, a.im + b.im}; }
__device__ __forceinline__ Cx operator-(Cx a, Cx b) { return {a.re - b.re, a.im - b.im}; }
__device__ __forceinline__ Cx operator-(Cx a) { return {-a.re, -a.im}; }
__device__ __forceinline__ Cx operator*(Cx a, Cx b) {
    return {a.re * b.re - a.im * b.im, a.re * b.im + a.im * b.re};
}
__device__ __forceinline__ Cx operator*(Cx a, double s) { return {a.re * s, a.im * s}; }
__device__ __forceinline__ Cx operator*(double s, Cx a) { return {a.re * s, a.im * s}; }
__device__ __forceinline__ Cx operator/(Cx a, double s) { return {a.re / s, a.im / s}; }
__device__ __forceinline__ Cx operator/(Cx a, Cx b) {
    // Smith's algorithm (robust scaling)
    if (fabs(b.re) >= fabs(b.im)) {
        const double r = b.im / b.re, d = b.re + b.im * r;
        return {(a.re + a.im * r) / d, (a.im - a.re * r) / d};
    }
    const double r = b.re / b.im, d = b.re * r + b.im;
    return {(a.re * r + a.im) / d, (a.im * r - a.re) / d};
}
__device__ __forceinline__ double cabs(Cx a) { return hypot(a.re, a.im); }
__device__ __forceinline__ double cnorm(Cx a) { return a.re * a.re + a.im * a.im; }
__device__ __forceinline__ Cx cexp(Cx a) {
    const double e = exp(a.re);
    double s, c;
    sincos(a.im, &s, &c);
    return {e * c, e * s};
}
__device__ __forceinline__ Cx cpolar(double m, double ph) {
    double s, c;
    sincos(ph, &s, &c);
    return {m * c, m * s};
}
__device__ __forceinline__ Cx csqrt(Cx z) {   // principal branch, as std::sqrt
    if (z.re == 0.0 && z.im == 0.0) return {0.0, z.im};
    const double r = hypot(z.re, z.im);
    if (z.re >= 0.0) {
        const double t = sqrt(0.5 * (r + z.re));
        return {t, z.im / (2.0 * t)};
    }
    const double t = sqrt(0.5 * (r - z.re));
    return {fabs(z.im) / (2.0 * t), copysign(t, z.im)};
}
__device__ const Cx kJ = {0.0, 1.0};

struct V3 {
    double x, y, z;
};
__device__ __forceinline__ V3 sub3(V3 a, V3 b) { return {a.x - b.x, a.y - b.y, a.z - b.z}; }
__device__ __forceinline__ V3 add3(V3 a, V3 b) { return {a.x + b.x, a.y + b.y, a.z + b.z}; }
__device__ __forceinline__ V3 mul3(V3 a, double s) { return {a.x * s, a.y * s, a.z * s}; }
__device__ __forceinline__ double dot3(V3 a, V3 b) { return a.x * b.x + a.y * b.y + a.z * b.z; }
__device__ __forceinline__ double norm3(V3 a) { return sqrt(dot3(a, a)); }
__device__ __forceinline__ V3 unit3(V3 a) {   // normalized: v / n
    const double n = norm3(a);
    return {a.x / n, a.y / n, a.z / n};
}
__device__ __forceinline__ double clampd(double v, double lo, double hi) { return v < lo ? lo : (hi < v ? hi : v); }

// fresnel_reflection (src/em.cpp:104-118)
__device__ Cx fresnel(double theta, double eps_r, double sigma, double f, int tm) {
    const Cx eps = {eps_r, -sigma / (2.0 * kPi * f * kEps0)};
    const double ct = cos(theta), st = sin(theta);
    const Cx root = csqrt(eps - cx(st * st));
    if (!tm) return (cx(ct) - root) / (cx(ct) + root);
    return (root - eps * ct) / (root + eps * ct);
}

// fresnel_tail (src/em.cpp:21-46): integral of exp(-j t^2) from x to infinity
__device__ Cx fresnel_tail(double x) {
    const Cx full = cx(sqrt(2.0 * kPi) / 4.0, -sqrt(2.0 * kPi) / 4.0);
    if (x < 4.5) {
        Cx sum = cx(0.0);
        Cx term = cx(x);
        for (int k = 0; k < 120; ++k) {
            sum = sum + term / static_cast<double>(2 * k + 1);
            term = term * ((-kJ) * (x * x) / static_cast<double>(k + 1));
            if (cabs(term) < 1e-18 && k > 8) break;
        }
        return full - sum;
    }
    const Cx lead = cexp((-kJ) * (x * x)) / ((2.0 * kJ) * x);
    Cx sum = cx(1.0);
    Cx term = cx(1.0);
    for (int m = 1; m < 24; ++m) {
        term = term * (cx(-static_cast<double>(2 * m - 1)) / ((2.0 * kJ) * (x * x)));
        if (cabs(term) > 1.0) break;
        sum = sum + term;
        if (cabs(term) < 1e-18) break;
    }
    return lead * sum;
}

// transition_function (src/em.cpp:89-94)
__device__ Cx transition(double x) {
    if (x == 0) return cx(0.0);
    const double r = sqrt(x);
    return (2.0 * kJ) * r * cexp(kJ * x) * fresnel_tail(r);
}

// wedge_term (src/em.cpp:51-67)
__device__ Cx wedge_term(double n, double beta, double sign, double kL) {
    const double big_n = round((sign * kPi + beta) / (2.0 * n * kPi));
    const double c = cos((2.0 * n * kPi * big_n - beta) / 2.0);
    const double a = 2.0 * (c * c);
    const double arg = (kPi + sign * beta) / (2.0 * n);
    const double eps = kPi + sign * (beta - 2.0 * n * kPi * big_n);
    if (fabs(sin(arg)) < 1e-5) {
        const Cx e4 = cexp(kJ * (kPi / 4.0));
        return n * e4 * (cx(sqrt(2.0 * kPi * kL) * (eps >= 0 ? 1.0 : -1.0)) - (2.0 * kL * eps) * e4);
    }
    return (cos(arg) / sin(arg)) * transition(kL * a);
}

__device__ __forceinline__ double grazing_fold(double phi) {
    double gz = fmod(phi, kPi);
    if (gz < 0) gz += kPi;
    if (gz > kPi / 2.0) gz = kPi - gz;
    return gz;
}

struct EmArgs {
    DevScene s;
    long long npaths;
    const visrt_path* paths;
    const double* mat;        // [n][2] eps_r, sigma
    const double* edge_ab;    // [nedges][6]
    const int32_t* edge_faces;
    visrt_em_config cfg;
    double* amp;              // [npaths][2]
    double* delay;
    int32_t* err;             // first error code (1: degenerate wedge / grazing ray)
};

__global__ void __launch_bounds__(128) k_ray_gains(EmArgs a) {
    const DevScene& s = a.s;
    const double f = a.cfg.frequency;
    const double lambda = kC / f;
    const double k = 2.0 * kPi / lambda;
    const double gain = pow(10.0, a.cfg.tx_gain_dbi / 20.0) * pow(10.0, a.cfg.rx_gain_dbi / 20.0);
    for (long long q = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; q < a.npaths;
         q += static_cast<long long>(gridDim.x) * blockDim.x) {
        const visrt_path& p = a.paths[q];
        const bool diff = p.edge >= 0;
        const int npts = p.nrefl + 2 + (diff ? 1 : 0);
        auto pt = [&](int i) { return V3{p.points[3 * i], p.points[3 * i + 1], p.points[3 * i + 2]}; };
        const V3 rx = pt(npts - 1);
        Cx amp;
        if (!diff) {
            // free_space_gain (src/em.cpp:96-102)
            amp = cpolar(lambda / (4.0 * kPi * p.length), -2.0 * kPi * p.length / lambda);
        } else {
            const double s_d = norm3(sub3(pt(npts - 2), rx));
            const double s_i = p.length - s_d;
            const double mag = lambda / (4.0 * kPi) / sqrt(s_i * s_d * (s_i + s_d));
            amp = cpolar(mag, -k * p.length);
        }
        for (int i = 0; i < p.nrefl; ++i) {
            const int fc = p.faces[i];
            const V3 dir = unit3(sub3(pt(i + 1), pt(i)));
            const double* N = s.normal + 3 * static_cast<size_t>(fc);
            const double ct = clampd(fabs(dot3(dir, V3{N[0], N[1], N[2]})), 0.0, 1.0);
            const double theta = acos(ct);
            amp = amp * fresnel(fmin(theta, kPi / 2.0 - 1e-9), a.mat[2 * fc], a.mat[2 * fc + 1], f,
                                a.cfg.polarization);
        }
        if (diff) {
            // wedge_geometry (src/em.cpp:115-152)
            const double* E = a.edge_ab + 6 * static_cast<size_t>(p.edge);
            const int f0 = a.edge_faces[2 * p.edge], f1 = a.edge_faces[2 * p.edge + 1];
            const V3 ea{E[0], E[1], E[2]}, eb{E[3], E[4], E[5]};
            const V3 e = unit3(sub3(eb, ea));
            const double* N0 = s.normal + 3 * static_cast<size_t>(f0);
            const double* N1 = s.normal + 3 * static_cast<size_t>(f1);
            const V3 n0{N0[0], N0[1], N0[2]};
            const double dotn = clampd(dot3(n0, V3{N1[0], N1[1], N1[2]}), -1.0, 1.0);
            const double interior = kPi - acos(dotn);
            const double wn = (2.0 * kPi - interior) / kPi;
            const double* C0 = s.samples + (static_cast<size_t>(f0) * kMaxSamples + s.nv[f0]) * 3;   // centroid
            const V3 c0{C0[0], C0[1], C0[2]};
            const V3 foot = add3(ea, mul3(e, dot3(sub3(c0, ea), e)));
            V3 w0 = sub3(c0, foot);
            w0 = unit3(sub3(w0, mul3(e, dot3(w0, e))));
            auto azimuth = [&](V3 dir) {
                const V3 pp = sub3(dir, mul3(e, dot3(dir, e)));
                double phi = atan2(dot3(pp, n0), dot3(pp, w0));
                if (phi < 0) phi += 2.0 * kPi;
                return phi;
            };
            const V3 prev = pt(npts - 3), at = pt(npts - 2);
            const V3 si = sub3(at, prev), sd = sub3(rx, at);
            const double s_i = norm3(si), s_d = norm3(sd);
            const V3 shat = unit3(si);
            const double beta = acos(clampd(fabs(dot3(shat, e)), 0.0, 1.0));
            const double phi_i = azimuth(sub3(prev, at));
            const double phi_d = azimuth(sub3(rx, at));
            // utd_diffraction (src/em.cpp:154-192)
            const double sb = sin(beta);
            if (!(wn > 1.0) || wn > 2.0 + 1e-9 || s_i <= 0 || s_d <= 0 || sb <= 1e-9) {
                atomicCAS(a.err, 0, 1);
                amp = cx(0.0);
            } else {
                const double kk = 2.0 * kPi * f / kC;
                const double L = s_i * s_d / (s_i + s_d) * sb * sb;
                const double kL = kk * L;
                const double bm = phi_d - phi_i, bp = phi_d + phi_i;
                const double th0 = clampd(kPi / 2.0 - grazing_fold(phi_i), 0.0, kPi / 2.0 - 1e-9);
                const double thn = clampd(kPi / 2.0 - grazing_fold(wn * kPi - phi_d), 0.0, kPi / 2.0 - 1e-9);
                const Cx r0 = fresnel(th0, a.mat[2 * f0], a.mat[2 * f0 + 1], f, a.cfg.polarization);
                const Cx rn = fresnel(thn, a.mat[2 * f0], a.mat[2 * f0 + 1], f, a.cfg.polarization);
                const Cx pref = -cexp((-kJ) * (kPi / 4.0)) / (2.0 * wn * sqrt(2.0 * kPi * kk) * sb);
                const Cx d = pref * (wedge_term(wn, bm, +1.0, kL) + wedge_term(wn, bm, -1.0, kL) +
                                     rn * wedge_term(wn, bp, +1.0, kL) + r0 * wedge_term(wn, bp, -1.0, kL));
                amp = amp * d;
            }
        }
        amp = amp * gain;
        a.amp[2 * q] = amp.re;
        a.amp[2 * q + 1] = amp.im;
        a.delay[q] = p.length / kC;
    }
}

// channel_stats (src/em.cpp:209-235), one thread per snapshot
__global__ void k_channel_stats(long long nsnap, const long long* off, const double* amp, const double* delay,
                                int8_t* outage, double* loss, double* rms) {
    for (long long k = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; k < nsnap;
         k += static_cast<long long>(gridDim.x) * blockDim.x) {
        double power = 0.0, m1 = 0.0, m2 = 0.0;
        for (long long q = off[k]; q < off[k + 1]; ++q) {
            const double p = cnorm(Cx{amp[2 * q], amp[2 * q + 1]});
            power += p;
            m1 += p * delay[q];
            m2 += p * delay[q] * delay[q];
        }
        if (off[k + 1] == off[k] || power <= 0) {
            outage[k] = 1;
            loss[k] = INFINITY;
            rms[k] = 0.0;
            continue;
        }
        outage[k] = 0;
        loss[k] = -10.0 * log10(power);
        m1 /= power;
        m2 /= power;
        rms[k] = sqrt(fmax(0.0, m2 - m1 * m1));
    }
}

}  // namespace
}  // namespace visrt

using visrt::ck;

extern "C" int visrt_ray_gains(visrt_scene* sc, int64_t npaths, const visrt_path* paths, const double* face_material,
                               int32_t nedges, const double* edge_ab, const int32_t* edge_faces,
                               const visrt_em_config* cfg, double* amp, double* delay, visrt_stats* stats,
                               void* stream) {
    return visrt::capi_guard([&] {
        visrt::ScopedDevice dev(sc);
        if (!cfg || !face_material || (npaths > 0 && (!paths || !amp || !delay)))
            throw visrt::UsageError("null argument");
        if (!(cfg->frequency > 0)) throw visrt::VisError("frequency must be positive");   // EmError
        const visrt::DevScene& ds = visrt::scene_dev(sc);
        for (int64_t q = 0; q < npaths; ++q) {
            if (paths[q].nrefl < 0 || paths[q].nrefl > 4) throw visrt::UsageError("bad path");
            if (paths[q].edge >= nedges) throw visrt::UsageError("path references unknown edge");
            if (!(paths[q].length > 0)) throw visrt::VisError("free-space distance must be positive");
        }
        cudaStream_t st = static_cast<cudaStream_t>(stream);
        std::vector<void*> tmp;
        visrt::FreeGuard guard{tmp};
        auto up = [&](const void* src, size_t bytes) {
            void* d = visrt::dalloc<char>(std::max<size_t>(bytes, 16), tmp);
            if (bytes && src) ck(cudaMemcpyAsync(d, src, bytes, cudaMemcpyHostToDevice, st), "H2D");
            return d;
        };
        visrt::EmArgs a{};
        a.s = ds;
        a.npaths = npaths;
        a.paths = static_cast<const visrt_path*>(up(paths, npaths * sizeof(visrt_path)));
        a.mat = static_cast<const double*>(up(face_material, static_cast<size_t>(ds.n) * 16));
        a.edge_ab = static_cast<const double*>(up(edge_ab, std::max(nedges, 0) * 48));
        a.edge_faces = static_cast<const int32_t*>(up(edge_faces, std::max(nedges, 0) * 8));
        a.cfg = *cfg;
        a.amp = visrt::dalloc<double>(2 * std::max<int64_t>(npaths, 1), tmp);
        a.delay = visrt::dalloc<double>(std::max<int64_t>(npaths, 1), tmp);
        a.err = visrt::dalloc<int32_t>(1, tmp);
        ck(cudaMemsetAsync(a.err, 0, 4, st), "memset");
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0);
        cudaEventCreate(&e1);
        cudaEventRecord(e0, st);
        if (npaths > 0) {
            const int blocks = static_cast<int>(std::min<long long>((npaths + 127) / 128, 148 * 8));
            visrt::k_ray_gains<<<blocks, 128, 0, st>>>(a);
            ck(cudaGetLastError(), "k_ray_gains");
        }
        cudaEventRecord(e1, st);
        int32_t err = 0;
        if (npaths > 0) {
            ck(cudaMemcpyAsync(amp, a.amp, npaths * 16, cudaMemcpyDeviceToHost, st), "D2H");
            ck(cudaMemcpyAsync(delay, a.delay, npaths * 8, cudaMemcpyDeviceToHost, st), "D2H");
        }
        ck(cudaMemcpyAsync(&err, a.err, 4, cudaMemcpyDeviceToHost, st), "D2H");
        ck(cudaStreamSynchronize(st), "sync");
        float ms = 0.f;
        cudaEventElapsedTime(&ms, e0, e1);
        cudaEventDestroy(e0);
        cudaEventDestroy(e1);
        if (err) throw visrt::VisError("degenerate wedge or ray parallel to the diffracting edge");
        if (stats) {
            *stats = visrt_stats{};
            stats->pairs = npaths;
            stats->ms = ms;
        }
    });
}

extern "C" int visrt_channel_stats(visrt_scene* sc, int64_t nsnap, const int64_t* path_off, const double* amp,
                                   const double* delay, int8_t* outage, double* path_loss_db,
                                   double* rms_delay_spread, void* stream) {
    return visrt::capi_guard([&] {
        visrt::ScopedDevice dev(sc);
        if (nsnap <= 0) return;
        if (!path_off || !outage || !path_loss_db || !rms_delay_spread) throw visrt::UsageError("null argument");
        cudaStream_t st = static_cast<cudaStream_t>(stream);
        const int64_t np = path_off[nsnap];
        std::vector<void*> tmp;
        visrt::FreeGuard guard{tmp};
        long long* d_off = visrt::dalloc<long long>(nsnap + 1, tmp);
        double* d_amp = visrt::dalloc<double>(2 * std::max<int64_t>(np, 1), tmp);
        double* d_dl = visrt::dalloc<double>(std::max<int64_t>(np, 1), tmp);
        int8_t* d_out = visrt::dalloc<int8_t>(nsnap, tmp);
        double* d_loss = visrt::dalloc<double>(nsnap, tmp);
        double* d_rms = visrt::dalloc<double>(nsnap, tmp);
        ck(cudaMemcpyAsync(d_off, path_off, (nsnap + 1) * 8, cudaMemcpyHostToDevice, st), "H2D");
        if (np) {
            ck(cudaMemcpyAsync(d_amp, amp, np * 16, cudaMemcpyHostToDevice, st), "H2D");
            ck(cudaMemcpyAsync(d_dl, delay, np * 8, cudaMemcpyHostToDevice, st), "H2D");
        }
        const int blocks = static_cast<int>(std::min<long long>((nsnap + 127) / 128, 148 * 8));
        visrt::k_channel_stats<<<blocks, 128, 0, st>>>(nsnap, d_off, d_amp, d_dl, d_out, d_loss, d_rms);
        ck(cudaGetLastError(), "k_channel_stats");
        ck(cudaMemcpyAsync(outage, d_out, nsnap, cudaMemcpyDeviceToHost, st), "D2H");
        ck(cudaMemcpyAsync(path_loss_db, d_loss, nsnap * 8, cudaMemcpyDeviceToHost, st), "D2H");
        ck(cudaMemcpyAsync(rms_delay_spread, d_rms, nsnap * 8, cudaMemcpyDeviceToHost, st), "D2H");
        ck(cudaStreamSynchronize(st), "sync");
    });
}
