// instances.cpp -- seeded synthetic instances for BASELINE.json's configs (host only).
// See include/bornsweep_instances.h.  Input synthesis, not part of the timed sweep.
#include "bornsweep_instances.h"

#include <algorithm>
#include <cmath>
#include <complex>
#include <cstring>
#include <random>
#include <vector>

#ifdef _OPENMP
#include <omp.h>
#endif

namespace {

constexpr double kPi = 3.14159265358979323846;

// RngState semantics of proj/include/bp/rng.hpp:10-62.
inline uint64_t splitmix64(uint64_t x) {
    x += 0x9e3779b97f4a7c15ULL;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
    return x ^ (x >> 31);
}

struct Rng {
    uint64_t seed;
    std::mt19937_64 gen;
    bool have_spare = false;
    double spare = 0.0;
    explicit Rng(uint64_t s) : seed(s), gen(splitmix64(s)) {}
    Rng split(uint64_t index) const { return Rng(splitmix64(seed ^ splitmix64(index + 0x51ed2701))); }
    double uniform() { return static_cast<double>(gen() >> 11) * 0x1.0p-53; }
    double normal() {
        if (have_spare) {
            have_spare = false;
            return spare;
        }
        double u1 = uniform();
        double u2 = uniform();
        while (u1 <= 0.0) u1 = uniform();
        const double r = std::sqrt(-2.0 * std::log(u1));
        const double t = 6.28318530717958647692 * u2;
        spare = r * std::sin(t);
        have_spare = true;
        return r * std::cos(t);
    }
};

Rng stream(uint64_t seed, int64_t index) {
    Rng root(seed);
    return index < 0 ? root : root.split(static_cast<uint64_t>(index));
}

// Separable Gaussian smoothing, zero padding (Dirichlet exterior), truncated at 4 sigma,
// weights normalised to unit sum.
void smooth(int nx, int ny, double sigma, const double* in, double* out) {
    if (sigma <= 0.0) {
        std::memcpy(out, in, sizeof(double) * static_cast<size_t>(nx) * ny);
        return;
    }
    const int R = static_cast<int>(std::ceil(4.0 * sigma));
    std::vector<double> w(2 * R + 1);
    double ws = 0.0;
    for (int d = -R; d <= R; ++d) ws += (w[d + R] = std::exp(-0.5 * d * d / (sigma * sigma)));
    for (double& x : w) x /= ws;
    std::vector<double> tmp(static_cast<size_t>(nx) * ny);
    for (int i = 0; i < nx; ++i)
        for (int j = 0; j < ny; ++j) {
            double s = 0.0;
            for (int d = -R; d <= R; ++d) {
                const int jj = j + d;
                if (jj >= 0 && jj < ny) s += w[d + R] * in[static_cast<size_t>(i) * ny + jj];
            }
            tmp[static_cast<size_t>(i) * ny + j] = s;
        }
    for (int i = 0; i < nx; ++i)
        for (int j = 0; j < ny; ++j) {
            double s = 0.0;
            for (int d = -R; d <= R; ++d) {
                const int ii = i + d;
                if (ii >= 0 && ii < nx) s += w[d + R] * tmp[static_cast<size_t>(ii) * ny + j];
            }
            out[static_cast<size_t>(i) * ny + j] = s;
        }
}

// 3-D separable smoothing (same kernel along z, y, x), zero padding
void smooth3(int n, double sigma, const double* in, double* out) {
    const size_t N3 = (size_t)n * n * n;
    if (sigma <= 0.0) {
        std::memcpy(out, in, sizeof(double) * N3);
        return;
    }
    const int R = static_cast<int>(std::ceil(4.0 * sigma));
    std::vector<double> w(2 * R + 1);
    double ws = 0.0;
    for (int d = -R; d <= R; ++d) ws += (w[d + R] = std::exp(-0.5 * d * d / (sigma * sigma)));
    for (double& x : w) x /= ws;
    std::vector<double> a(in, in + N3), b(N3);
    const size_t strides[3] = {1, (size_t)n, (size_t)n * n};
    for (int ax = 0; ax < 3; ++ax) {
        const size_t st = strides[ax];
        for (size_t idx = 0; idx < N3; ++idx) {
            const int pos = static_cast<int>((idx / st) % n);
            double s = 0.0;
            for (int d = -R; d <= R; ++d) {
                const int pp = pos + d;
                if (pp >= 0 && pp < n) s += w[d + R] * a[idx + (long)d * (long)st];
            }
            b[idx] = s;
        }
        a.swap(b);
    }
    std::memcpy(out, a.data(), sizeof(double) * N3);
}

// sponge_profile (proj/src/samplers.cpp:130-150)
void sponge(int nx, int ny, int layer, double strength, double* out) {
    auto ramp = [layer](int dist) {
        if (dist >= layer) return 0.0;
        const double t = static_cast<double>(layer - dist) / layer;
        return t * t;
    };
    for (int i = 0; i < nx; ++i) {
        const double qx = layer > 0 ? ramp(std::min(i, nx - 1 - i)) : 0.0;
        for (int j = 0; j < ny; ++j) {
            const double qy = layer > 0 ? ramp(std::min(j, ny - 1 - j)) : 0.0;
            out[static_cast<size_t>(i) * ny + j] = layer > 0 ? strength * std::max(qx, qy) : 0.0;
        }
    }
}

// gaussian_bump on a DirichletInterior grid (proj/src/samplers.cpp:86-105,
// coordinates proj/include/bp/grid.hpp:27-40: x(ix) = (ix+1) h, h = lx/(nx+1)).
void bump(int nx, int ny, double lx, double ly, double cx, double cy, double width, double amp,
          double* out, bool accumulate) {
    const double hx = lx / (nx + 1), hy = ly / (ny + 1);
    for (int i = 0; i < nx; ++i) {
        const double dx = (i + 1) * hx - cx;
        for (int j = 0; j < ny; ++j) {
            const double dy = (j + 1) * hy - cy;
            const double v = amp * std::exp(-(dx * dx + dy * dy) / (2.0 * width * width));
            double& o = out[static_cast<size_t>(i) * ny + j];
            o = accumulate ? o + v : v;
        }
    }
}

void make_one(const bp_instance_spec& s, int64_t index, std::complex<double>* k2,
              std::complex<double>* f, double* k0_out, double* eta_out) {
    const int n = s.n, N = n - 1;
    const bool d3 = s.dim == 3;
    const size_t npts = static_cast<size_t>(N) * N * (d3 ? N : 1);
    const double h = 1.0 / n;
    Rng rng = stream(s.seed, index);
    std::vector<double> noise(npts), g(npts);
    for (double& v : noise) v = rng.normal();
    if (d3) smooth3(N, s.sigma_cells, noise.data(), g.data());
    else smooth(N, N, s.sigma_cells, noise.data(), g.data());
    double gmax = 0.0;
    for (double v : g) gmax = std::max(gmax, std::abs(v));
    if (gmax <= 0.0) gmax = 1.0;
    const double omega = 2.0 * kPi / (s.ppw * h);
    std::vector<double> kk(npts);
    double ksum = 0.0;
    for (size_t i = 0; i < npts; ++i) {
        double c = 1.0 + s.contrast * (g[i] / gmax);
        c = std::min(std::max(c, 1.0 - s.contrast), 1.0 + s.contrast);
        kk[i] = omega / c;
        ksum += kk[i];
    }
    const double k0 = ksum / static_cast<double>(npts);
    const int layer = s.sponge_points < 0 ? N / 8 : s.sponge_points;
    std::vector<double> d(npts, 0.0);
    if (layer > 0 && s.sponge_strength > 0.0) {
        if (d3) {
            // 3-D analogue of sponge_profile: strength * max over the three axes of the ramp
            auto ramp = [layer](int dist) {
                if (dist >= layer) return 0.0;
                const double t = static_cast<double>(layer - dist) / layer;
                return t * t;
            };
            for (int i = 0; i < N; ++i)
                for (int j = 0; j < N; ++j)
                    for (int k = 0; k < N; ++k) {
                        const double q = std::max(std::max(ramp(std::min(i, N - 1 - i)),
                                                           ramp(std::min(j, N - 1 - j))),
                                                  ramp(std::min(k, N - 1 - k)));
                        d[((size_t)i * N + j) * N + k] = s.sponge_strength * q;
                    }
        } else {
            sponge(N, N, layer, s.sponge_strength, d.data());
        }
    }
    // k2 -> k2 (1 + i d)  (proj/src/helmholtz.cpp:67-72); eta rule of helmholtz.cpp:80-85 with
    // the config's factor, floored like HelmholtzOptions::eta_floor.
    double dev = 0.0;
    const double k0sq = k0 * k0;
    for (size_t i = 0; i < npts; ++i) {
        const double k2r = kk[i] * kk[i];
        k2[i] = k2r * std::complex<double>(1.0, d[i]);
        dev = std::max(dev, std::abs(k2[i] - k0sq));
    }
    *k0_out = k0;
    *eta_out = std::max(s.eta_factor * dev, 1e-3);
    std::vector<double> src(npts, 0.0);
    const double width = s.src_sigma_cells * h;
    if (d3) {
        // unit 3-D Gaussian bump(s): centre, or n_sources seeded uniform positions
        const int ns = s.n_sources <= 0 ? 1 : s.n_sources;
        for (int m = 0; m < ns; ++m) {
            double cx = 0.5, cy = 0.5, cz = 0.5;
            if (s.n_sources > 0) {
                cx = rng.uniform();
                cy = rng.uniform();
                cz = rng.uniform();
            }
            for (int i = 0; i < N; ++i) {
                const double dx = (i + 1) * h - cx;
                for (int j = 0; j < N; ++j) {
                    const double dy = (j + 1) * h - cy;
                    for (int k = 0; k < N; ++k) {
                        const double dz = (k + 1) * h - cz;
                        src[((size_t)i * N + j) * N + k] +=
                            std::exp(-(dx * dx + dy * dy + dz * dz) / (2.0 * width * width));
                    }
                }
            }
        }
    } else if (s.n_sources <= 0) {
        bump(N, N, 1.0, 1.0, 0.5, 0.5, width, 1.0, src.data(), false);
    } else {
        for (int k = 0; k < s.n_sources; ++k) {
            const double cx = rng.uniform(), cy = rng.uniform();
            bump(N, N, 1.0, 1.0, cx, cy, width, 1.0, src.data(), k > 0);
        }
    }
    for (size_t i = 0; i < npts; ++i) f[i] = std::complex<double>(src[i], 0.0);
}

// Separable Gaussian smoothing with reflective (cell-centred Neumann) padding, truncated at
// 3 sigma, unit-sum weights.
void smooth_reflect(int n, double sigma, const double* in, double* out) {
    const size_t N2 = (size_t)n * n;
    if (sigma <= 0.0) {
        std::memcpy(out, in, sizeof(double) * N2);
        return;
    }
    const int R = static_cast<int>(std::ceil(3.0 * sigma));
    std::vector<double> w(2 * R + 1);
    double ws = 0.0;
    for (int d = -R; d <= R; ++d) ws += (w[d + R] = std::exp(-0.5 * d * d / (sigma * sigma)));
    for (double& x : w) x /= ws;
    auto refl = [n](int i) {
        while (i < 0 || i >= n) i = i < 0 ? -i - 1 : 2 * n - i - 1;
        return i;
    };
    // 1-D pass along contiguous lines through a reflected, padded copy (vectorisable dot)
    auto pass = [&](const double* src, double* dst) {
        std::vector<double> ext(n + 2 * R);
        for (int i = 0; i < n; ++i) {
            const double* line = src + (size_t)i * n;
            for (int k = 0; k < n + 2 * R; ++k) ext[k] = line[refl(k - R)];
            double* o = dst + (size_t)i * n;
            for (int j = 0; j < n; ++j) {
                const double* e = ext.data() + j;
                double acc = 0.0;
                for (int d = 0; d <= 2 * R; ++d) acc += w[d] * e[d];
                o[j] = acc;
            }
        }
    };
    auto transpose = [n](const double* a, double* b) {
        for (int i = 0; i < n; ++i)
            for (int j = 0; j < n; ++j) b[(size_t)j * n + i] = a[(size_t)i * n + j];
    };
    std::vector<double> t1(N2), t2(N2);
    pass(in, t1.data());
    transpose(t1.data(), t2.data());
    pass(t2.data(), t1.data());
    transpose(t1.data(), out);
}

void make_cdr_one(const bp_cdr_spec& s, int64_t index, double* bx, double* by, double* sigma,
                  double* sigma0, double* f) {
    const int n = s.n;
    const size_t N2 = (size_t)n * n;
    Rng rng = stream(s.seed, index);
    const double sm = s.smooth_cells > 0 ? s.smooth_cells : n / 16.0;
    const double sf = s.src_smooth_cells > 0 ? s.src_smooth_cells : n / 32.0;
    double* outs[4] = {sigma, bx, by, f};
    std::vector<double> noise(N2);
    for (int k = 0; k < 4; ++k) {
        for (double& v : noise) v = rng.normal();
        smooth_reflect(n, k == 3 ? sf : sm, noise.data(), outs[k]);
        double mx = 0.0;
        for (size_t i = 0; i < N2; ++i) mx = std::max(mx, std::abs(outs[k][i]));
        if (mx <= 0.0) mx = 1.0;
        for (size_t i = 0; i < N2; ++i) outs[k][i] /= mx;
    }
    const double bs = s.b_max / std::sqrt(2.0);
    double ssum = 0.0;
    for (size_t i = 0; i < N2; ++i) {
        sigma[i] = 0.5 * s.sigma_max * (1.0 + sigma[i]);
        ssum += sigma[i];
        bx[i] *= bs;
        by[i] *= bs;
    }
    *sigma0 = ssum / static_cast<double>(N2);
}

}  // namespace

extern "C" {

int bp_make_cdr_instances(const bp_cdr_spec* spec, int64_t first, int32_t count, double* bx,
                          double* by, double* sigma, double* sigma0, double* f, int32_t nthreads) {
    if (!spec || spec->n < 4 || spec->b_max < 0.0 || spec->sigma_max < 0.0) return 1;
    const size_t N2 = (size_t)spec->n * spec->n;
#ifdef _OPENMP
    const int nt = nthreads > 0 ? nthreads : omp_get_max_threads();
#pragma omp parallel for schedule(dynamic) num_threads(nt)
#endif
    for (int b = 0; b < count; ++b)
        make_cdr_one(*spec, first + b, bx + N2 * b, by + N2 * b, sigma + N2 * b, sigma0 + b, f + N2 * b);
    (void)nthreads;
    return 0;
}

int bp_make_instances(const bp_instance_spec* spec, int64_t first, int32_t count, double* k2,
                      double* f, double* k0, double* eta, int32_t nthreads) {
    if (!spec || spec->n < 3 || !(spec->ppw > 2.0) || spec->contrast < 0.0 || spec->contrast >= 1.0)
        return 1;
    const size_t npts = static_cast<size_t>(spec->n - 1) * (spec->n - 1) * (spec->dim == 3 ? spec->n - 1 : 1);
    auto* K = reinterpret_cast<std::complex<double>*>(k2);
    auto* F = reinterpret_cast<std::complex<double>*>(f);
#ifdef _OPENMP
    const int nt = nthreads > 0 ? nthreads : omp_get_max_threads();
#pragma omp parallel for schedule(dynamic) num_threads(nt)
#endif
    for (int b = 0; b < count; ++b)
        make_one(*spec, first + b, K + npts * b, F + npts * b, k0 + b, eta + b);
    (void)nthreads;
    return 0;
}

void bp_rng_normals(uint64_t seed, int64_t index, int32_t count, double* out) {
    Rng r = stream(seed, index);
    for (int i = 0; i < count; ++i) out[i] = r.normal();
}

void bp_rng_uniforms(uint64_t seed, int64_t index, int32_t count, double* out) {
    Rng r = stream(seed, index);
    for (int i = 0; i < count; ++i) out[i] = r.uniform();
}

void bp_sponge_profile(int32_t nx, int32_t ny, int32_t layer, double strength, double* out) {
    sponge(nx, ny, layer, strength, out);
}

void bp_gaussian_bump(int32_t nx, int32_t ny, double lx, double ly, double cx, double cy,
                      double width, double amplitude, double* out) {
    bump(nx, ny, lx, ly, cx, cy, width, amplitude, out, false);
}

void bp_gaussian_smooth(int32_t nx, int32_t ny, double sigma_cells, const double* in, double* out) {
    smooth(nx, ny, sigma_cells, in, out);
}

}  // extern "C"
