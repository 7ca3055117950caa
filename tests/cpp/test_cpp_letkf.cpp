// C++ API test of the LETKF arm (include/turbda/letkf.hpp) on the GPU: the
// Eigen-free cases of the reference's proj/tests/test_letkf.cpp, written
// against the B200 headers and run with the doctest-compatible harness of
// oracle/reftests.  Built by tests/cpp/Makefile, run by
// tests/test_gpu_cpp_api.py.
#include <algorithm>
#include <cmath>
#include <vector>

#include "doctest.h"
#include "turbda/ensemble.hpp"
#include "turbda/letkf.hpp"
#include "turbda/observation.hpp"
#include "turbda/rng.hpp"

using namespace turbda;

namespace {

GridSpec grid_n(int n) {
    GridSpec g;
    g.nx = g.ny = n;
    g.lx = g.ly = 62.83185307179586 * (n / 64.0);
    return g;
}

std::vector<double> normals(std::size_t n, std::uint64_t seed, double mean = 0.0, double sd = 1.0) {
    RngStream rng(seed, StreamUse::generic, 9000);
    std::vector<double> v(n);
    for (auto& x : v) x = mean + sd * rng.normal();
    return v;
}

Ensemble members(int m, std::size_t d, std::uint64_t seed, double mean = 0.0, double sd = 1.0) {
    Ensemble e;
    e.valid_time = 0.0;
    for (int j = 0; j < m; ++j) {
        e.members.push_back(normals(d, seed * 1000 + std::uint64_t(j), mean, sd));
        e.member_seeds.push_back(std::uint64_t(j) + 1);
    }
    return e;
}

Observation dense_obs(const GridSpec& g, std::vector<double> y, double r) {
    Observation o;
    o.op = make_grid_operator(g, 0);
    o.locations = operator_locations(g, o.op);
    o.y = std::move(y);
    o.r_diag.assign(o.y.size(), r);
    o.time = 0.0;
    return o;
}

double max_abs_diff(const std::vector<double>& a, const std::vector<double>& b) {
    double w = 0.0;
    for (std::size_t i = 0; i < a.size(); ++i) w = std::max(w, std::fabs(a[i] - b[i]));
    return w;
}

}  // namespace

TEST_CASE("gaspari_cohn closed forms through the C++ API") {
    CHECK(gaspari_cohn(0.0) == 1.0);
    CHECK(gaspari_cohn(0.5) == doctest::Approx(263.0 / 384.0).epsilon(1e-14));
    CHECK(gaspari_cohn(1.0) == doctest::Approx(5.0 / 24.0).epsilon(1e-14));
    CHECK(gaspari_cohn(1.5) == doctest::Approx(19.0 / 1152.0).epsilon(1e-13));
    CHECK(gaspari_cohn(2.0) == 0.0);
    CHECK_THROWS_AS(gaspari_cohn(-0.1), ConfigError);
}

TEST_CASE("letkf: zero innovation keeps the mean, seeds and time") {
    const GridSpec g = grid_n(8);
    const Ensemble e = members(6, g.grid_size(), 55, 0.2, 1.0);
    const Ensemble an = letkf_analyze(e, dense_obs(g, ensemble_mean(e), 0.5), LetkfConfig{}, g);
    CHECK(max_abs_diff(ensemble_mean(an), ensemble_mean(e)) < 1e-10);
    CHECK(an.valid_time == e.valid_time);
    CHECK(an.member_seeds == e.member_seeds);
    double moved = 0.0;
    for (int j = 0; j < an.size(); ++j)
        moved = std::max(moved, max_abs_diff(an.members[size_t(j)], e.members[size_t(j)]));
    CHECK(moved > 1e-6);
}

TEST_CASE("letkf: near-perfect collocated observations pull the mean onto them") {
    const GridSpec g = grid_n(8);
    const Ensemble e = members(8, g.grid_size(), 66);
    const auto y = normals(g.grid_size(), 9, 0.5, 1.0);
    LetkfConfig cfg;
    cfg.cutoff_km = 1000.0;
    cfg.rtps_alpha = 0.0;
    const Ensemble an = letkf_analyze(e, dense_obs(g, y, 1e-8), cfg, g);
    CHECK(max_abs_diff(ensemble_mean(an), y) < 1e-4);
}

TEST_CASE("letkf: member permutation equivariance and reproducibility") {
    const GridSpec g = grid_n(8);
    const Ensemble e = members(5, g.grid_size(), 88);
    const Observation o = dense_obs(g, normals(g.grid_size(), 12), 1.0);
    const Ensemble a = letkf_analyze(e, o, LetkfConfig{}, g);
    Ensemble rev = e;
    std::reverse(rev.members.begin(), rev.members.end());
    std::reverse(rev.member_seeds.begin(), rev.member_seeds.end());
    const Ensemble b = letkf_analyze(rev, o, LetkfConfig{}, g);
    double worst = 0.0;
    for (int j = 0; j < 5; ++j)
        worst = std::max(worst, max_abs_diff(a.members[size_t(j)], b.members[size_t(4 - j)]));
    CHECK(worst < 1e-9);
    CHECK(letkf_analyze(e, o, LetkfConfig{}, g, 1).members ==
          letkf_analyze(e, o, LetkfConfig{}, g, 8).members);
}

TEST_CASE("rtps: identity at alpha 0 and the two-member hand case") {
    Ensemble bg, an;
    bg.members = {{1.0}, {-1.0}};
    bg.member_seeds = {1, 2};
    an.members = {{0.5}, {0.0}};
    an.member_seeds = {1, 2};
    CHECK(rtps_inflate(an, bg, 0.0).members == an.members);
    const Ensemble out = rtps_inflate(an, bg, 1.0);
    CHECK(out.members[0][0] == doctest::Approx(1.25).epsilon(1e-13));
    CHECK(out.members[1][0] == doctest::Approx(-0.75).epsilon(1e-13));
}

TEST_CASE("letkf: input validation") {
    const GridSpec g = grid_n(8);
    const Ensemble e = members(4, g.grid_size(), 60);
    const Observation o = dense_obs(g, std::vector<double>(g.grid_size(), 0.0), 1.0);
    LetkfConfig bad;
    bad.rtps_alpha = 1.5;
    CHECK_THROWS_AS(bad.validate(), ConfigError);
    Observation late = o;
    late.time = 12.0;
    CHECK_THROWS_AS(letkf_analyze(e, late, LetkfConfig{}, g), ConfigError);
    GridSpec aniso = g;
    aniso.ny = 16;
    aniso.ly = 2.0 * aniso.lx;
    CHECK_THROWS_AS(letkf_analyze(e, o, LetkfConfig{}, aniso), ConfigError);
    const Ensemble tiny = members(4, 10, 61);
    CHECK_THROWS_AS(letkf_analyze(tiny, o, LetkfConfig{}, g), DimensionError);
    // one member: Ensemble::validate() rejects it before any solve
    const Ensemble one = members(1, g.grid_size(), 62);
    CHECK_THROWS_AS(letkf_analyze(one, o, LetkfConfig{}, g), DimensionError);
}
