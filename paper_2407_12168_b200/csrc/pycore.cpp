// Python module paper_2407_12168_b200._core - the B200 counterpart of the
// reference binding (proj/python/bindings.cpp): ensf_analyze (:140-155) and
// letkf_analyze (:157-172) keep the reference signatures and defaults, with
// keyword-only extras for the observation thinning, the arithmetic and the
// devices; arrays go straight from numpy to the device through the C-ABI.
// GridSpec / SqgParams, nature_run / advance (:87-109, the GPU model),
// default_config_json / config_hash (:196-202) and the exceptions (:223-224)
// follow the reference, as do ke_spectrum / fit_loglog_slope (:111-138).
// run_experiment lives in experiment.py (the GPU-resident cycle driver);
// the budget helpers (:204-220) are plain host arithmetic.
#include <pybind11/numpy.h>
#include <pybind11/pybind11.h>
#include <pybind11/stl.h>

#include <cmath>
#include <string>
#include <vector>

#include "turbda/budget.hpp"
#include "turbda/config.hpp"
#include "turbda/errors.hpp"
#include "turbda/forecast.hpp"
#include "turbda/grid.hpp"
#include "turbda/osse.hpp"
#include "turbda_b200.h"

namespace py = pybind11;

namespace {

using darray = py::array_t<double, py::array::c_style | py::array::forcecast>;

[[noreturn]] void raise(int code, const turbda_status& st) {
    switch (code) {
        case TURBDA_CONFIG: throw turbda::ConfigError(st.msg);
        case TURBDA_DIMENSION: throw turbda::DimensionError(st.msg);
        case TURBDA_DIVERGED: throw turbda::SamplerDivergedError(st.diverged_t);
        case TURBDA_DOMAIN: throw std::domain_error(st.msg);
        case TURBDA_SINGULAR: throw turbda::SingularAnalysisError(st.diverged_particle, st.diverged_step);
        default: throw std::runtime_error(std::string("turbda_b200: ") + st.msg);
    }
}

int parse_precision(const std::string& s) {
    if (s == "fp32" || s == "float32") return TURBDA_FP32;
    if (s == "fp64" || s == "float64") return TURBDA_FP64;
    throw turbda::ConfigError("precision must be 'fp32' or 'fp64'");
}

py::array_t<double> ensf_analyze(const darray& members, const turbda::GridSpec& grid,
                                 const darray& y, double r, std::uint64_t seed,
                                 std::uint64_t cycle, int n_steps, double relax_factor,
                                 int /*workers*/, int thinning, const std::string& precision,
                                 int device, int device_count, double eps, int minibatch_j,
                                 double damping_t, const std::string& obs_operator,
                                 const std::string& score_mode, py::object out_obj) {
    if (members.ndim() != 2) throw turbda::DimensionError("members must be (M, d)");
    const auto m = members.shape(0);
    const auto d = members.shape(1);
    // Ensemble::validate(false)
    if (m < 1) throw turbda::DimensionError("ensemble: empty");
    // make_grid_operator(grid, thinning) + Observation::validate
    const int64_t state_dim = int64_t(grid.grid_size());
    std::vector<int64_t> idx;
    if (thinning > 1)
        for (int64_t k = 0; k < state_dim; k += thinning) idx.push_back(k);
    const int64_t obs_dim = thinning > 1 ? int64_t(idx.size()) : state_dim;
    if (y.size() != obs_dim) throw turbda::DimensionError("observation: length mismatch");
    if (!(r > 0.0)) throw turbda::ConfigError("observation: r_diag > 0");
    if (state_dim != d) throw turbda::DimensionError("analyze: observation operator dimension");

    turbda_ensf_params p;
    turbda_ensf_params_init(&p);
    p.d_total = d;
    p.d_local = d;
    p.obs_dim = obs_dim;
    p.n_members = int32_t(m);
    p.n_steps = n_steps;
    p.minibatch_j = minibatch_j;
    if (obs_operator != "linear" && obs_operator != "arctan")
        throw turbda::ConfigError("obs_operator must be 'linear' or 'arctan'");
    p.obs_kind = (thinning > 1 ? 1 : 0) + (obs_operator == "arctan" ? 2 : 0);
    if (score_mode != "componentwise" && score_mode != "joint")
        throw turbda::ConfigError("score_mode must be 'componentwise' or 'joint'");
    p.score_mode = score_mode == "joint" ? TURBDA_SCORE_JOINT : TURBDA_SCORE_COMPONENTWISE;
    p.eps = eps;
    p.damping_t = damping_t;
    p.relax_factor = relax_factor;
    p.seed = seed;
    p.cycle = cycle;
    p.precision = parse_precision(precision);
    p.device = device;
    p.device_count = device_count;
    p.flags = TURBDA_R_UNIFORM;  // the scalar r, not an obs_dim-long copy of it

    // out=: a caller-owned (M, d) float64 C-contiguous array (e.g. pinned
    // host memory) receives the analysis; otherwise a new array is returned
    py::array_t<double> out;
    if (out_obj.is_none()) {
        out = py::array_t<double>({m, d});
    } else {
        out = py::array_t<double>::ensure(out_obj);
        if (!out || out.ndim() != 2 || out.shape(0) != m || out.shape(1) != d ||
            !(out.flags() & py::array::c_style) || out.ptr() != out_obj.ptr())
            throw turbda::DimensionError("out must be a C-contiguous float64 (M, d) array");
    }
    turbda_status st{};
    int rc;
    {
        py::gil_scoped_release nogil;
        rc = turbda_ensf_analyze(&p, members.data(), y.data(), &r,
                                 idx.empty() ? nullptr : idx.data(), out.mutable_data(), nullptr,
                                 &st);
    }
    if (rc) raise(rc, st);
    return out;
}

py::array_t<double> letkf_analyze(const darray& members, const turbda::GridSpec& grid,
                                  const darray& y, double r, double cutoff_km, double rtps_alpha,
                                  int /*workers*/, int thinning, int device) {
    if (members.ndim() != 2) throw turbda::DimensionError("members must be (M, d)");
    grid.validate();
    const auto m = members.shape(0), d = members.shape(1);
    if (int64_t(grid.grid_size()) != d)
        throw turbda::DimensionError("letkf_analyze: state/grid size mismatch");
    std::vector<int64_t> idx;
    if (thinning > 1)
        for (int64_t k = 0; k < d; k += thinning) idx.push_back(k);
    const int64_t obs_dim = thinning > 1 ? int64_t(idx.size()) : d;
    if (y.size() != obs_dim) throw turbda::DimensionError("observation: length mismatch");
    if (!(r > 0.0)) throw turbda::ConfigError("observation: r_diag > 0");
    turbda_letkf_params p;
    turbda_letkf_params_init(&p);
    p.nx = grid.nx;
    p.ny = grid.ny;
    p.n_members = int32_t(m);
    p.obs_kind = thinning > 1 ? 1 : 0;
    p.obs_dim = obs_dim;
    p.cutoff_km = cutoff_km;
    p.rtps_alpha = rtps_alpha;
    p.device = device;
    p.flags = TURBDA_R_UNIFORM;
    if (grid.nx != grid.ny || grid.lx != grid.ly)
        throw turbda::ConfigError("letkf_analyze: isotropic metric needs nx == ny");
    py::array_t<double> out({m, d});
    turbda_status st{};
    int rc;
    {
        py::gil_scoped_release nogil;
        rc = turbda_letkf_analyze(&p, members.data(), y.data(), &r,
                                  idx.empty() ? nullptr : idx.data(), nullptr, out.mutable_data(),
                                  nullptr, &st);
    }
    if (rc) raise(rc, st);
    return out;
}

py::array_t<double> field_array(const turbda::GridSpec& g, const std::vector<double>& v) {
    py::array_t<double> out({g.nz, g.ny, g.nx});
    std::copy(v.begin(), v.end(), out.mutable_data());
    return out;
}

}  // namespace

PYBIND11_MODULE(_core, mod) {
    mod.doc() = "B200-native EnSF analysis step (sm_100a) behind the turbda binding API";

    py::class_<turbda::GridSpec>(mod, "GridSpec")
        .def(py::init<>())
        .def_readwrite("nx", &turbda::GridSpec::nx)
        .def_readwrite("ny", &turbda::GridSpec::ny)
        .def_readwrite("nz", &turbda::GridSpec::nz)
        .def_readwrite("lx", &turbda::GridSpec::lx)
        .def_readwrite("ly", &turbda::GridSpec::ly)
        .def_readwrite("h", &turbda::GridSpec::h)
        .def("grid_size", &turbda::GridSpec::grid_size)
        .def("validate", &turbda::GridSpec::validate);

    mod.def("ensf_analyze", &ensf_analyze, py::arg("members"), py::arg("grid"), py::arg("y"),
            py::arg("r") = 1.0, py::arg("seed") = 7, py::arg("cycle") = 1,
            py::arg("n_steps") = 100, py::arg("relax_factor") = 1.0, py::arg("workers") = 0,
            py::kw_only(), py::arg("thinning") = 0, py::arg("precision") = "fp32",
            py::arg("device") = -1, py::arg("device_count") = 1, py::arg("eps") = 0.01,
            py::arg("minibatch_j") = 0, py::arg("damping_t") = 1.0,
            py::arg("obs_operator") = "linear", py::arg("score_mode") = "componentwise",
            py::arg("out") = py::none(),
            "EnSF analysis of an (M, d) float64 forecast ensemble on the GPU; returns (M, d)");

    py::class_<turbda::SqgParams>(mod, "SqgParams")
        .def(py::init<>())
        .def_readwrite("f", &turbda::SqgParams::f)
        .def_readwrite("n", &turbda::SqgParams::n)
        .def_readwrite("u0", &turbda::SqgParams::u0)
        .def_readwrite("hyper_order", &turbda::SqgParams::hyper_order)
        .def_readwrite("hyper_efold", &turbda::SqgParams::hyper_efold)
        .def_readwrite("dt", &turbda::SqgParams::dt)
        .def_readwrite("drag_tau", &turbda::SqgParams::drag_tau)
        .def("validate", &turbda::SqgParams::validate);

    mod.def(
        "nature_run",
        [](const turbda::GridSpec& grid, const turbda::SqgParams& params, double spinup,
           double duration, double interval, std::uint64_t seed) {
            std::vector<std::vector<double>> snaps;
            {
                py::gil_scoped_release nogil;
                snaps = turbda::nature_run(grid, params, spinup, duration, interval, seed);
            }
            py::list out;
            for (const auto& s : snaps) out.append(field_array(grid, s));
            return out;
        },
        py::arg("grid"), py::arg("params"), py::arg("spinup"), py::arg("duration"),
        py::arg("interval"), py::arg("seed"),
        "clean model run on the GPU; returns a list of (nz, ny, nx) snapshots");

    mod.def(
        "advance",
        [](const turbda::GridSpec& grid, const turbda::SqgParams& params, const darray& state,
           double hours) {
            std::vector<double> v(state.data(), state.data() + state.size());
            {
                py::gil_scoped_release nogil;
                turbda::SqgStepper stepper(grid, params);
                stepper.advance(v, hours);
            }
            return field_array(grid, v);
        },
        py::arg("grid"), py::arg("params"), py::arg("state"), py::arg("hours"));

    mod.def(
        "ke_spectrum",
        [](const turbda::GridSpec& grid, const turbda::SqgParams& params, const darray& state) {
            if (size_t(state.size()) != grid.grid_size())
                throw turbda::DimensionError("ke_spectrum: state size does not match grid");
            std::vector<turbda::KeBin> bins;
            {
                py::gil_scoped_release nogil;
                turbda::SqgModel model(grid, params);
                bins = model.ke_spectrum(state.data());
            }
            py::array_t<double> kappa(py::ssize_t(bins.size())), energy(py::ssize_t(bins.size()));
            for (size_t s = 0; s < bins.size(); ++s) {
                kappa.mutable_data()[s] = bins[s].kappa;
                energy.mutable_data()[s] = bins[s].energy;
            }
            return py::make_tuple(kappa, energy);
        },
        py::arg("grid"), py::arg("params"), py::arg("state"));

    mod.def(
        "fit_loglog_slope",
        [](const darray& kappa, const darray& energy, int lo_shell, int hi_shell) {
            std::vector<turbda::KeBin> bins(size_t(kappa.size()));
            for (size_t s = 0; s < bins.size(); ++s)
                bins[s] = {kappa.data()[s], energy.data()[s]};
            return turbda::fit_loglog_slope(bins, lo_shell, hi_shell);
        },
        py::arg("kappa"), py::arg("energy"), py::arg("lo_shell"), py::arg("hi_shell"));

    mod.def("letkf_analyze", &letkf_analyze, py::arg("members"), py::arg("grid"), py::arg("y"),
            py::arg("r") = 1.0, py::arg("cutoff_km") = 2000.0, py::arg("rtps_alpha") = 0.3,
            py::arg("workers") = 0, py::kw_only(), py::arg("thinning") = 0,
            py::arg("device") = -1,
            "LETKF analysis of an (M, d) float64 forecast ensemble on the GPU; returns (M, d)");

    mod.def("default_config_json",
            [] { return turbda::config_to_json(turbda::ExperimentConfig{}).dump(2); });
    mod.def("config_hash", [](const std::string& config_json) {
        return turbda::config_hash(turbda::config_from_json(nlohmann::json::parse(config_json)));
    });

    mod.def("vit_param_count", &turbda::vit_param_count, py::arg("layers"), py::arg("embed_dim"),
            py::arg("mlp_ratio"));
    mod.def(
        "estimate_training_flops",
        [](const std::vector<long long>& input_dims, const std::vector<long long>& patch_dims,
           double epochs, double params, double images) {
            turbda::BudgetSpec spec;
            spec.input_dims = input_dims;
            spec.patch_dims = patch_dims;
            spec.epochs = epochs;
            spec.params = params;
            spec.dataset_images = images;
            return turbda::estimate_training_flops(spec);
        },
        py::arg("input_dims"), py::arg("patch_dims"), py::arg("epochs"), py::arg("params"),
        py::arg("images"));
    mod.def("format_sig", &turbda::format_sig, py::arg("x"), py::arg("digits") = 4);

    mod.def("device_count", &turbda_device_count);
    mod.def("build_arch", [] { return std::string(turbda_build_arch()); });
    mod.def("launch_count", [] { return turbda_launch_count(); });

    py::register_exception<turbda::ConfigError>(mod, "ConfigError", PyExc_ValueError);
    py::register_exception<turbda::DimensionError>(mod, "DimensionError", PyExc_ValueError);
}
