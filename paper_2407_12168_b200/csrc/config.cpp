// JSON side of the OSSE layer (include/turbda/config.hpp, the reference's
// proj/src/config.cpp schema): config_to_json / config_from_json through one
// field table (section, key, member), load/save, the FNV-1a config hash, and
// MetricsSeries::to_jsonl.  nlohmann/json is header-only.
#include <cstdio>
#include <fstream>
#include <functional>
#include <string>
#include <vector>

#include "turbda/config.hpp"

namespace turbda {

namespace {

using nlohmann::json;
using nlohmann::ordered_json;

// one scalar field of the schema: where it lives in the JSON and in the config
struct Field {
    const char* section;  // nullptr: top level
    const char* key;
    std::function<void(const ExperimentConfig&, ordered_json&)> put;
    std::function<void(const json&, ExperimentConfig&)> get;
};

template <class T, class Ref>
Field field(const char* section, const char* key, Ref ref) {
    return Field{section, key,
                 [key, ref](const ExperimentConfig& c, ordered_json& o) {
                     o[key] = static_cast<T>(ref(const_cast<ExperimentConfig&>(c)));
                 },
                 [key, ref](const json& j, ExperimentConfig& c) { ref(c) = j.at(key).get<T>(); }};
}

#define TB_FIELD(T, sec, key, expr) field<T>(sec, key, [](ExperimentConfig& c) -> T& { return expr; })

const std::vector<Field>& schema() {
    static const std::vector<Field> f = {
        TB_FIELD(int, "grid", "nx", c.grid.nx),
        TB_FIELD(int, "grid", "ny", c.grid.ny),
        TB_FIELD(int, "grid", "nz", c.grid.nz),
        TB_FIELD(double, "grid", "lx", c.grid.lx),
        TB_FIELD(double, "grid", "ly", c.grid.ly),
        TB_FIELD(double, "grid", "h", c.grid.h),
        TB_FIELD(double, "sqg", "f", c.sqg.f),
        TB_FIELD(double, "sqg", "n", c.sqg.n),
        TB_FIELD(double, "sqg", "u0", c.sqg.u0),
        TB_FIELD(int, "sqg", "hyper_order", c.sqg.hyper_order),
        TB_FIELD(double, "sqg", "hyper_efold", c.sqg.hyper_efold),
        TB_FIELD(double, "sqg", "dt", c.sqg.dt),
        TB_FIELD(double, "sqg", "drag_tau", c.sqg.drag_tau),
        TB_FIELD(double, "sqg", "dealias_fraction", c.sqg.dealias_fraction),
        TB_FIELD(int, "ensf", "n_steps", c.ensf.n_steps),
        TB_FIELD(double, "ensf", "eps", c.ensf.eps),
        TB_FIELD(int, "ensf", "minibatch_j", c.ensf.minibatch_j),
        TB_FIELD(double, "ensf", "damping_t", c.ensf.damping_t),
        TB_FIELD(double, "ensf", "relax_factor", c.ensf.relax_factor),
        TB_FIELD(double, "letkf", "cutoff_km", c.letkf.cutoff_km),
        TB_FIELD(double, "letkf", "domain_km", c.letkf.domain_km),
        TB_FIELD(double, "letkf", "rtps_alpha", c.letkf.rtps_alpha),
        TB_FIELD(int, "letkf", "obs_thinning", c.letkf.obs_thinning),
    };
    return f;
}

const std::vector<Field>& tail_schema() {  // after model_error / obs / variant
    static const std::vector<Field> f = {
        TB_FIELD(int, nullptr, "cycles", c.cycles),
        TB_FIELD(double, nullptr, "obs_interval", c.obs_interval),
        TB_FIELD(int, nullptr, "ensemble_size", c.ensemble_size),
        TB_FIELD(std::uint64_t, nullptr, "seed", c.seed),
        TB_FIELD(double, nullptr, "spinup_hours", c.spinup_hours),
        TB_FIELD(double, nullptr, "clim_hours", c.clim_hours),
        TB_FIELD(int, nullptr, "fit_lo_shell", c.fit_lo_shell),
        TB_FIELD(int, nullptr, "fit_hi_shell", c.fit_hi_shell),
    };
    return f;
}

#undef TB_FIELD

void put_fields(const std::vector<Field>& fs, const ExperimentConfig& cfg, ordered_json& j) {
    for (const Field& f : fs) f.put(cfg, f.section ? j[f.section] : j);
}

void get_fields(const std::vector<Field>& fs, const json& j, ExperimentConfig& cfg) {
    for (const Field& f : fs) {
        const json* where = &j;
        if (f.section) {
            const auto s = j.find(f.section);
            if (s == j.end()) continue;
            where = &*s;
        }
        if (where->contains(f.key)) f.get(*where, cfg);  // absent keys keep the defaults
    }
}

}  // namespace

ordered_json config_to_json(const ExperimentConfig& cfg) {
    ordered_json j;
    put_fields(schema(), cfg, j);
    json mixture = json::array();
    for (const auto& c : cfg.model_error.mixture)
        mixture.push_back(json{{"probability", c.first}, {"amplitude_fraction", c.second}});
    j["model_error"]["enabled"] = cfg.model_error.enabled;
    j["model_error"]["base_amplitude"] = cfg.model_error.base_amplitude;
    j["model_error"]["mixture"] = mixture;
    j["obs"]["r"] = cfg.obs.r;
    j["obs"]["thinning_stride"] = cfg.obs.thinning_stride;
    j["variant"] = variant_name(cfg.variant);
    j["model_quality"] = quality_name(cfg.model_quality);
    put_fields(tail_schema(), cfg, j);
    return j;
}

ExperimentConfig config_from_json(const json& j) {
    ExperimentConfig cfg;
    get_fields(schema(), j, cfg);
    if (const auto m = j.find("model_error"); m != j.end()) {
        if (m->contains("enabled")) cfg.model_error.enabled = m->at("enabled").get<bool>();
        if (m->contains("base_amplitude"))
            cfg.model_error.base_amplitude = m->at("base_amplitude").get<double>();
        if (const auto mix = m->find("mixture"); mix != m->end()) {
            cfg.model_error.mixture.clear();
            for (const json& c : *mix)
                cfg.model_error.mixture.emplace_back(c.at("probability").get<double>(),
                                                     c.at("amplitude_fraction").get<double>());
        }
    }
    if (const auto o = j.find("obs"); o != j.end()) {
        if (o->contains("r")) cfg.obs.r = o->at("r").get<double>();
        if (o->contains("thinning_stride")) cfg.obs.thinning_stride = o->at("thinning_stride").get<int>();
    }
    if (j.contains("variant")) cfg.variant = variant_from_name(j.at("variant").get<std::string>());
    if (j.contains("model_quality"))
        cfg.model_quality = quality_from_name(j.at("model_quality").get<std::string>());
    get_fields(tail_schema(), j, cfg);
    return cfg;
}

ExperimentConfig load_config(const std::filesystem::path& path) {
    std::ifstream in(path);
    if (!in) throw IoError("cannot open config '" + path.string() + "'");
    json j;
    try {
        in >> j;
    } catch (const json::exception& e) {
        throw IoError("bad config '" + path.string() + "': " + e.what());
    }
    return config_from_json(j);
}

void save_config(const ExperimentConfig& cfg, const std::filesystem::path& path) {
    std::ofstream out(path);
    if (!out) throw IoError("cannot write config '" + path.string() + "'");
    out << config_to_json(cfg).dump(2) << '\n';
}

std::string config_hash(const ExperimentConfig& cfg) {
    // sorted keys (plain json) make the hash independent of key order
    const std::string canonical = json(config_to_json(cfg)).dump();
    std::uint64_t h = 0xcbf29ce484222325ull;  // FNV-1a 64
    for (const unsigned char ch : canonical) h = (h ^ ch) * 0x100000001b3ull;
    char hex[17];
    std::snprintf(hex, sizeof hex, "%016llx", static_cast<unsigned long long>(h));
    return hex;
}

std::string MetricsSeries::to_jsonl() const {
    std::string out;
    for (const CycleRecord& r : records) {
        ordered_json o;
        o["cycle"] = r.cycle;
        o["time"] = r.time;
        o["forecast_rmse"] = r.forecast_rmse;
        o["analysis_rmse"] = r.analysis_rmse;
        o["forecast_spread"] = r.forecast_spread;
        o["analysis_spread"] = r.analysis_spread;
        out += o.dump() + '\n';
    }
    return out;
}

}  // namespace turbda
