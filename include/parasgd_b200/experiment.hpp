// parasgd_b200/experiment.hpp — the reference's config files and `cmd_train`
// (config.hpp:203-430, experiment.hpp:185-231) driving the B200 drop-in, plus the B200
// config keys.  Build with `-I include/parasgd_shim -I include -I <reference>/include`:
// the shim routes the reference's `parasgd/model.hpp` / `parasgd/schemes.hpp` includes to
// parasgd_b200, so the reference's ExperimentConfig, load_experiment_data, materialize_net,
// make_scheme_context, cmd_train and csv::write_trace run unmodified on the GPUs.
//
// Extension keys (absent = the reference's behaviour; every reference key keeps its meaning
// and checks, and unknown keys are still rejected by the reference's parser):
//   net.preset       = cifar10_quick | alexnet | googlenet   (besides mlp / lenet-small)
//   sgd.weight_decay = L2 decay (>= 0), scaled per tensor by the presets' decay_mult
//   precision        = fp32 | tf32   (strict SIMT / tcgen05 tensor cores)
//   device.count     = GPUs the workers may use (0 = all visible)
//   average.mode     = ordered | fast  (weights_mean order / ncclAllReduce avg)
#pragma once

#include <cstdlib>
#include <map>
#include <sstream>
#include <string>

#include "parasgd/experiment.hpp"
#include "parasgd_b200/presets.hpp"

namespace parasgd {
namespace b200 {

struct ExperimentConfigB200 {
  ExperimentConfig base;  // parsed and range-checked by the reference's own parser
  std::string preset;     // a Caffe preset, or empty
  Extension ext;
  std::string average = "ordered";

  bool extended() const {
    return !preset.empty() || ext.weight_decay > 0.0 || ext.tf32 || ext.max_devices > 0;
  }

  static ExperimentConfigB200 from_text(const std::string& text) {
    const KeyValues kv = KeyValues::parse(text);  // syntax / duplicate-key checks
    ExperimentConfigB200 c;
    std::ostringstream rest;  // everything but the extension keys -> the reference parser
    for (const auto& [key, value] : kv.raw()) {
      if (key == "net.preset" && is_caffe_preset(value)) {
        c.preset = value;
      } else if (key == "sgd.weight_decay") {
        c.ext.weight_decay = number(key, value);
        if (!(c.ext.weight_decay >= 0.0)) throw ConfigError(key, "must be >= 0");
      } else if (key == "precision") {
        if (value != "fp32" && value != "tf32")
          throw ConfigError(key, "unknown precision '" + value + "'; valid: fp32, tf32");
        c.ext.tf32 = value == "tf32";
      } else if (key == "device.count") {
        const double d = number(key, value);
        if (d < 0 || d != static_cast<int>(d)) throw ConfigError(key, "must be an integer >= 0");
        c.ext.max_devices = static_cast<int>(d);
      } else if (key == "average.mode") {
        if (value != "ordered" && value != "fast")
          throw ConfigError(key, "unknown mode '" + value + "'; valid: ordered, fast");
        c.average = value;
      } else {
        rest << key << " = " << value << "\n";
      }
    }
    if (!c.preset.empty() && kv.has("net.spec"))
      throw ConfigError("net.preset", "a Caffe preset cannot be combined with net.spec");
    c.base = ExperimentConfig::from_text(rest.str());
    if (!c.preset.empty()) {
      c.base.net_preset = c.preset;
      c.ext.graph = [](const SchemeContext& ctx) {
        const Dataset& d = *ctx.train_data;
        return caffe_preset(active_preset(), ctx.batch, d.channels(), d.height(), d.width(),
                            d.num_classes);
      };
    }
    return c;
  }

  static ExperimentConfigB200 load(const std::string& path) {
    std::ifstream in(path);
    if (!in) throw ConfigError("config", "cannot open " + path);
    std::stringstream buffer;
    buffer << in.rdbuf();
    return from_text(buffer.str());
  }

  static std::string& active_preset() {
    thread_local std::string p;
    return p;
  }

 private:
  static double number(const std::string& key, const std::string& v) {
    try {
      std::size_t used = 0;
      const double d = std::stod(v, &used);
      if (used != v.size()) throw std::invalid_argument(v);
      return d;
    } catch (const std::exception&) {
      throw ConfigError(key, "expected a number, got '" + v + "'");
    }
  }
};

/// While alive, the schemes build their Nets with the config's extension settings.
class ExtensionScope {
 public:
  explicit ExtensionScope(const ExperimentConfigB200& cfg) : prev_(active_extension()) {
    ExperimentConfigB200::active_preset() = cfg.preset;
    active_extension() = &cfg.ext;
    const char* a = std::getenv("PARASGD_AVERAGE");
    prev_avg_ = a ? a : "";
    had_avg_ = a != nullptr;
    setenv("PARASGD_AVERAGE", cfg.average.c_str(), 1);
  }
  ~ExtensionScope() {
    active_extension() = prev_;
    if (had_avg_)
      setenv("PARASGD_AVERAGE", prev_avg_.c_str(), 1);
    else
      unsetenv("PARASGD_AVERAGE");
  }
  ExtensionScope(const ExtensionScope&) = delete;
  ExtensionScope& operator=(const ExtensionScope&) = delete;

 private:
  const Extension* prev_;
  std::string prev_avg_;
  bool had_avg_ = false;
};

/// `train` (experiment.hpp:185-231): the reference's own cmd_train on the B200 drop-in.
inline int cmd_train(const ExperimentConfigB200& cfg, std::ostream& log) {
  ExtensionScope scope(cfg);
  return parasgd::cmd_train(cfg.base, log);
}

}  // namespace b200
}  // namespace parasgd
