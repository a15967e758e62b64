// The reference's config files and its own `cmd_train` (experiment.hpp:185-231, unmodified,
// reached through include/parasgd_shim) on the B200 drop-in, plus the B200 config keys
// (include/parasgd_b200/experiment.hpp).
//
//   config_test parse FILE...    parse each config (reference + extension keys) and print one
//                                JSON object per file ({"ok": false, "field", "error"} on a
//                                ConfigError) — host only, no GPU
//   config_test train FILE       cmd_train on the GPUs (trace.csv into out.dir /
//                                $PARASGD_OUT), exit codes as cli.hpp:79-85
//
// Built by __graft_entry__.build() with -I include/parasgd_shim -I include -I <reference>.
#include <cstdio>
#include <iostream>
#include <string>

#include "parasgd_b200/experiment.hpp"

using parasgd::ConfigError;
using parasgd::b200::ExperimentConfigB200;

namespace {

std::string scheme_name(const parasgd::ExperimentConfig& c) {
  if (!c.scheme) return "";
  switch (*c.scheme) {
    case parasgd::SchemeKind::Serial: return "serial";
    case parasgd::SchemeKind::Naive: return "naive";
    case parasgd::SchemeKind::Sparknet: return "sparknet";
  }
  return "";
}

void print_parsed(const std::string& path) {
  try {
    const ExperimentConfigB200 c = ExperimentConfigB200::load(path);
    const parasgd::ExperimentConfig& b = c.base;
    std::printf(
        "{\"file\": \"%s\", \"ok\": true, \"scheme\": \"%s\", \"workers\": %d, \"tau\": %d, "
        "\"batch\": %zu, \"lr\": %.17g, \"momentum\": %.17g, \"net\": \"%s\", \"preset\": \"%s\", "
        "\"weight_decay\": %.17g, \"tf32\": %s, \"devices\": %d, \"average\": \"%s\", "
        "\"classes\": %d, \"shape\": [%zu, %zu, %zu], \"extended\": %s}\n",
        path.c_str(), scheme_name(b).c_str(), b.workers, b.tau, b.batch, b.learning_rate,
        b.momentum, b.net_preset.c_str(), c.preset.c_str(), c.ext.weight_decay,
        c.ext.tf32 ? "true" : "false", c.ext.max_devices, c.average.c_str(), b.classes,
        b.channels, b.height, b.width, c.extended() ? "true" : "false");
  } catch (const ConfigError& e) {
    std::printf("{\"file\": \"%s\", \"ok\": false, \"field\": \"%s\", \"error\": \"%s\"}\n",
                path.c_str(), e.field().c_str(), e.what());
  }
}

}  // namespace

int main(int argc, char** argv) {
  if (argc < 3) {
    std::fprintf(stderr, "usage: config_test parse FILE... | train FILE\n");
    return 2;
  }
  const std::string cmd = argv[1];
  if (cmd == "parse") {
    for (int i = 2; i < argc; ++i) print_parsed(argv[i]);
    return 0;
  }
  try {  // cli.hpp:79-85: config errors exit 2, runtime errors 1
    const ExperimentConfigB200 c = ExperimentConfigB200::load(argv[2]);
    return parasgd::b200::cmd_train(c, std::cout);
  } catch (const ConfigError& e) {
    std::fprintf(stderr, "config error: %s\n", e.what());
    return 2;
  } catch (const std::exception& e) {
    std::fprintf(stderr, "error: %s\n", e.what());
    return 1;
  }
}
