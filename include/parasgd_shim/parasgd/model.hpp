// Include-path shim: put `-I include/parasgd_shim` BEFORE the reference's include directory
// and every `#include "parasgd/model.hpp"` of the unmodified reference headers (schemes.hpp,
// analysis.hpp, config.hpp, experiment.hpp, cli.hpp, the tests) resolves to the B200
// drop-in.  The reference files are not edited.
#pragma once
#include "parasgd_b200/model.hpp"
