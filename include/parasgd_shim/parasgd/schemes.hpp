// Include-path shim (see parasgd/model.hpp beside this file): the reference's
// `#include "parasgd/schemes.hpp"` (analysis.hpp, config.hpp, csv.hpp, svg.hpp,
// experiment.hpp) resolves to the B200 run_sparknet / run_naive / run_serial.
#pragma once
#include "parasgd_b200/schemes.hpp"
