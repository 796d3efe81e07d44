// One-line forwarder: the reference's bench.hpp includes <nlohmann/json_fwd.hpp>;
// the image ships the single-header nlohmann 3.11.3 json.hpp (see oracle/Makefile).
#pragma once
#include <nlohmann/json.hpp>
