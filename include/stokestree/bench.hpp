// Drop-in name for the reference header stokestree/bench.hpp (see stokestree/harness.hpp).
#pragma once
#include "stokestree/harness.hpp"
