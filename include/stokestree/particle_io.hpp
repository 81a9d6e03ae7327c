// Drop-in name for the reference header stokestree/particle_io.hpp (see stokestree/harness.hpp).
#pragma once
#include "stokestree/harness.hpp"
