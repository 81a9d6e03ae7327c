// Drop-in name for the reference header stokestree/taylor_coeffs.hpp; the whole API lives in
// stokestree/stokestree.hpp (backed by libstokestree_b200.so).
#pragma once
#include "stokestree/stokestree.hpp"
