// Umbrella header of the drop-in host API (mirrors /root/reference/proj/include/bcad).
#pragma once

#include "bcad/errors.hpp"
#include "bcad/forward.hpp"
#include "bcad/hmlstm.hpp"
#include "bcad/kernel.hpp"
#include "bcad/mixed.hpp"
#include "bcad/rng.hpp"
#include "bcad/shape.hpp"
#include "bcad/tape.hpp"
#include "bcad/tensor.hpp"
