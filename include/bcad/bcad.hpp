// Umbrella header of the drop-in host API (mirrors /root/reference/proj/include/bcad).
#pragma once

#include "bcad/arity_workload.hpp"
#include "bcad/broadcast.hpp"
#include "bcad/counters.hpp"
#include "bcad/dual.hpp"
#include "bcad/errors.hpp"
#include "bcad/forward.hpp"
#include "bcad/hmlstm.hpp"
#include "bcad/kernel.hpp"
#include "bcad/mixed.hpp"
#include "bcad/oracle.hpp"
#include "bcad/parallel.hpp"
#include "bcad/rng.hpp"
#include "bcad/shape.hpp"
#include "bcad/tape.hpp"
#include "bcad/tensor.hpp"
