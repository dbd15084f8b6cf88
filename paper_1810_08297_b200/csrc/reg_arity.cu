// Registration group: the arity-scaling workload tanh_product_<A>, A <= 8
// (3 and 5: the arities the reference's acceptance program and tests name)
// (the wide arities are in reg_arity_wide*.cu: separate translation units
// compile in parallel)
// (proj/include/bcad/arity_workload.hpp:19-28; paper Fig. 3 register study).
#include "bodies.cuh"
#include "launch.cuh"

// Every arity is registered with the all-full-shape signature as well: the
// A-wide loops lose their per-argument class branches and per-store null
// checks. Measured at 4096^2 fp32 K1 (scripts/lab "arity", means, fraction of
// the copy peak, runtime classes -> static): A4 0.86 -> 0.96, A8 0.85 -> 0.99,
// A16 0.71 -> 0.93, A18 0.71 -> 0.92, A32 0.62 -> 0.79.
using bcad_cu_impl::SigAllFull;
static const bcad_cu_kernel_entry kEntries[] = {
    BCAD_ENTRY(bcad_dev::KTanhProduct<1>, SigAllFull<1>), BCAD_ENTRY(bcad_dev::KTanhProduct<2>, SigAllFull<2>),
    BCAD_ENTRY(bcad_dev::KTanhProduct<3>, SigAllFull<3>), BCAD_ENTRY(bcad_dev::KTanhProduct<4>, SigAllFull<4>),
    BCAD_ENTRY(bcad_dev::KTanhProduct<5>, SigAllFull<5>), BCAD_ENTRY(bcad_dev::KTanhProduct<8>, SigAllFull<8>),
};

int bcad_reg_arity(const bcad_cu_kernel_entry** out) {
    *out = kEntries;
    return int(sizeof(kEntries) / sizeof(kEntries[0]));
}
