// Registration group: tanh_product_<A> for A in {32}
// (proj/include/bcad/arity_workload.hpp:19-28), with the all-full-shape
// signature on the forward (the benchmarked kernel; the pullback keeps
// runtime classes, which halves this unit's compile time); see reg_arity.cu
// for the measurements.
#include "bodies.cuh"
#include "launch.cuh"

using bcad_cu_impl::SigAllFull;
static const bcad_cu_kernel_entry kEntries[] = {
    BCAD_ENTRY_FWD_SIG(bcad_dev::KTanhProduct<32>, SigAllFull<32>),
};

int bcad_reg_arity_wide32(const bcad_cu_kernel_entry** out) {
    *out = kEntries;
    return int(sizeof(kEntries) / sizeof(kEntries[0]));
}
