// Registration group: the arity-scaling workload tanh_product_<A>
// (proj/include/bcad/arity_workload.hpp:19-28; paper Fig. 3 register study).
#include "bodies.cuh"
#include "launch.cuh"

static const bcad_cu_kernel_entry kEntries[] = {
    BCAD_ENTRY(bcad_dev::KTanhProduct<1>),  BCAD_ENTRY(bcad_dev::KTanhProduct<2>),  BCAD_ENTRY(bcad_dev::KTanhProduct<4>),
    BCAD_ENTRY(bcad_dev::KTanhProduct<8>),  BCAD_ENTRY(bcad_dev::KTanhProduct<16>), BCAD_ENTRY(bcad_dev::KTanhProduct<18>),
    BCAD_ENTRY(bcad_dev::KTanhProduct<32>),
};

int bcad_reg_arity(const bcad_cu_kernel_entry** out) {
    *out = kEntries;
    return int(sizeof(kEntries) / sizeof(kEntries[0]));
}
