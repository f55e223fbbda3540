// Host-side setup structures (C++), shared by host_setup.cpp and the device
// upload code.
#pragma once

#include <cstdint>
#include <memory>
#include <string>
#include <vector>

#include "../../include/dflb200.h"
#include <nvtx3/nvToolsExt.h>

namespace dfl {

// NVTX range for the phases of setup and solve (header-only NVTX 3: no cost
// unless a profiler injects itself, nsys / ncu --nvtx show the ranges)
struct NvtxRange {
    explicit NvtxRange(const char *name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
    NvtxRange(const NvtxRange &) = delete;
    NvtxRange &operator=(const NvtxRange &) = delete;
};

struct Csr {
    int64_t nrows = 0, ncols = 0;
    std::vector<int64_t> ptr{0};
    std::vector<int64_t> col;
    std::vector<double> val;
    int64_t nnz() const { return (int64_t)col.size(); }
};

struct Level {
    Csr A, P, R;
    std::vector<double> w;           // relaxation weights (damping/a_ii or SPAI-0)
    bool bottom = false;
    std::vector<double> bottom_inv;  // dense inverse of the bottom block
};

struct Hierarchy {
    std::vector<Level> levels;
    int relax = DFL_RELAX_DAMPED_JACOBI;
};

void set_setup_error(const std::string &s);
const char *setup_error();

Csr csr_from_view(const dfl_csr *v);
Csr transpose(const Csr &a);
Csr spgemm(const Csr &a, const Csr &b);
bool diagonal(const Csr &a, std::vector<double> &d, const char *what);
int lu_inverse(int64_t n, const double *a, double *inv);
int build_hierarchy(const Csr &a0, const dfl_amg_options &o, Hierarchy &h);
int64_t aggregate(const Csr &s, std::vector<int64_t> &label);
int close_bottom(Hierarchy &h, Csr &&a);
// device-side products (setup_dev.cu)
void set_setup_device(int device);
int setup_device();
int build_hierarchy_dev(const Csr &a0, const dfl_amg_options &o, Hierarchy &h);
int basis_az(const dfl_csr *A, int k, const double *zext, const int32_t *owner,
             const int32_t *rowsub, int64_t K, int sub0, int nsub, int keep_zeros, Csr &az,
             double *E_rows);

}  // namespace dfl

// opaque handle of the C ABI
struct dfl_hier {
    // shared with the device contexts it is added to (no deep copy on dfl_ctx_add_hierarchy)
    std::shared_ptr<dfl::Hierarchy> sp = std::make_shared<dfl::Hierarchy>();
    dfl::Hierarchy &h = *sp;
};

// the opaque host CSR handle of the C ABI (dfl_matrix_shape / _copy / _free)
struct dfl_matrix {
    dfl::Csr m;
};
