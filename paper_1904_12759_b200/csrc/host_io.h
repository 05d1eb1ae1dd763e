// Internal host-side declarations shared by gen.cpp (synthetic inputs),
// mm_io.cpp (Matrix Market + binary CSR cache) and api.cu (device loaders).
// Not part of the public ABI.
#pragma once

#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#include "expmc_b200.h"

// Mirrored, row-sorted adjacency + diagonal: the SparseSymmetric view
// (proj/include/expmc/sparse_matrix.hpp:25-61).
struct expmc_csr {
    uint64_t n = 0;
    std::vector<uint64_t> row_ptr;
    std::vector<uint32_t> col;
    std::vector<double> val;
    std::vector<double> diag;
};

// One parsed Matrix Market coordinate file: the first half of
// load_matrix_market (proj/src/matrix_market.cpp:51-131), before the
// general-symmetry fold and from_entries.
struct expmc_mm {
    std::string path;
    uint64_t n = 0;
    bool general = false;     // symmetry "general" (both triangles listed)
    bool pattern = false;     // field "pattern" (weights 1)
    uint64_t last_line = 0;   // line number of the last entry line read
    std::vector<uint32_t> r, c;  // 0-based, file order
    std::vector<double> w;
};

namespace expmc_b200 {

// Message slot behind expmc_gen_last_error() (thread-local, trivially
// destructible so that late errors during exit cannot touch a destroyed
// string).
void set_host_error(const char* m);
const char* host_error_str();

template <class F>
int host_guarded(F&& f) {
    try {
        f();
        return EXPMC_OK;
    } catch (const std::invalid_argument& e) {
        set_host_error(e.what());
        return EXPMC_INVALID_ARGUMENT;
    } catch (const std::exception& e) {
        set_host_error(e.what());
        return EXPMC_RUNTIME_ERROR;
    } catch (...) {
        set_host_error("unknown error");
        return EXPMC_RUNTIME_ERROR;
    }
}

// load_matrix_market's parse (matrix_market.cpp:51-131) with its messages,
// "path:line: what" as std::runtime_error.  `threads` = 0: all host cores.
void mm_parse(const char* path, expmc_mm& out, unsigned threads = 0);

// The reference's parse_fail message (matrix_market.cpp:17-20).
std::string mm_message(const std::string& path, uint64_t line, const std::string& what);

}  // namespace expmc_b200
