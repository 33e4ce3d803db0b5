// generate.cuh — on-device generators of the BASELINE factors (generate.cu).
#pragma once

#include "common.cuh"

namespace lsb {

struct GeneratedCsr;
GeneratedCsr* generate_stencil_rows(const int64_t grid[3], int32_t rows_per_node, int32_t max_entries, const int32_t* offsets,
                                    const double* coefs, int32_t device);
void generated_view(const GeneratedCsr* g, lsamgdd_csr* out);
void generated_export(const GeneratedCsr* g, int64_t* off, int64_t* col, double* val);
void generated_destroy(GeneratedCsr* g);

}  // namespace lsb
