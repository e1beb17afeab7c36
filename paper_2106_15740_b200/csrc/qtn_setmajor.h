// Set-major executor for small networks evaluated over many angle sets.
#pragma once

#include <cstdint>
#include <vector>

#include "qtn_internal.h"

namespace qtn {

struct SetMajor;

// Build from the SMEM-eligible plans of a batch and their tensor recipes
// (network i = plans[k] is batch index gidx[k]; recipes of batch network i
// at rec[offsets[i] .. offsets[i+1])).  Host work + device upload.
int setmajor_build(SetMajor** out, const std::vector<const qtn_plan*>& plans,
                   const std::vector<int32_t>& gidx, const qtn_tensor_recipe* rec,
                   const int64_t* offsets, int32_t n_total);
int64_t setmajor_workspace(const SetMajor* S, int32_t n_sets);
int setmajor_launches(const SetMajor* S, int32_t n_sets);
// bytes per stored element: 8 (complex64 rows) or 16 (complex128 rows)
int setmajor_elem_bytes(const SetMajor* S);
// results[s*n_total + gidx[k]] for every set s
int setmajor_run(SetMajor* S, const double* angles, int32_t n_angles, int32_t n_sets,
                 void* workspace, void* results, void* stream);
void setmajor_destroy(SetMajor* S);

}  // namespace qtn
