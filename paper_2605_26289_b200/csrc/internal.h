// Internal launch helpers shared between translation units.
#pragma once
#include <cuda_runtime.h>
#include "../../include/deltaserve_b200.h"

namespace ds {
void launch_next_draft(const ds_forward_args* a, const ds_kv_store* kv, cudaStream_t stream);
void launch_row_hash(const ds_forward_args* a, const ds_kv_store* kv, uint64_t* row_hash,
                     cudaStream_t stream);
void launch_token_policy(const ds_forward_args* a, const ds_kv_store* kv, uint64_t* row_hash,
                         uint64_t* amax, int model_vocab, cudaStream_t hash_stream,
                         cudaStream_t stream);
}  // namespace ds
