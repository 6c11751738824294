// codec.cuh — launchers of the device codec (codec.cu).
#pragma once

#include "device_common.cuh"

namespace bmq {

// Compress nblk blocks (descriptors in device memory) into the byte region
// `out` starting at *d_cursor (device). Payload offsets/sizes land in d_bp
// and, when meta_off is given, in meta_off[id] / meta_size[id].
void launch_compress(cudaStream_t st, const CmpBlock* d_blks, uint64_t nblk, uint32_t nch_max, const DevTables& t,
                     uint8_t* out, uint64_t out_cap, uint64_t* d_cursor, uint64_t* d_range, BlockPlan* d_bp,
                     ChunkPlan* d_cp, uint64_t* meta_off, uint64_t* meta_size, bool virtual_zero, DevError* d_err,
                     uint64_t* launches);

// Decompress nblk payloads into their planar output buffers.
void launch_decompress(cudaStream_t st, const DecBlock* d_blks, uint64_t nblk, uint32_t nch_max, const DevTables& t,
                       DecInfo* d_info, DecChunk* d_dc, bool check_bound, bool want_sums, DevError* d_err,
                       uint64_t* launches);

}  // namespace bmq
