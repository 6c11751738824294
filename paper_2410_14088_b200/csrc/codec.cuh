// codec.cuh — launchers of the device codec (codec_cmp.cu, codec_dec.cu).
#pragma once

#include "device_common.cuh"

namespace bmq {

// Compress nblk blocks (descriptors in device memory) into the byte region
// `out` starting at *d_cursor (device). When have_pk is false the blocks'
// scalars (CmpBlock::in) are quantised first into CmpBlock::pk and d_cp;
// otherwise a producer (the fused gate epilogue) already filled both, with
// d_cp zero-initialised before it ran. Payload offsets/sizes land in d_bp and,
// when meta_off is given, in meta_off[id] / meta_size[id].
void launch_compress(cudaStream_t st, const CmpBlock* d_blks, uint64_t nblk, uint32_t nch_max, const DevTables& t,
                     uint8_t* out, uint64_t out_cap, uint64_t* d_cursor, uint64_t* d_range, BlockPlan* d_bp,
                     ChunkPlan* d_cp, uint64_t* meta_off, uint64_t* meta_size, bool virtual_zero, bool have_pk,
                     DevError* d_err, uint64_t* launches);

// The two halves of launch_compress: quantise (unless have_pk) + plan, and
// alloc + zero + emit (which may be launched again after DE_POOL_FULL).
void launch_compress_plan(cudaStream_t st, const CmpBlock* d_blks, uint64_t nblk, uint32_t nch_max,
                          const DevTables& t, BlockPlan* d_bp, ChunkPlan* d_cp, bool have_pk, DevError* d_err,
                          uint64_t* launches);
// edge zeroing + emit: every BlockPlan::out_off already holds its payload's
// device address (~0 = virtual ALL_ZERO)
void launch_compress_emit_placed(cudaStream_t st, const CmpBlock* d_blks, uint64_t nblk, uint32_t nch_max,
                                 const DevTables& t, BlockPlan* d_bp, ChunkPlan* d_cp, DevError* d_err,
                                 uint64_t* launches);
void launch_compress_emit(cudaStream_t st, const CmpBlock* d_blks, uint64_t nblk, uint32_t nch_max,
                          const DevTables& t, uint8_t* out, uint64_t out_cap, uint64_t* d_cursor, uint64_t* d_range,
                          BlockPlan* d_bp, ChunkPlan* d_cp, uint64_t* meta_off, uint64_t* meta_size,
                          bool virtual_zero, uint32_t align, DevError* d_err, uint64_t* launches,
                          uint64_t meta_base = 0, uint64_t meta_tag = 0);

// Decompress nblk payloads into their planar output buffers. mode 0: doubles;
// 1: packed code words, 4 bytes per scalar, in DecBlock::out reinterpreted as
// uint32_t*; 2: no output, dequantised sums only (DecInfo::sumsq, ...);
// 3: no scalars, one DecRow per 32-scalar word into rows (planar word order,
// nch_max * 128 records per block) for a first gate pass that decodes itself.
void launch_decompress(cudaStream_t st, const DecBlock* d_blks, uint64_t nblk, uint32_t nch_max, const DevTables& t,
                       DecInfo* d_info, DecChunk* d_dc, bool check_bound, bool want_sums, DevError* d_err,
                       uint64_t* launches, int mode = 0, uint8_t* zflag = nullptr, uint32_t* imnz = nullptr,
                       DecRow* rows = nullptr, PermSrc* psrc = nullptr);
// (zflag, mode 1: one byte per (block, chunk) marking all-zero chunks, which
// are then not written (k_dec_index); mode 0: one byte per 32-scalar group of
// the output, 0 for an all-zero group that was not stored.)
// (imnz, mode 1 with zflag: set to 1 when a chunk of some block's imaginary
// half is not all zero; mode 0 with zflag: set to 1 when some group flag is
// 0. The caller zeroes it first.)

}  // namespace bmq
