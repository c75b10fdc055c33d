// Host-side helpers shared by the C-ABI entry points (error state, device
// check, TMA tensor-map encoding through the driver entry point so the library
// needs no -lcuda link).
#pragma once
#include <cstdint>
#include <cuda.h>
#include <cuda_runtime.h>

int zp_fail(int code, const char* msg);
int zp_fail_cuda(cudaError_t e, const char* where);
int zp_check_device();
// 2-D bf16 tensor map: inner dim `cols` (elements), outer dim `rows`,
// row pitch in bytes, box (box_cols x box_rows), SWIZZLE_128B, OOB -> zero.
int zp_make_tmap_2d_bf16(CUtensorMap* map, const void* base, uint64_t cols, uint64_t rows,
                         uint64_t row_pitch_bytes, uint32_t box_cols, uint32_t box_rows);
// 2-D fp32 tensor map without swizzle (row-major staging tiles, e.g. the
// TMA reduce-add of the backward's dQ).
int zp_make_tmap_2d_f32(CUtensorMap* map, const void* base, uint64_t cols, uint64_t rows,
                        uint64_t row_pitch_bytes, uint32_t box_cols, uint32_t box_rows);
