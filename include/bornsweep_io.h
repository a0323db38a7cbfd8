/*
 * bornsweep_io.h -- the reference's field / trace file formats (host-only C ABI,
 * libbornsweep_host.so): the wire format for fixtures, parity diffs and problem manifests.
 *
 * BPFD field file (proj/src/field.cpp:37-133): 4-byte magic "BPFD", uint32 nx, uint32 ny,
 * uint32 dtype (0 = real64, 1 = complex128), then the payload row-major, x slow
 * (data[ix*ny + iy], complex interleaved re/im), native little-endian.  Errors follow the
 * reference's std::runtime_error texts ("field file: bad magic", "field file: truncated
 * header", "field file: expected real64" / "expected complex128", "field file: truncated
 * payload", "cannot open for reading: <path>", "cannot open for writing: <path>").
 *
 * Return codes as bornsweep.h: 0 ok, BP_EINVAL (1) invalid argument, BP_ERUNTIME (2) the
 * reference's runtime_error cases; message via bp_io_last_error().
 */
#ifndef BORNSWEEP_IO_H
#define BORNSWEEP_IO_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { BP_BPFD_REAL64 = 0, BP_BPFD_COMPLEX128 = 1 };

const char* bp_io_last_error(void);
/* save_field / save_complex_array (field.cpp:75-91,115-122) */
int bp_bpfd_save(const char* path, int32_t nx, int32_t ny, int32_t dtype, const double* data);
/* header only: shape and dtype of a field file */
int bp_bpfd_info(const char* path, int32_t* nx, int32_t* ny, int32_t* dtype);
/* load_real_field / load_complex_field (field.cpp:93-113): dtype must match the file's,
 * nx, ny the file's shape (bp_bpfd_info first) */
int bp_bpfd_load(const char* path, int32_t nx, int32_t ny, int32_t dtype, double* out);
/* export_csv (field.cpp:140-161): "ix,iy,re,im" / "ix,iy,value", 17 significant digits */
int bp_csv_export(const char* path, int32_t nx, int32_t ny, int32_t dtype, const double* data);
/* write_trace_csv (iterate.cpp:155-162): "step,res_l2_rel,res_Reta_rel", 17 significant digits */
int bp_trace_csv_write(const char* path, int32_t n, const double* res_l2, const double* res_reta);

#ifdef __cplusplus
}
#endif

#endif
