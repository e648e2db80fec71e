/*
 * cg_debug.h — inspection hooks of libcg.so (tests and profiling notes only;
 * not part of the evaluation path).
 */
#ifndef CG_DEBUG_H
#define CG_DEBUG_H
#include <stddef.h>
#include <stdint.h>
#include "cg.h"
#ifdef __cplusplus
extern "C" {
#endif
/* Generate and NVRTC-compile (for sm_100a, no GPU needed) the kernel of every
 * fused elementwise / reduction group of a planned graph.  Returns the number
 * compiled, or CG_E_NVRTC with the compiler log and the source in `log`. */
int64_t cgx_codegen_check(cg_graph* g, int num_sms, char* log, size_t cap);
/* CUDA source generated for group `gi` (with its launch geometry as a comment). */
int64_t cgx_kernel_source(cg_graph* g, int gi, int num_sms, char* buf, size_t cap);
/* The internal work stream (cudaStream_t) every kernel of g is launched on, so
 * a harness can time kernels with CUDA events on their own stream. */
void* cgx_work_stream(const cg_graph* g);
#ifdef __cplusplus
}
#endif
#endif
