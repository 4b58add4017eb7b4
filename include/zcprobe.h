/* zcprobe.h -- measurement probes of the host link and the zero-copy read
 * path (libzcprobe_b200.so).  Tool library, not part of the traversal ABI
 * (include/zcgraph.h): the bench uses zc_link_probe for its measured peaks,
 * tools/ the rest.  Status codes and zc_last_error() are zcgraph.h's. */
#ifndef ZCPROBE_H_
#define ZCPROBE_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Host-link probe: pinned cudaMemcpy H2D GB/s and a zero-copy streaming
 * read kernel GB/s over `bytes` of pinned memory (the denominators). */
int zc_link_probe(int32_t device, uint64_t bytes, int iters, double *memcpy_h2d_gbs,
                  double *zerocopy_read_gbs, double *hbm_read_gbs);

/* Read microbenchmark (the paper's zero-copy toy kernel):
 * warps read chunk_bytes contiguous bytes per request at consecutive
 * (pattern 0) or random (pattern 1) chunk-aligned offsets of a `bytes`
 * buffer allocated by cudaHostAlloc (alloc 0), transparent-huge-page
 * mmap + cudaHostRegister (alloc 1), cudaMalloc (alloc 2), a host-NUMA
 * VMM allocation (cuMemCreate, alloc 3), hugetlbfs 2 MB pages +
 * cudaHostRegister (alloc 4) or cudaMallocManaged preferred on the CPU and
 * accessed-by the device (alloc 5). */
int zc_read_probe(int32_t device, uint64_t bytes, int pattern, uint32_t chunk_bytes, int alloc,
                  int iters, double *gbs);

/* Host-NUMA VMM allocation check: allocates `bytes` with cuMemCreate
 * (CU_MEM_LOCATION_TYPE_HOST_NUMA, node 0), maps it for the device and the
 * CPU, frees it; *granularity = the recommended allocation granularity. */
int zc_vmm_host_probe(int32_t device, uint64_t bytes, uint64_t *granularity);

/* TMA bulk-copy (cp.async.bulk) streaming read of pinned host memory:
 * `chunk`-byte copies into a 4-stage shared-memory ring per CTA. */
int zc_bulk_probe(int32_t device, uint64_t bytes, uint32_t chunk, int ctas_per_sm, int iters,
                  double *gbs);

/* Pinned-allocation cost of `bytes`: mode 0 cudaHostAlloc; 1 mmap + huge
 * pages + `threads`-way first touch + cudaHostRegister; 2 the same with 4 KB
 * pages; 3 mmap + huge pages + cudaHostRegister without prefault. */
int zc_pin_probe(uint64_t bytes, int mode, int threads, double *alloc_s, double *register_s);

/* Gather roofline of the in-HBM control run: G random 4-byte loads per
 * second into a `bytes`-sized device array (16 MB = the K27 visited bitmap,
 * L2-resident); mode 1 adds an atomicOr for 1 load in 16 (the claims). */
int zc_gather_probe(int32_t device, uint64_t bytes, int mode, double *gloads_per_s);

#ifdef __cplusplus
}
#endif
#endif /* ZCPROBE_H_ */
