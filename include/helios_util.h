/*
 * helios_util.h -- the data-parallel primitives libhelios.so uses inside
 * helios_build_accel and helios_simulate, exported on caller buffers so the
 * tests can check them against independent implementations (numpy's stable
 * argsort and cumsum).  Hand-written for sm_100a (csrc/sort_scan.cu); no
 * library sort or scan is used on the build or the hot path.
 *
 * Why they exist (DESIGN.md s.7): the acceleration structure that replaces
 * the paper's kd-tree is built from the triangles sorted by Morton
 * code (K2: radix sort), and the lossless packed outputs (the per-pulse
 * waveform support rows and the used return slots, "fullwaveIndex"
 * linkage) are placed by prefix sums of per-pulse lengths.
 *
 * Both calls are blocking (they synchronise `stream`), take CUDA device
 * pointers, allocate their temporary storage from the library's pool, and
 * return 0 on success, 1 for invalid arguments, 2 when out of device memory,
 * 3 for any other CUDA error.
 */
#ifndef HELIOS_UTIL_H_
#define HELIOS_UTIL_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Stable ascending sort of (d_keys[i], d_vals[i]), i < n, by the low
 * key_bits bits of the keys (1..64; higher bits are ignored), in place:
 * LSD radix, 8 bits per pass.  Pairs with equal (masked) keys keep their
 * input order.  n < 2^32. */
int helios_util_sort_pairs_u64(uint64_t* d_keys, uint32_t* d_vals, uint64_t n, int key_bits,
                               void* stream);

/* d_out[i] = sum_{j <= i} d_in[j] (inclusive != 0) or sum_{j < i} d_in[j]
 * (inclusive == 0), modulo 2^64.  d_out may equal d_in. */
int helios_util_scan_u64(const uint64_t* d_in, uint64_t* d_out, uint64_t n, int inclusive,
                         void* stream);

/* Measured fp64 FMA throughput of the device (TFLOP/s, 2 flops per FMA):
 * every SM, 8 independent DFMA chains per thread, timed with CUDA events.
 * The fp64 ceiling of the voxel march and the decisions (DESIGN.md s.7),
 * reported by bench.py beside the copy bandwidth of MEASURED_PEAKS.json. */
int helios_util_fp64_fma_tflops(double* tflops, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* HELIOS_UTIL_H_ */
