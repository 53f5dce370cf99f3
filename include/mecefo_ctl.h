/* mecefo_ctl.h — C-ABI of the native host control-plane streams (libmecefo_ctl.so).
 *
 * The degraded step's integer path (failure injection, token sampling) draws
 * from numpy's PCG64 in the reference. This library is a bit-exact C++
 * restatement of those streams so the control plane does not depend on numpy:
 *
 *   - SeedSequence entropy pool + generate_state (numpy bit_generator.pyx,
 *     NEP 19), as used by `np.random.PCG64(seed)`:
 *       reference cluster.py:98  `Generator(PCG64(scenario.seed))`
 *       reference data.py:95-98 `PCG64(SeedSequence((seed, 0xDA7A, i)))`
 *   - PCG64 (XSL-RR 128/64) next_uint64 / buffered next_uint32,
 *   - Generator.random()  (53-bit double)       reference cluster.py:148-150
 *   - Generator.integers(0, high) (Lemire bounded, 32- or 64-bit path)
 *                                               reference cluster.py:160-162
 *
 * Host-only (no CUDA). Every function returns 0 on success or
 * MECEFO_CTL_CONTRACT (1) on a bad argument. Streams are caller-owned
 * structs: copy one to fork the stream.
 */
#ifndef MECEFO_CTL_H
#define MECEFO_CTL_H

#include <stdint.h>
#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif

#define MECEFO_CTL_OK 0
#define MECEFO_CTL_CONTRACT 1
#define MECEFO_CTL_UNRECOVERABLE 2

typedef struct {
    uint64_t state_hi, state_lo; /* 128-bit LCG state */
    uint64_t inc_hi, inc_lo;     /* 128-bit odd increment */
    int32_t has_uint32;          /* numpy's buffered upper half for next_uint32 */
    uint32_t uinteger;
} mecefo_pcg64_t;

/* np.random.PCG64(np.random.SeedSequence(entropy)) where `entropy` is a tuple of
 * n non-negative integers, each given as 64-bit words (n <= 64); n == 1 is
 * np.random.PCG64(seed). */
int mecefo_pcg64_seed(mecefo_pcg64_t* s, const uint64_t* entropy, int32_t n);

/* Raw draws (bit_generator.random_raw / next_uint32). */
int mecefo_pcg64_next_u64(mecefo_pcg64_t* s, uint64_t* out, size_t count);
int mecefo_pcg64_next_u32(mecefo_pcg64_t* s, uint32_t* out, size_t count);

/* Generator.random(size=count): doubles in [0, 1). */
int mecefo_pcg64_random(mecefo_pcg64_t* s, double* out, size_t count);

/* Generator.integers(low, high, size=count) with int64 output, high > low. */
int mecefo_pcg64_integers(mecefo_pcg64_t* s, int64_t low, int64_t high, int64_t* out, size_t count);

/* Ring-successor takeover on one ring of n members (reference cluster.py:207-218,
 * the NDB reassignment of reassign_takeover on one DP rank's stages): failed
 * members in descending order each adopt the first following member that is
 * neither failed nor already adopting. failed[j] != 0 marks member j;
 * executor[j] receives the member that runs j's work (j itself if healthy).
 * Returns MECEFO_CTL_UNRECOVERABLE when some failed member has no adopter. */
int mecefo_ring_route(int32_t n, const uint8_t* failed, int32_t* executor);

#ifdef __cplusplus
}
#endif

#endif /* MECEFO_CTL_H */
