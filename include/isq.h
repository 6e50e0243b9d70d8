/*
 * libisq — B200-native (sm_100a) QEQEA / GPUGA generation loop for Ising-model
 * circuit synthesis (arXiv 1809.11134), C ABI.
 *
 * The reference (`isingsynth`, pure Python + numpy) has no FFI: its boundary is
 * the engine duck type driven by report.run_engine (report.py:127-168) plus the
 * functional API used by its tests (engine.py:105-263, gates.py:187-195,
 * fitness.py:36-49).  Each entry point below names the reference interface it
 * replaces.  Plain pointers and sizes only; every host pointer is borrowed for
 * the duration of the call; complex matrices are interleaved (re, im) doubles
 * in row-major order, i.e. numpy complex128 C layout.
 *
 * Status codes map onto the reference's exception types (errors.py:1-9):
 *   ISQ_ERR_CONFIG    -> ConfigurationError (ValueError)
 *   ISQ_ERR_INVARIANT -> InvariantViolation (AssertionError)
 *   ISQ_ERR_CUDA      -> RuntimeError (device failure)
 *   ISQ_ERR_UNSUPPORTED -> ConfigurationError (shape this build does not implement)
 * isq_last_error() returns the message of the calling thread's last failure.
 *
 * Gate codes (uint8), shared by the GA genome, the best-circuit readout and
 * isq_fitness_batch (ga.py:47-59 gate_choices order):
 *   code = 3*(wire-1) + axis     rotation, axis X,Y,Z = 0,1,2   (gates.py:30-33,60-64)
 *   code = 3*n + t               ZZ interaction on the t-th wire pair in
 *                                lexicographic order           (gates.py:76-98)
 */
#ifndef ISQ_H
#define ISQ_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef int32_t isq_status;
#define ISQ_OK 0
#define ISQ_ERR_CONFIG 1
#define ISQ_ERR_INVARIANT 2
#define ISQ_ERR_CUDA 3
#define ISQ_ERR_COMM 4
#define ISQ_ERR_UNSUPPORTED 5

/* Smallest / largest numberOfWires the device kernels are compiled for. */
#define ISQ_MIN_WIRES 2
#define ISQ_MAX_WIRES 5

const char* isq_last_error(void);
int32_t isq_abi_version(void);

/*
 * Fitness of `count` explicit circuits of `length` gates each:
 *   fitness[c] = fitness_value(compose_gates(gates_c, n), target)
 * Replaces: gates.py:187-195 compose_gates + fitness.py:36-49 fitness_value
 * (and ga.py:76-78 decode_genome + ga.py:167-170 GA scoring).
 * codes/thetas: count*length, row c = circuit c, position 0 applied first.
 * target: 2*D*D doubles.  unitary_out (nullable): count*2*D*D doubles, receives
 * the composed unitaries (compose_gates).  Host buffers; synchronous.
 */
isq_status isq_fitness_batch(int32_t n, int32_t length, int64_t count, const uint8_t* codes,
                             const double* thetas, const double* target, double* fitness_out,
                             double* unitary_out, int32_t device);

/* Same on device pointers, enqueued on `stream` (cudaStream_t, may be NULL). */
isq_status isq_fitness_batch_device(int32_t n, int32_t length, int64_t count,
                                    const uint8_t* codes_dev, const double* thetas_dev,
                                    const double* target_dev, double* fitness_dev,
                                    double* unitary_dev, void* stream);

/*
 * fitness_value(S_c, T) for `count` explicit dim x dim matrices S (host,
 * count*2*dim*dim doubles) against one target T.  Replaces fitness.py:36-49
 * when the caller already holds a matrix.  Synchronous.
 */
isq_status isq_fitness_of_unitaries(int64_t dim, int64_t count, const double* unitaries,
                                    const double* target, double* fitness_out, int32_t device);

/*
 * Diagnostics (host-side, no device needed): block `block` (1-based) of the
 * Philox4x64-10 stream (seed, domain, gen, index, sub) that the kernels use,
 * i.e. numpy Philox(key=[seed, domain], counter=[0, gen, index, sub]) after
 * `block` counter increments.  out: 4 words.
 */
void isq_philox_block(uint64_t seed, uint64_t domain, uint64_t gen, uint64_t index, uint64_t sub,
                      uint64_t block, uint64_t* out);

/* Diagnostics: measured FP64 (fp64 != 0) or FP32 CUDA-core FMA peak in flop/s
 * on `device` (roofline denominator of the fitness kernel). */
isq_status isq_fma_peak(int32_t fp64, int32_t device, double* flops_per_s);

#ifdef __cplusplus
}
#endif

#endif /* ISQ_H */
