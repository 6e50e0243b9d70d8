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

/* Smallest / largest numberOfWires the device kernels handle; up to
 * ISQ_MAX_FAST_WIRES the fitness runs in the register-resident kernels, above
 * it (fp64 only, no fused single-block launch) in a block-per-circuit kernel
 * with the 2^n x 2^n state in device scratch, up to the reference's default
 * cap 4^n <= 2^26 (n <= 13, engine.py:43; a raised memory_cap_entries above
 * that is ISQ_ERR_UNSUPPORTED here). */
#define ISQ_MIN_WIRES 2
#define ISQ_MAX_FAST_WIRES 5
#define ISQ_MAX_WIRES 13

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

/* Same on device pointers, enqueued on `stream` (cudaStream_t, may be NULL).
 * Asynchronous: a circuit holding a code that is not a gate of this wire
 * count gets a NaN fitness (the host-buffer entry points return
 * ISQ_ERR_CONFIG instead). */
isq_status isq_fitness_batch_device(int32_t n, int32_t length, int64_t count,
                                    const uint8_t* codes_dev, const double* thetas_dev,
                                    const double* target_dev, double* fitness_dev,
                                    double* unitary_dev, void* stream);

/*
 * Arithmetic of the fitness kernel.  FP64 meets the north-star bound
 * (|dfitness| <= 1e-9 |fitness| + 1e-12 against the reference); FP32 keeps the
 * composed unitary in single precision (gate parameters and the overlap
 * accumulate in double): |dfitness| <= 1e-4 |fitness| + 1e-6, about 1.5x the
 * throughput.  Composition (unitary_out) is always FP64.
 */
#define ISQ_PRECISION_FP64 0
#define ISQ_PRECISION_FP32 1
isq_status isq_fitness_batch_ex(int32_t n, int32_t length, int64_t count, const uint8_t* codes,
                                const double* thetas, const double* target, double* fitness_out,
                                int32_t device, int32_t precision);
isq_status isq_fitness_batch_device_ex(int32_t n, int32_t length, int64_t count,
                                       const uint8_t* codes_dev, const double* thetas_dev,
                                       const double* target_dev, double* fitness_dev,
                                       int32_t precision, void* stream);

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

/* ------------------------------------------------------------------------
 * QEQEA engine (QeqeaEngine, engine.py:266-384).  One handle owns one device
 * bank: committed angles theta[Q], qutrit amplitudes qamp[3][Qt] (complex,
 * axis-major), slot_max[Q], plus per-generation scratch.  Every random draw
 * comes from the counter streams documented in csrc/np_random.cuh, so a
 * generation's result depends only on (seed, generation, bank).
 * ---------------------------------------------------------------------- */
typedef struct isq_qeqea_config {
  int32_t number_of_wires;          /* PopulationConfig.number_of_wires      */
  int32_t size_of_individual;       /* PopulationConfig.size_of_individual   */
  int64_t size_of_population;       /* PopulationConfig.size_of_population   */
  double probability_of_mutation;   /* default 0.3  (engine.py:38)           */
  double mutation_range;            /* default pi/4 (engine.py:39)           */
  int32_t n_meas;                   /* default 1    (engine.py:40)           */
  int32_t rank;                     /* this process's shard of the circuits  */
  int64_t max_generations;          /* default 10,000,000                    */
  double target_fitness;            /* default 0.999                         */
  uint64_t seed;
  int32_t world;                    /* number of ranks sharing the population */
  int32_t precision;                /* ISQ_PRECISION_FP64 (0) or _FP32 (1): fitness arithmetic */
} isq_qeqea_config;

typedef struct isq_generation_record {
  double gen_best;      /* step() return value 0: max fitness of the generation  */
  double gen_mean;      /* step() return value 1: mean fitness of the generation */
  double best_fitness;  /* engine.best_fitness after the generation              */
  double reserved;
} isq_generation_record;

/* Create a handle (PopulationConfig validation engine.py:45-63 ->
 * ISQ_ERR_CONFIG) and initialise the bank on the device from the init streams.
 * target: 2*D*D doubles.  max_batch: record capacity = most generations per
 * isq_qeqea_step call / per begin_batch..read_batch window. */
isq_status isq_qeqea_create(const isq_qeqea_config* cfg, const double* target, int32_t device,
                            int32_t max_batch, void** handle);
isq_status isq_qeqea_destroy(void* handle);
/* Enqueue all subsequent work on an external cudaStream_t (e.g. the stream the
 * caller runs its NCCL collectives on). */
isq_status isq_qeqea_set_stream(void* handle, void* stream);
/* Run up to n generations (QeqeaEngine.step x n, single rank) entirely on the
 * device; stops exactly at the first generation meeting a stop rule
 * (engine.py:354-358).  records[i] describes the i-th generation run; *stop_reason
 * is 0 (running), 1 (target-reached) or 2 (generation-limit). */
isq_status isq_qeqea_step(void* handle, int32_t n, isq_generation_record* records,
                          int32_t* n_done, int32_t* stop_reason);
/* How isq_qeqea_step / isq_ga_step launch their generations (results are
 * identical in every mode):
 *   AUTO     FUSED for <= 8 candidates and <= 4096 gate slots, GRAPH for
 *            <= 2^22 gate slots, else KERNELS
 *   KERNELS  one launch per kernel per generation
 *   GRAPH    16-generation CUDA graphs replayed on the handle's stream
 *   FUSED    n generations in one single-block launch */
#define ISQ_LAUNCH_AUTO 0
#define ISQ_LAUNCH_KERNELS 1
#define ISQ_LAUNCH_GRAPH 2
#define ISQ_LAUNCH_FUSED 3
isq_status isq_qeqea_set_launch_mode(void* handle, int32_t mode);
/*
 * Split-phase generation (population sharding over `world` ranks, one GPU
 * each).  Rank r scores circuits [r*S, (r+1)*S) (S = shard,
 * padded) and owns the bank slots of positions [b[r], b[r+1]) of every slot
 * kind and individual (b = isq_qeqea_exchange_buffers.position_bounds); the
 * touches of position p always go to its owner.  Per generation, on the
 * handle's stream (isq_qeqea_buffers / exchange.stream):
 *   isq_qeqea_prepare   sample this rank's circuits; world > 1: group their
 *                       touches by owner into send_flats
 *   [caller]            all-to-all send_flats -> recv_flats: S*(b[o+1]-b[o])
 *                       uint32 to / from each rank o, in rank order
 *   isq_qeqea_values    owned touches: live slot + measured gate code (world 1: no-op,
 *                       prepare already did it)
 *   [caller]            all-to-all send_codes -> recv_codes (uint8) and send_thetas
 *                       -> recv_thetas (double): S*(b[r+1]-b[r]) to each rank,
 *                       S*(b[o+1]-b[o]) from rank o
 *   isq_qeqea_score     compose + score this rank's circuits into fitness[r*S ..];
 *                       world > 1: also this shard's best circuit into elite[r]
 *   [caller]            all-gather fitness (world*S doubles, S per rank) and
 *                       elite (world*elite_len doubles) in place
 *   isq_qeqea_finish    reductions, best-so-far (+ gates from the elite of the
 *                       rank holding it), commit + table update of the owned
 *                       touches, advance / stop
 * World 1: isq_qeqea_eval == prepare + score and no collective is needed.
 * begin_batch marks the start of a record window (read_batch).
 */
isq_status isq_qeqea_begin_batch(void* handle);
isq_status isq_qeqea_eval(void* handle);
isq_status isq_qeqea_prepare(void* handle);
isq_status isq_qeqea_values(void* handle);
isq_status isq_qeqea_score(void* handle);
isq_status isq_qeqea_finish(void* handle);

#define ISQ_MAX_WORLD 64
typedef struct isq_qeqea_exchange_buffers {
  int32_t world, rank;
  int64_t shard;                               /* S                                   */
  int32_t elite_len;                           /* doubles per rank in `elite`         */
  int32_t position_bounds[ISQ_MAX_WORLD + 1];  /* rank o owns [b[o], b[o+1])          */
  void* send_flats;   /* uint32 S*L, grouped by owner (world > 1, else NULL)          */
  void* recv_flats;   /* uint32 world*S*Lr, rows = global circuits                    */
  void* send_codes;   /* uint8  world*S*Lr  */
  void* recv_codes;   /* uint8  S*L, grouped by owner */
  void* send_thetas;  /* double world*S*Lr  */
  void* recv_thetas;  /* double S*L, grouped by owner */
  void* fitness;      /* double world*S (all-gather in place)                         */
  void* elite;        /* double world*elite_len (all-gather in place)                 */
  void* stream;       /* cudaStream_t of the handle                                    */
} isq_qeqea_exchange_buffers;
isq_status isq_qeqea_exchange(void* handle, isq_qeqea_exchange_buffers* out);

/*
 * NVLink peer transport (the fused alternative to the collectives above):
 * once every rank's exchange buffers are mapped into every process, the
 * producing kernels store straight into the consuming ranks' buffers at the
 * places the collectives would put the data — prepare into the owners'
 * recv_flats, values into the circuit ranks' recv_codes / recv_thetas, score
 * into every rank's fitness and elite — so the data moves while the kernels
 * compute, and the caller only orders the phases with a stream-ordered
 * barrier (e.g. a one-element all-reduce) before prepare and after prepare,
 * values and score.
 *   isq_qeqea_ipc_export  this rank's 5 buffers (recv_flats, recv_codes,
 *                         recv_thetas, fitness, elite) as cudaIpcMemHandle_t
 *   isq_qeqea_ipc_open    all ranks' handles (world x 5, rank-major) -> maps the
 *                         other ranks' buffers and enables the transport
 *   isq_qeqea_set_peers   the same from device pointers already valid in this
 *                         process (e.g. several ranks' handles on one device);
 *                         NULL disables the transport (back to collectives)
 */
#define ISQ_PEER_BUFFERS 5
typedef struct isq_ipc_handle {
  char bytes[64];
} isq_ipc_handle;
typedef struct isq_qeqea_peer_buffers {
  void *recv_flats, *recv_codes, *recv_thetas, *fitness, *elite;
} isq_qeqea_peer_buffers;
isq_status isq_qeqea_ipc_export(void* handle, isq_ipc_handle* out);
isq_status isq_qeqea_ipc_open(void* handle, const isq_ipc_handle* all);
isq_status isq_qeqea_set_peers(void* handle, const isq_qeqea_peer_buffers* peers);
isq_status isq_qeqea_read_batch(void* handle, isq_generation_record* records, int32_t* n_done,
                                int32_t* stop_reason, uint64_t* generation, double* best_fitness);
/* Stop rule of later generations (engine.py:354-358): pushes a changed
 * engine.cfg.max_generations / target_fitness and engine.stop_reason (0 none,
 * 1 target-reached, 2 generation-limit) to the device, e.g. the reference's
 * resume_experiment(max_generations=...) (harness.py:95-110) replacing
 * engine.cfg and clearing stop_reason, or step() after a stop, which runs
 * another generation as the reference's does (engine.py:318-361). */
isq_status isq_qeqea_set_limits(void* handle, int64_t max_generations, double target_fitness,
                                int32_t stop);
isq_status isq_qeqea_buffers(void* handle, void** fitness_dev, int64_t* shard_len, void** stream);
/* engine.best_gates / best_fitness (gate codes + angles of length L). */
isq_status isq_qeqea_best(void* handle, uint8_t* codes, double* thetas, double* fitness);
/* Committed bank + table + counters (pickling, engine.py:301-304); set_state
 * also serves init from host arrays (init_population injection).  Arrays
 * cover this rank's owned slots in local order (kind, individual, owned
 * position); world 1: the reference's flat order, theta[Q], qamp[3][Qt],
 * slot_max[Q]. */
isq_status isq_qeqea_get_state(void* handle, double* theta, double* qamp, double* slot_max,
                               uint64_t* generation, double* best_fitness, int32_t* stop);
isq_status isq_qeqea_set_state(void* handle, const double* theta, const double* qamp,
                               const double* slot_max, uint64_t generation, double best_fitness,
                               int32_t stop, const uint8_t* best_codes, const double* best_thetas);
/* engine.pop: the live bank (committed values with the pending mutation of
 * the last generation applied); qutrits as Qt x 3 complex (numpy layout). */
isq_status isq_qeqea_live_population(void* handle, double* theta, double* qutrits);
/* Blueprints (flat slots), measured gate codes and live angles of circuits
 * [c0, c1) at the current generation (sample_circuit + construct_segments).
 * World 1 only. */
isq_status isq_qeqea_sample(void* handle, int64_t c0, int64_t c1, int64_t* flats, uint8_t* codes,
                            double* thetas);
/* Fitness vector of the last evaluated generation (P doubles). */
isq_status isq_qeqea_fitness(void* handle, double* out);

/* ------------------------------------------------------------------------
 * GA engine (GaEngine, ga.py:141-214).  Genomes are P x L gate codes + angles
 * resident on the device; same split-phase protocol as the QEQEA handle.
 * ---------------------------------------------------------------------- */
typedef struct isq_ga_config {
  int32_t number_of_wires;   /* GaConfig.number_of_wires                    */
  int32_t size_of_individual;
  int64_t population;        /* default 50                                  */
  double mutation_rate;      /* default 0.1                                 */
  double mutation_range;     /* default pi/8                                */
  double structural_rate;    /* default 0.1                                 */
  int64_t max_generations;
  double target_fitness;
  uint64_t seed;
  int32_t rank;
  int32_t world;
  int32_t precision;         /* ISQ_PRECISION_FP64 (0) or _FP32 (1)        */
  int32_t reserved;
} isq_ga_config;

isq_status isq_ga_create(const isq_ga_config* cfg, const double* target, int32_t device,
                         int32_t max_batch, void** handle);
isq_status isq_ga_destroy(void* handle);
isq_status isq_ga_set_stream(void* handle, void* stream);
isq_status isq_ga_step(void* handle, int32_t n, isq_generation_record* records, int32_t* n_done,
                       int32_t* stop_reason);
isq_status isq_ga_begin_batch(void* handle);
isq_status isq_ga_eval(void* handle);
isq_status isq_ga_finish(void* handle);
isq_status isq_ga_read_batch(void* handle, isq_generation_record* records, int32_t* n_done,
                             int32_t* stop_reason, uint64_t* generation, double* best_fitness);
isq_status isq_ga_buffers(void* handle, void** fitness_dev, int64_t* shard_len, void** stream);
isq_status isq_ga_set_launch_mode(void* handle, int32_t mode);
isq_status isq_ga_best(void* handle, uint8_t* codes, double* thetas, double* fitness);
/* Current genomes (engine.genomes) as P x L codes + angles; set_state injects them. */
isq_status isq_ga_get_state(void* handle, uint8_t* codes, double* thetas, uint64_t* generation,
                            double* best_fitness, int32_t* stop);
isq_status isq_ga_set_state(void* handle, const uint8_t* codes, const double* thetas,
                            uint64_t generation, double best_fitness, int32_t stop,
                            const uint8_t* best_codes, const double* best_thetas);
/* GaEngine counterpart of isq_qeqea_set_limits (ga.py:165-194 stop rule). */
isq_status isq_ga_set_limits(void* handle, int64_t max_generations, double target_fitness,
                             int32_t stop);
isq_status isq_ga_fitness(void* handle, double* out);
/* Parents drawn by SUS in the last finished generation (P int32). */
isq_status isq_ga_parents(void* handle, int32_t* out);

/* ------------------------------------------------------------------------
 * Functional API (the reference's module-level operators, engine.py:105-263,
 * ga.py:62-138) on the device.  The reference draws from a sequential numpy
 * Generator passed by the caller; these take the counter-stream position
 * instead (seed, generation, index -- csrc/np_random.cuh), i.e. exactly the
 * draws the engines make for that unit, so each call reproduces one step of
 * the engine.  Host buffers, synchronous.  Complex arrays are numpy
 * complex128 (interleaved re, im).
 * ---------------------------------------------------------------------- */
/* init_population (engine.py:105-112): thetas[Q], qutrits[Qt][3] from the
 * per-slot init streams (theta uniform, Box-Muller qutrit). */
isq_status isq_init_population(int32_t n, int32_t length, int64_t population, uint64_t seed, double* thetas,
                               double* qutrits, int32_t device);
/* construct_segments (engine.py:156-171): measured axis (0 X, 1 Y, 2 Z) of
 * every qutrit row s from stream (seed, MEASURE, generation, s). */
isq_status isq_construct_segments(int32_t n, int32_t length, int64_t population, int32_t n_meas, uint64_t seed,
                                  uint64_t generation, const double* qutrits, int8_t* axes, int32_t device);
/* sample_circuit (engine.py:174-184) for circuits [c0, c0 + count) of a
 * generation: count * length flat slot indices (Eq. 9). */
isq_status isq_sample_circuits(int32_t n, int32_t length, int64_t population, uint64_t seed, uint64_t generation,
                               int64_t c0, int64_t count, int64_t* flats, int32_t device);
/* mutate_population (engine.py:228-263) at the end of `generation`, in place
 * on thetas[Q] / qutrits[Qt][3] with slot_max[Q]; mutated[s] = 0 untouched,
 * 1 angle mutation, 2 qutrit mutation (uses cfg: wires, length, population,
 * probability_of_mutation, mutation_range, seed). */
isq_status isq_mutate_population(const isq_qeqea_config* cfg, uint64_t generation, double* thetas, double* qutrits,
                                 const double* slot_max, uint8_t* mutated, int32_t device);
/* SegmentFitnessTable (engine.py:202-222) on the device: entries keyed by
 * (flat, position) in a device hash, slot_max[Q].  update: `count`
 * blueprints of `length` flats and their fitness, in order; improved[c * length
 * + p] = 1 when that touch raised its entry (the reference's improved set is
 * the set of their flats).  read: slot_max (nullable), entry count, and
 * (nullable) the entries as keys flat * length + position and values. */
isq_status isq_table_create(int64_t qubit_count, int32_t length, int32_t device, void** table);
isq_status isq_table_destroy(void* table);
isq_status isq_table_update(void* table, int64_t count, const int64_t* blueprints, const double* fitness,
                            uint8_t* improved);
isq_status isq_table_read(void* table, double* slot_max, int64_t* n_entries, int64_t* keys, double* values);
isq_status isq_table_set_slot_max(void* table, const double* slot_max);
/* apply_gate (gates.py:173-184) for gate sequences: acc_out[c] = G_{L-1} ... G_0
 * acc_in[c] (each gate left-multiplied in order, exact gate matrices), for
 * `count` circuits of `length` gate codes / angles and count x 2^n x 2^n
 * complex matrices (numpy complex128); n = 2..13.  compose_gates is
 * acc_in = I; expand_rotation / interaction_gate one gate on I. */
isq_status isq_apply_gates(int32_t n, int32_t length, int64_t count, const uint8_t* codes, const double* thetas,
                           const double* acc_in, double* acc_out, int32_t device);
/* random_genome (ga.py:68-73) of genomes [first, first + count): count * length codes / angles. */
isq_status isq_ga_random_genomes(int32_t n, int32_t length, uint64_t seed, int64_t first, int64_t count,
                                 uint8_t* codes, double* thetas, int32_t device);
/* sus_select (ga.py:95-116): `count` picks from P fitness values, stream (seed, SUS, generation). */
isq_status isq_ga_sus_select(int64_t population, const double* fitness, int64_t count, uint64_t seed,
                             uint64_t generation, int64_t* picks, int32_t device);
/* two_point_crossover cuts (ga.py:81-92) of pairs [first, first + count): (p, q) per pair. */
isq_status isq_ga_crossover_cuts(int32_t length, uint64_t seed, uint64_t generation, int64_t first, int64_t count,
                                 int32_t* cuts, int32_t device);
/* ga_mutate (ga.py:119-138) of children [first, first + count), in place
 * (uses cfg: wires, length, mutation_rate, mutation_range, structural_rate, seed). */
isq_status isq_ga_mutate_genomes(const isq_ga_config* cfg, uint64_t generation, int64_t first, int64_t count,
                                 uint8_t* codes, double* thetas, int32_t device);

/* Diagnostics: measured FP64 (fp64 != 0) or FP32 CUDA-core FMA peak in flop/s
 * on `device` (roofline denominator of the fitness kernel). */
isq_status isq_fma_peak(int32_t fp64, int32_t device, double* flops_per_s);

/* ----------------------------------------------------------------------
 * encoding.py's per-unit operators (encoding.py:40-132), batched: element i
 * is unit `first + i` of the streams the engines draw from -- the mutation
 * stream after the engine's mask and coin draws (mutate_angle / mutate_qutrit:
 * the step mutate_population gives that slot), the measurement stream
 * (estimate_axis, as construct_segments), (MEASURE, sub 1) for
 * measure_qutrit, the init stream (random_angle / random_qutrit).  Qutrits
 * are count x 3 complex128.  The Born entries return ISQ_ERR_INVARIANT
 * (InvariantViolation) when a norm² deviates from 1 by more than 1e-6.
 * ---------------------------------------------------------------------- */
/* mutate_angle (encoding.py:45-53): out[i] = (theta + sign (1 - f) range) mod 2 pi. */
isq_status isq_mutate_angles(int64_t count, const double* thetas, const double* segment_fitness,
                             double mutation_range, uint64_t seed, uint64_t generation, int64_t first, double* out,
                             int32_t device);
/* mutate_qutrit (encoding.py:119-132): one SU(3) parameter scaled by (1 - f), renormalised. */
isq_status isq_mutate_qutrits(int64_t count, const double* qutrits, const double* segment_fitness, uint64_t seed,
                              uint64_t generation, int64_t first, double* out, int32_t device);
/* born_probabilities (encoding.py:66-71): probs[count][3]. */
isq_status isq_born_probabilities(int64_t count, const double* qutrits, double* probs, int32_t device);
/* estimate_axis (encoding.py:80-84): plurality of multinomial(n_meas, born), ties to the lower axis. */
isq_status isq_estimate_axes(int64_t count, const double* qutrits, int32_t n_meas, uint64_t seed, uint64_t generation,
                             int64_t first, int8_t* axes, int32_t device);
/* measure_qutrit (encoding.py:74-77): Generator.choice(3, p=born). */
isq_status isq_measure_qutrits(int64_t count, const double* qutrits, uint64_t seed, uint64_t generation,
                               int64_t first, int8_t* axes, int32_t device);
/* su3_operator (encoding.py:87-116): params[count][8] (theta1..3, phi1..5) -> out[count][3][3] complex128. */
isq_status isq_su3_operators(int64_t count, const double* params, double* out, int32_t device);
/* random_angle / random_qutrit (encoding.py:56-63) on the init streams: thetas[count] (bit-exact
 * uniform(0, 2 pi)), and with with_qutrit a normalised complex Gaussian (Box-Muller) per unit. */
isq_status isq_init_slots(int64_t count, uint64_t seed, int64_t first, int32_t with_qutrit, double* thetas,
                          double* qutrits, int32_t device);

#ifdef __cplusplus
}
#endif

#endif /* ISQ_H */
