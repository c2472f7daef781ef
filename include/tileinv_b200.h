/*
 * tileinv_b200.h -- C ABI of the B200-native tile Cholesky + selected-inversion
 * path (drop-in for the hot path of the reference `tileinv`, arXiv 2504.19171).
 *
 * Plain pointers, sizes and opaque handles only; no C++ or torch types.  Every
 * call is synchronous and returns a status code (TIB_OK = 0); the message of
 * the last failure on the calling thread is available from
 * tib_last_error_message().  Status codes map one-to-one onto the reference's
 * exception classes (proj/include/tileinv/errors.hpp:8-58) and its Python
 * translation (proj/bindings/module.cpp:131-132).
 *
 * Each entry point names the reference interface it replaces (file:line under
 * /root/reference/proj).  Device-resident objects (factor, selected inverse)
 * stay in HBM until freed; host copies are made only on request.
 */
#ifndef TILEINV_B200_H
#define TILEINV_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes (errors.hpp:8-58) ------------------------------------ */
#define TIB_OK 0
#define TIB_ERR_GENERIC 1          /* tileinv::Error */
#define TIB_ERR_INVALID_ARGUMENT 2 /* InvalidArgumentError */
#define TIB_ERR_NOT_SPD 3          /* NotSpdError{pivot, tile_i, tile_j} */
#define TIB_ERR_SINGULAR_TILE 4    /* SingularTileError */
#define TIB_ERR_CONTRACT 5         /* ContractError */
#define TIB_ERR_CONSISTENCY 6      /* ConsistencyError */
#define TIB_ERR_STRUCTURE 7        /* StructureError */
#define TIB_ERR_PARSE 8            /* ParseError */
#define TIB_ERR_FORMAT 9           /* FormatError */
#define TIB_ERR_CUDA 10            /* device / runtime failure (no reference analogue) */

/* ---- selection presets (selinv.hpp:12-24, module.cpp:34-44) ------------- */
#define TIB_SELECT_ENTRIES 0  /* explicit (r, c) list */
#define TIB_SELECT_DIAGONAL 1 /* "diagonal"  */
#define TIB_SELECT_PATTERN 2  /* "pattern"   */
#define TIB_SELECT_ALL 3      /* "all"       */

typedef struct tib_matrix_s* tib_matrix; /* TiledSymmetricMatrix (storage.hpp:40-44), host */
typedef struct tib_factor_s* tib_factor; /* TiledFactor (storage.hpp:46-51), device */
typedef struct tib_sigma_s* tib_sigma;   /* SelectedInverse (selinv.hpp:61-68), device */

/* ---- library ------------------------------------------------------------ */
const char* tib_version(void);                 /* version.hpp:5 kVersion */
const char* tib_last_error_message(void);      /* what() of the last failure */
/* NotSpdError fields of the last TIB_ERR_NOT_SPD (errors.hpp:38-44). */
int tib_last_not_spd(long* pivot, int* tile_i, int* tile_j);
int tib_device_count(int* count);

/* ---- matrices (host side; input formats) --------------------------------- */
/* generate_arrowhead (matgen.hpp:54, matgen.cpp:59-120), bit-exact values.  */
int tib_matrix_generate(long n, long bandwidth, long thickness, double density, uint64_t seed,
                        int tile_size, tib_matrix* out);
/* generate_arrowhead at density 1 ON THE DEVICE (generate.cu; values
 * bit-identical to tib_matrix_generate and to the reference): the matrix
 * lives as parameters, each sweep generates it straight into its A store (no
 * host copy, no H2D).  Host-side accessors (tiles, write_mm, checksum)
 * materialise the values from the device on first use.                      */
int tib_matrix_generate_device(long n, long bandwidth, long thickness, uint64_t seed, int tile_size, int device,
                               tib_matrix* out);
/* BASELINE config 4 (not generable by the reference, which reads it as Matrix
 * Market, matgen.cpp:321-327): joint INLA precision of an AR1(rho) in time
 * (nt steps) x SPDE (alpha = 2, K = kappa2 I + lattice Laplacian, Q_s =
 * tau^2 K^2) on an nx x ny lattice latent field, time-major, plus p fixed
 * effects (prior precision q_beta, Gaussian likelihood precision tau_y,
 * covariates from SplitMix64 draws of `seed`) as the dense arrow.           */
int tib_matrix_generate_kronecker(int nt, int nx, int ny, int p, double rho, double kappa2, double tau,
                                  double tau_y, double q_beta, uint64_t seed, int tile_size, tib_matrix* out);
/* payload_checksum (storage.cpp:34-48) of the matrix tiles: FNV-1a over the
 * column-major tile keys and b*b payloads, equal to the reference's value
 * for the same matrix.                                                       */
int tib_matrix_checksum(tib_matrix m, uint64_t* out);
/* from_dense (module.cpp:46-74): row-major n x n, lower triangle read.      */
int tib_matrix_from_dense(long n, int tile_size, const double* a, tib_matrix* out);
/* Tiles (i >= j), each b*b row-major, as a TileBlocks payload list.         */
int tib_matrix_from_tiles(long n, int tile_size, long count, const int* ti, const int* tj,
                          const double* payload, tib_matrix* out);
/* read_matrix_market (matgen.cpp:208-319) from a text buffer.                */
int tib_matrix_read_mm(const char* text, size_t len, int tile_size, tib_matrix* out);
/* write_matrix_market (matgen.cpp:146-184); *len_inout is the buffer size; on
 * return the full text size (call with buf = NULL to query).                 */
int tib_matrix_write_mm(tib_matrix m, char* buf, size_t* len_inout);
int tib_matrix_info(tib_matrix m, long* n, int* tile_size, int* n_tiles, long* stored_tiles);
/* stored tiles in column-major tile order; payload is count * b * b doubles */
int tib_matrix_tiles(tib_matrix m, int* ti, int* tj, double* payload);
int tib_matrix_free(tib_matrix m);

/* ---- symbolic analysis (layout.cpp, cholesky.cpp:17-49, selinv.cpp:85-150) */
/* Filled factor pattern of m (symbolic_fill): count, then coordinates.       */
int tib_symbolic_pattern(tib_matrix m, long* count, int* ti, int* tj);
/* Closure of a request over the factor pattern (select_tiles +
 * symbolic_inversion): count, then coordinates; growth_warning optional.    */
int tib_symbolic_closure(tib_matrix m, int preset, const long* rows, const long* cols,
                         long nentries, long* count, int* ti, int* tj, int* growth_warning);
/* Task-model FLOPs of factorize / phase 1 / phase 2.        */
int tib_flops(tib_matrix m, int preset, const long* rows, const long* cols, long nentries,
              double* factorize, double* phase1, double* phase2);

/* ---- task-graph / complexity analyzer (dag.hpp:12-77, dag.cpp:79-342;
 * Python dag_report / export_dot / predict_gemm_count, module.cpp:217-236) --
 * report[9] = {n_tiles, band_b (-1: none), trsm, trmm, lauum, gemm_actual,
 * gemm_predicted (-1: none), critical_path, match}.                          */
/* count_kernels(build_band_arrow_dag(n_tiles, band > 0 ? band : n_tiles))   */
int tib_dag_report(int n_tiles, int band, long long* report);
/* count_kernels(build_dag(closure of the request, filled pattern of m))     */
int tib_dag_report_matrix(tib_matrix m, int preset, const long* rows, const long* cols, long nentries,
                          long long* report);
/* export_dot(assign_cores(build_band_arrow_dag(...), cores) if cores > 0);
 * *len_inout is the buffer size, on return the full text size.              */
int tib_dag_export_dot(int n_tiles, int band, int cores, char* buf, size_t* len_inout);
/* predict_gemm_count (dag.cpp:272-280)                                        */
int tib_predict_gemm_count(int n_tiles, int band, long long* out);

/* ---- factorization (cholesky.hpp:28-33, selinv.cpp:195-237) --------------- */
/* symbolic_cholesky + factorize on `device`.  The factor stays in HBM; the
 * phase-1 transform (U_j, W_kj) is produced in the same column sweep.  On
 * TIB_ERR_NOT_SPD, tib_last_not_spd() carries the global pivot and tile.      */
int tib_factorize(tib_matrix m, int device, tib_factor* out);
int tib_factor_info(tib_factor f, long* n, int* tile_size, long* stored_tiles);
/* Tiles (ti[k], tj[k]) of the factor L, b x b row-major each (host).        */
int tib_factor_get_tiles(tib_factor f, long count, const int* ti, const int* tj, double* payload);
/* Overwrites tiles of L in the device store and recomputes the phase-1
 * transform and the log-determinant: the factor of a matrix that differs from
 * the factored one only in a trailing block (the partitioned single-matrix
 * path: the border block of a rank's local system).  No
 * reference counterpart (the reference has no partitioned mode).           */
int tib_factor_replace_tiles(tib_factor f, long count, const int* ti, const int* tj, const double* payload);
/* 2 * sum_r log L_rr (not a reference API).               */
int tib_factor_logdet(tib_factor f, double* out);
/* Download L (phase = 1) or the phase-1 tiles U/W (phase = 2), column-major
 * tile order, b*b row-major each (the reference TileBlocks payload).          */
int tib_factor_tiles(tib_factor f, int phase, int* ti, int* tj, double* payload);
/* payload_checksum (storage.cpp:34-48) of the L tiles as stored here.         */
int tib_factor_checksum(tib_factor f, uint64_t* out);
int tib_factor_free(tib_factor f);
/* PhaseTag of the factor's tiles (storage.hpp:11-16): 1 = kFactor (L and the
 * phase-1 tiles on the device), 2 = kPhase1 (phase-1 tiles only).          */
int tib_factor_phase(tib_factor f, int* phase);
/* factor_from_tile_file (tileio.cpp:109-117) from host tiles: phase 1 = the
 * factor L (phase 1 then runs on the device), phase 2 = phase-1 tiles U / W
 * (selected inversion skips phase 1 for them, selinv.cpp:355).  Tiles are
 * b*b row-major in any order; every diagonal tile must be present.         */
int tib_factor_from_tiles(long n, int tile_size, int phase, long count, const int* ti, const int* tj,
                          const double* payload, int device, tib_factor* out);

/* ---- STLS tile files (tileio.cpp:30-94, tileio.hpp:9-15), byte-compatible - */
/* "STLS" | u32 version 1 | n | b | N | phase | count, then per tile (column-
 * major) u32 i, u32 j, b*b float64.  Read errors: TIB_ERR_PARSE (bad magic,
 * version, truncation, grid mismatch, upper-triangle tile, unknown phase),
 * TIB_ERR_FORMAT (a file of the wrong phase for the call).                  */
int tib_matrix_read_stls(const char* path, tib_matrix* out);      /* matrix_from_tile_file */
int tib_matrix_write_stls(tib_matrix m, const char* path);         /* write_tile_file, kMatrix */
/* factor_from_tile_file: kFactor (L) or kPhase1 (U / W) files; the factor
 * lives on `device` (the --factor reuse of tileinv_main.cpp:183-185).       */
int tib_factor_read_stls(const char* path, int device, tib_factor* out);
/* phase 1: the factor L as kFactor; phase 2: the phase-1 tiles as kPhase1. */
int tib_factor_write_stls(tib_factor f, int phase, const char* path);

/* ---- selected inversion (selinv.hpp:70-85) -------------------------------- */
/* selected_inverse(const TiledSymmetricMatrix&, request, workers)
 * (selinv.cpp:359-367): factorize -> select -> closure -> phase1 -> phase2.  */
int tib_selected_inverse(tib_matrix m, int preset, const long* rows, const long* cols,
                         long nentries, int device, tib_sigma* out);
/* selected_inverse(const TiledFactor&, request, workers) (selinv.cpp:347-357) */
int tib_selected_inverse_of_factor(tib_factor f, int preset, const long* rows, const long* cols,
                                   long nentries, tib_sigma* out);
int tib_sigma_info(tib_sigma s, long* n, int* tile_size, long* closure_tiles, int* growth_warning);
/* logdet of the factor the result came from.                                  */
int tib_sigma_logdet(tib_sigma s, double* out);
/* Marginal variances diag(Sigma), n doubles (requires the diagonal tiles in
 * the closure; TIB_ERR_CONTRACT otherwise, like entry_from_closure).          */
int tib_sigma_diagonal(tib_sigma s, double* out);
/* extract_entries (selinv.cpp:387-439) for the request the result was built
 * with: count first (rows/cols/vals NULL), then the entries.                 */
int tib_sigma_entries(tib_sigma s, long* count, long* rows, long* cols, double* vals);
/* Closure tiles, column-major tile order, b*b row-major each.                */
int tib_sigma_tiles(tib_sigma s, int* ti, int* tj, double* payload);
/* payload_checksum (storage.cpp:34-48) of the result tiles.                   */
int tib_sigma_checksum(tib_sigma s, uint64_t* out);
/* write_selected_inverse (selinv.cpp:441): the closure tiles, kSelectedInverse. */
int tib_sigma_write_stls(tib_sigma s, const char* path);
int tib_sigma_free(tib_sigma s);

/* ---- batched selected inversion (INLA hyper-parameter sweeps) -------------- */
/* count matrices sharing one tile pattern, run as one batched sweep on device:
 * logdet[count] and diag[count * n] (marginal variances) are written back.   */
int tib_selected_inverse_batch(const tib_matrix* ms, int count, int device, double* logdet,
                               double* diag);

/* ---- dataflow plans (host only; inspection and CPU-side simulation) -------- */
/* Builds the device task plan of one sweep (which = 0: fused factorization +
 * phase 1, which = 1: phase 2 for the request) WITHOUT a GPU and copies it
 * out, as the engine builds it for a launch of `batch` matrices (split > 0:
 * the two-chain order's plan).  sizes[0..9] = {tasks, queue-0 tasks, segments, deps, signals,
 * counters, bp, scratch doubles, executed FLOPs, sizeof(DTask)}; call with
 * NULL buffers to query.  Layouts are the POD structs of taskfmt.hpp.        */
typedef struct tib_resident_s* tib_resident;
int tib_plan_export(tib_matrix m, int preset, const long* rows, const long* cols, long nentries, int which,
                    int crit_workers, int split, int batch, double* sizes, void* tasks, void* segs, void* deps,
                    void* sigs);
/* Two-chain elimination order of a single-matrix call: for a
 * band + arrow tile pattern, order[k] (N entries, may be NULL) = the original
 * tile at position k of [I_0 ascending, I_1 descending, separator, arrow];
 * *split = first position of the second chain, -1 when the pattern admits no
 * such order without fill.  No reference counterpart (the reference
 * eliminates in natural order; results agree to rounding).                  */
int tib_matrix_two_chain_order(tib_matrix m, int* order, int* split);
/* The matrix symmetrically permuted into its two-chain order (host tiles;
 * upper tiles of the original become transposed lower tiles).              */
int tib_matrix_two_chain_permuted(tib_matrix m, tib_matrix* out);

/* ---- timing support (bench.py) -------------------------------------------- */
/* A device-resident copy of m with all sweep stores allocated; each run
 * re-copies A on device and executes the fused factorization + selected
 * inversion (pattern) `reps` times.  Times are CUDA events on the library
 * stream: total over reps and the two sweeps of the last rep.                */
int tib_resident_create(tib_matrix m, int device, tib_resident* out);
/* The same for `count` matrices of one tile pattern, run as one batch (every
 * sweep is one launch for the whole batch; BASELINE config 5).               */
int tib_resident_create_batch(const tib_matrix* ms, int count, int device, tib_resident* out);
int tib_resident_run(tib_resident r, int reps, double* ms_total, double* ms_factor, double* ms_phase2);
int tib_resident_info(tib_resident r, double* task_model_flops, double* executed_flops, double* logdet,
                      long* kernel_launches_per_rep);
int tib_resident_free(tib_resident r);
/* Device-resident run: uploads m once, then `reps` times runs the fused
 * factorize + selected inversion (pattern) from the resident copy; returns
 * the per-rep device time in ms (CUDA events on the sweep stream) and the
 * device time of each sweep phase of the last rep.                            */
int tib_bench_resident(tib_matrix m, int device, int reps, int warmup, double* ms_per_rep,
                       double* ms_factor, double* ms_phase2, double* logdet);

#ifdef __cplusplus
}
#endif

#endif /* TILEINV_B200_H */
