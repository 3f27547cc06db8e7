/*
 * tk.h -- C ABI of the B200-native symmetric-tensor contraction library (libtk_b200.so).
 *
 * The operations are those of the paper (PAPER.md = arXiv 2508.10076, TensorKit.jl):
 *   tk_space_*    graded vector space V = (+)_a C^{N_a} (x) V^(a) with a duality flag
 *                 (P:880-915 eq. gradedrepresentation/gradedbasis)
 *   tk_tensor_*   block layout of a tensor map W_1(x)..(x)W_N2 -> V_1(x)..(x)V_N1
 *                 (P:204-224 definition; storage t = G_V^dag o t~ o G_W, P:296-316;
 *                 abelian grouping eq. abeliangrouping; fusion-tree pairs and
 *                 the block-diagonal embedding P:1475-1495)
 *   tk_permute    generalized permute with fusion-tree recoupling (Alg. 2 P:471-488,
 *                 Alg. 6, Alg. 10)
 *   tk_contract   pairwise contraction = permute, permute, per-sector GEMM, permute
 *                 (Alg. 4, Alg. 8; reading C1: B uses (p^B, q^B))
 *
 * Conventions:
 *  - Sector labels are int32 tuples of the kind's width: "Z2"/"fZ2" {g}, "U1" {q},
 *    "U1xU1"/"fU1xU1" {N, 2Sz} (fermion parity N mod 2), "SU2" {2j}, "fU1xSU2" {N, 2j} (the Hubbard
 *    fZ2 x U1 x SU2 Deligne product, P:2380-2412 / P:2582-2591; fermion parity N mod 2), "fSU2xSU2"
 *    {2j_charge, 2j_spin} (fZ2 x SU2 x SU2 at half filling; j_charge + j_spin integer,
 *    fermion parity 2j_spin mod 2), "Fib" {0: I, 1: tau}, "Ising" {0: I, 1: sigma, 2: psi} (
 *    their R-symbols are complex, so only planar -- cyclic -- permutes are available: anything that
 *    would braid returns TK_ERR_BRAIDING_UNAVAILABLE).
 *  - A space lists the sectors of the UNDERLYING space V; is_dual = 1 makes it V*. Fusion
 *    trees label a dual leg by the dual sector (reading C6).
 *  - Legs are numbered codomain first, then domain, 0-based in this ABI.
 *  - Layout (readings C4/C5): blocks by coupled sector ascending, each block a column-major
 *    rows x cols matrix, blocks concatenated; trees in a block ordered by (uncoupled labels,
 *    first leg most significant; then inner labels); a tree pair's reduced array is the
 *    strided region at (row_off, col_off), column-major over (cod legs..., dom legs...).
 *  - Fermionic kinds: permute signs follow reading C13 (Koszul sign of the bent order),
 *    fixed by the paper's SVect data under the unitary convention.
 *  - SU(2): F from eq. SU2FSymbol, R^{j1j2}_{j3} = (-1)^{j1+j2-j3}
 *    (reading C8: the printed sign at P:2329 violates the unit axiom), Z phase reading C7.
 *
 * Ownership: tk_space / tk_tensor are immutable, reference-counted host objects; a tensor
 * retains its spaces. All tensor DATA lives in caller-owned device memory (e.g. PyTorch
 * tensors passed as raw pointers); the caller also provides the workspace. The library's
 * only device allocations are the small per-plan descriptor tables, owned by the plan cache.
 * Plans are memoised per (structure, labels, device) in a mutex-guarded, bounded LRU cache
 * (P:1547-1549); a plan's tables are uploaded once, on the device that is current when the
 * plan is first used, in a capture-safe way (relaxed capture mode, a private stream), so the
 * first tk_contract of a new pattern may run inside CUDA-graph capture. A graph captured from
 * tk_* calls references those tables: do not call tk_cache_clear (which frees them) while such
 * a graph is still replayed, nor while another thread is capturing. Layout and workspace
 * queries (tk_*_output, tk_*_workspace) need no device. Float64 data is double[]; ComplexF64
 * is interleaved (re, im). Data pointers must be 8-byte aligned; workspace pointers 256-byte
 * aligned. The C ABI cannot check buffer sizes: data buffers must hold tk_tensor_nelems
 * elements and the workspace the bytes tk_*_workspace returned.
 *
 * Errors: every call returns a tk_status; tk_last_error() returns a thread-local message.
 * Validation errors (every status but TK_ERR_CUDA) are raised before anything is launched, so
 * outputs are untouched. Kernels run asynchronously on the given stream; a failing launch maps
 * to TK_ERR_CUDA (the launch's own status, not an unrelated earlier error) and may leave the
 * earlier launches of the same call enqueued, i.e. the output is then unspecified.
 */
#ifndef TK_H_
#define TK_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  TK_OK = 0,
  TK_ERR_INVALID_ARGUMENT = 1,
  TK_ERR_UNKNOWN_LABEL = 2,        /* a label/sector not valid for the kind */
  TK_ERR_SECTOR_MISMATCH = 3,      /* spaces of different sector kinds combined */
  TK_ERR_SPACE_MISMATCH = 4,       /* contracted legs not dual, or output space != required */
  TK_ERR_INVALID_PERMUTATION = 5,  /* (p, q) not a permutation of the legs */
  TK_ERR_BRAIDING_UNAVAILABLE = 6,
  TK_ERR_MALFORMED_NETWORK = 7,    /* label list inconsistent (repeats, missing open labels) */
  TK_ERR_UNSUPPORTED = 8,
  TK_ERR_WORKSPACE_TOO_SMALL = 9,
  TK_ERR_CUDA = 10
} tk_status;

typedef enum { TK_F64 = 0, TK_C64 = 1 } tk_dtype;

typedef struct tk_space tk_space;
typedef struct tk_tensor tk_tensor;
typedef struct CUstream_st* tk_stream; /* = cudaStream_t; NULL = legacy default stream */

/* ------------------------------------------------------------------ spaces (host) */
/* kind: "Z2" | "fZ2" | "U1" | "U1xU1" | "fU1xU1" | "SU2" | "fU1xSU2" | "fSU2xSU2" | "Fib" | "Ising"
 * (also the Deligne spellings "fZ2xU1xU1", "fZ2xU1xSU2", "fZ2xSU2xSU2" of the three fermionic products;
 * blanks around 'x' are ignored by tk_space_parse, so "fZ2 x U1 x SU2[...]" parses).
 * labels: n_sectors x width int32,
 * degeneracies: n_sectors int64 > 0 (zero entries are dropped). Sectors may be given
 * in any order; they are stored ascending. Duplicate labels -> TK_ERR_INVALID_ARGUMENT. */
tk_status tk_space_create(const char* kind, int32_t n_sectors, const int32_t* labels,
                          const int64_t* degeneracies, int32_t is_dual, tk_space** out);
/* Grammar "U1[-2:3, 0:5]'" / "SU2[0:1, 1/2:2]" / "U1xU1[(1,-1):2]" / "fU1xSU2[(1,1/2):3]";
 * trailing ' = dual. */
tk_status tk_space_parse(const char* text, tk_space** out);
/* n_sectors, total dim = sum N_a d_a, is_dual, label width (any out pointer may be NULL). */
tk_status tk_space_info(const tk_space* s, int32_t* n_sectors, int64_t* dim, int32_t* is_dual,
                        int32_t* width);
/* Copy the underlying sectors (ascending) and degeneracies; arrays sized by tk_space_info. */
tk_status tk_space_sectors(const tk_space* s, int32_t* labels, int64_t* degeneracies);
tk_status tk_space_dual(const tk_space* s, tk_space** out);
void tk_space_retain(tk_space* s);
void tk_space_release(tk_space* s);

/* ----------------------------------------------------------------- tensors (host) */
/* Block layout of W_1..W_{n_dom} -> V_1..V_{n_cod}. Host only. At least one leg
 * (the kind comes from the spaces); rank-0 (scalar) tensors arise from tk_contract_output of full
 * contractions: one 1 x 1 block at the unit sector. */
tk_status tk_tensor_create(tk_dtype dtype, int32_t n_cod, tk_space* const* cod, int32_t n_dom,
                           tk_space* const* dom, tk_tensor** out);
/* Stored scalars (Float64 count; ComplexF64: complex count -- buffer holds 2x doubles). */
tk_status tk_tensor_nelems(const tk_tensor* t, int64_t* n);
/* n_cod, n_dom, dtype, sector width, number of blocks, number of subblocks, key length
 * (int32 per subblock key = width * (n_cod + max(n_cod-2,0) + 1 + n_dom + max(n_dom-2,0))). */
tk_status tk_tensor_info(const tk_tensor* t, int32_t* n_cod, int32_t* n_dom, int32_t* dtype,
                         int32_t* width, int32_t* n_blocks, int32_t* n_subblocks, int32_t* key_len);
/* Per block (ascending coupled label): coupled (width int32), rows, cols, element offset. */
tk_status tk_tensor_blocks(const tk_tensor* t, int32_t* coupled, int64_t* rows, int64_t* cols,
                           int64_t* offset);
/* Per subblock (block by block, fusion tree major, splitting tree minor): the tree-pair key
 * (cod uncoupled, cod inner, coupled, dom uncoupled, dom inner labels; key_len int32),
 * block index, row_off, col_off, extents (n_cod + n_dom int64 each, padded to 8 per subblock),
 * and the flat element offset of element (0,..,0). Any array may be NULL. */
tk_status tk_tensor_subblocks(const tk_tensor* t, int32_t* keys, int32_t* block, int64_t* row_off,
                              int64_t* col_off, int64_t* extents8, int64_t* offset);
void tk_tensor_retain(tk_tensor* t);
void tk_tensor_release(tk_tensor* t);

/* Output HomSpace of a contraction from @tensor labels: C[labC] := A[labA] * B[labB], the
 * first n_cod_C labels of labC forming C's codomain (spaces by the selection rule of Alg. 2,
 * P:471-486). Errors: MALFORMED_NETWORK (repeats / labC != open labels), SPACE_MISMATCH
 * (contracted legs not a ket/bra pair). */
tk_status tk_contract_output(const tk_tensor* A, const int32_t* labA, const tk_tensor* B,
                             const int32_t* labB, const int32_t* labC, int32_t n_cod_C,
                             tk_tensor** C);

/* ---------------------------------------------------------------- device operations */
/* C = alpha * permute(A, (p, q)) + beta * C   (Alg. 2/6/10). p: np codomain legs of C taken
 * from A's legs, q: nq domain legs; C must have exactly the spaces the selection rule gives
 * (else TK_ERR_SPACE_MISMATCH). beta == 0 never reads C. a, c: device pointers, must not
 * overlap. ws/ws_bytes: device workspace (tk_permute_workspace bytes; currently 0). */
tk_status tk_permute_workspace(const tk_tensor* A, const int32_t* p, int32_t np, const int32_t* q,
                               int32_t nq, const tk_tensor* C, size_t* bytes);
tk_status tk_permute(const tk_tensor* A, const void* a, const int32_t* p, int32_t np,
                     const int32_t* q, int32_t nq, const tk_tensor* C, void* c, double alpha,
                     double beta, void* ws, size_t ws_bytes, tk_stream stream);

/* C[labC] = alpha * sum A[labA] B[labB] + beta * C (labels as in tk_contract_output; C must
 * have the HomSpace tk_contract_output returns). conjA/conjB: complex-conjugate the operand
 * (ComplexF64 only; must be 0 for Float64). Workspace holds the permuted operands A~, B~ and
 * C~ (reading C2 tuples) -- query its size with tk_contract_workspace. */
tk_status tk_contract_workspace(const tk_tensor* A, const int32_t* labA, const tk_tensor* B,
                                const int32_t* labB, const tk_tensor* C, const int32_t* labC,
                                size_t* bytes);
tk_status tk_contract(const tk_tensor* A, const void* a, const int32_t* labA, int32_t conjA,
                      const tk_tensor* B, const void* b, const int32_t* labB, int32_t conjB,
                      const tk_tensor* C, void* c, const int32_t* labC, double alpha, double beta,
                      void* ws, size_t ws_bytes, tk_stream stream);

/* Two consecutive contractions, C[labC] = alpha * ((A[labA] B1[labB1] -> T[labT]) [labT] B2[labB2])
 * + beta * C: exactly tk_contract(A, B1 -> T, alpha 1, beta 0) followed by tk_contract(T, B2 -> C,
 * alpha, beta), each reading C2 for its own tuples (the pairwise order of a contraction sequence,
 * P:1414-1420; the MPO steps of the DMRG two-site update, Alg. 12). T is a descriptor only
 * (its HomSpace must be tk_contract_output(A, labA, B1, labB1, labT)); its data is never materialised
 * when both steps are gathered skinny contractions whose output needs no permute -- then one kernel
 * applies both steps per fiber of T with the same per-element arithmetic. Otherwise the two
 * contractions run as they are with T in the workspace. Float64 only (ComplexF64: call tk_contract
 * twice); no conj flags. Data pointers are device memory in the canonical layouts; C is read only
 * if beta != 0; the workspace (size from tk_contract2_workspace, 256-byte aligned) is caller-owned.
 * tk_contract2_workspace also reports (*fused, if non-NULL) whether the pair runs as one kernel.
 * Errors as tk_contract (raised before any launch). */
tk_status tk_contract2_workspace(const tk_tensor* A, const int32_t* labA, const tk_tensor* B1,
                                 const int32_t* labB1, const tk_tensor* T, const int32_t* labT,
                                 const tk_tensor* B2, const int32_t* labB2, const tk_tensor* C,
                                 const int32_t* labC, size_t* bytes, int32_t* fused);
tk_status tk_contract2(const tk_tensor* A, const void* a, const int32_t* labA, const tk_tensor* B1,
                       const void* b1, const int32_t* labB1, const tk_tensor* T, const int32_t* labT,
                       const tk_tensor* B2, const void* b2, const int32_t* labB2, const tk_tensor* C,
                       void* c, const int32_t* labC, double alpha, double beta, void* ws,
                       size_t ws_bytes, tk_stream stream);

/* Low-level Alg. 4 entry (Alg. 8; reading C1: B~ = permute(B, (pB, qB))):
 *   A~ = permute(A, (pA, qA)),  B~ = permute(B, (pB, qB)),  C~ = A~ o B~,
 *   C  = alpha * permute(C~, (pAB, qAB)) + beta * C.
 * The tuples are given explicitly instead of being derived from labels by reading C2, so a caller can
 * fix the operand orders -- for fermionic kinds they are part of the definition (reading C13).
 * tup: the six 0-based tuples concatenated, pA | qA | pB | qB | pAB | qAB; ntup[6]: their lengths.
 * (pA, qA) must permute A's legs and (pB, qB) B's (else TK_ERR_INVALID_PERMUTATION), |qA| == |pB|,
 * leg qA[c] of A and pB[c] of B a ket/bra pair (else TK_ERR_SPACE_MISMATCH), (pAB, qAB) a permutation of
 * the |pA| + |qB| legs of C~ (codomain: pA legs in pA order, domain: qB legs in qB order).
 * tk_contract_tuples_output returns C's HomSpace; data, conj flags, alpha / beta, workspace and stream
 * behave as in tk_contract. */
tk_status tk_contract_tuples_output(const tk_tensor* A, const tk_tensor* B, const int32_t* tup,
                                   const int32_t* ntup, tk_tensor** C);
tk_status tk_contract_tuples_workspace(const tk_tensor* A, const tk_tensor* B, const tk_tensor* C,
                                       const int32_t* tup, const int32_t* ntup, size_t* bytes);
tk_status tk_contract_tuples(const tk_tensor* A, const void* a, int32_t conjA, const tk_tensor* B,
                             const void* b, int32_t conjB, const tk_tensor* C, void* c,
                             const int32_t* tup, const int32_t* ntup, double alpha, double beta,
                             void* ws, size_t ws_bytes, tk_stream stream);

/* ncon-style network contraction (the @tensor network convention):
 * n tensors T[i] with label lists labels[i] (one label per leg, codomain legs first): positive labels
 * are contracted and appear exactly twice -- on two tensors, or twice on one tensor, which is a partial
 * trace (Alg. 3, tk_trace; done first, bosonic and planar kinds); negative labels -1, -2, ..., -m are the open legs, which become the
 * output's legs in that order, the first n_cod_out of them its codomain. `order` lists every positive
 * label; the network is contracted pairwise in that order, a left fold -- each step takes the two
 * tensors holding the next label and contracts all labels they share (tk_contract, reading C2), the
 * running intermediate as the left operand A (two inputs: in list order; for fermionic kinds the
 * operand order is part of the definition, reading C13). Disconnected pieces are joined by outer
 * products at the end. Intermediates live in the workspace (tk_ncon_workspace bytes, 256-byte aligned,
 * caller-owned) together with the pairwise scratch; their leg order is the library's choice (it
 * changes no value): the producer's C~ order, or the consumer's operand order when the consumer would
 * otherwise permute it in a pass of its own. Consecutive steps that tk_contract2 fuses (the abelian MPO
 * pair) run as one kernel. alpha / beta apply to the output only. Errors: MALFORMED_NETWORK, UNKNOWN_LABEL (order), SPACE_MISMATCH (legs or C's HomSpace),
 * WORKSPACE_TOO_SMALL; a single tensor is TK_ERR_UNSUPPORTED (use tk_permute). */
tk_status tk_ncon_output(int32_t n, const tk_tensor* const* T, const int32_t* const* labels, const int32_t* order,
                         int32_t norder, int32_t n_cod_out, tk_tensor** C);
tk_status tk_ncon_workspace(int32_t n, const tk_tensor* const* T, const int32_t* const* labels, const int32_t* order,
                            int32_t norder, int32_t n_cod_out, size_t* bytes);
tk_status tk_ncon(int32_t n, const tk_tensor* const* T, const void* const* data, const int32_t* const* labels,
                  const int32_t* order, int32_t norder, int32_t n_cod_out, const tk_tensor* C, void* c,
                  double alpha, double beta, void* ws, size_t ws_bytes, tk_stream stream);

/* -------------------------------------------------- blockwise truncated SVD */
/* A~ = permute(A, (p, q)) = U S Vh, block by block (eq. svd, "directly acting on the matrix
 * representation" P:799-809; Alg. 9). U: (A~ codomain) <- W, S: W <- W diagonal, Vh: W <- (A~
 * domain), with W the new bond space: one sector per coupled sector c of A~, degeneracy k_c = kept values.
 * Float64 and ComplexF64 (A = U S Vh with unitary-block U, Vh and real S stored in A's dtype). Three steps, all
 * on the caller's workspace (tk_svd_workspace bytes, 256-byte aligned):
 *   tk_svd          permute + one-sided Jacobi SVD of every block (async on `stream`);
 *   tk_svd_truncate synchronises `stream`, reads the spectrum, applies the global truncation rule
 *                   (values sorted descending over all blocks, ties by block then index; a value of block c
 *                   weighs d_c; max_dim > 0 keeps greedily while sum_kept d_c <= max_dim; rel_tol > 0 drops
 *                   the smallest values while sqrt(sum_dropped d_c s^2) <= rel_tol ||A||; both may be set;
 *                   neither: keep all min(rows, cols) values) and returns new host objects W, U, S, Vh, the
 *                   truncation error sqrt(sum_dropped d_c s^2) and ||A|| = sqrt(sum_c d_c sum s^2);
 *   tk_svd_extract  writes U, S, Vh (canonical layouts, caller-owned device buffers) from the workspace.
 * The workspace must not change between the three calls. Blocks with min(rows, cols) > 8192 ->
 * TK_ERR_UNSUPPORTED. Zero singular values give zero U (or Vh) columns. */
tk_status tk_svd_workspace(const tk_tensor* A, const int32_t* p, int32_t np, const int32_t* q, int32_t nq,
                           size_t* bytes);
tk_status tk_svd(const tk_tensor* A, const void* a, const int32_t* p, int32_t np, const int32_t* q, int32_t nq,
                 void* ws, size_t ws_bytes, tk_stream stream);
/* Host copy of all block spectra (sorted descending per block, blocks in A~'s order): n_blocks, per
 * block count min(rows, cols), sigma = concatenation. Synchronises `stream`. Any output may be NULL. */
tk_status tk_svd_spectrum(const tk_tensor* A, const int32_t* p, int32_t np, const int32_t* q, int32_t nq,
                          const void* ws, tk_stream stream, int32_t* n_blocks, int64_t* counts, double* sigma);
tk_status tk_svd_truncate(const tk_tensor* A, const int32_t* p, int32_t np, const int32_t* q, int32_t nq,
                          const void* ws, int64_t max_dim, double rel_tol, tk_stream stream, tk_space** W,
                          tk_tensor** U, tk_tensor** S, tk_tensor** Vh, double* trunc_err, double* norm);
tk_status tk_svd_extract(const tk_tensor* A, const int32_t* p, int32_t np, const int32_t* q, int32_t nq,
                         const void* ws, const tk_tensor* U, void* u, const tk_tensor* S, void* s,
                         const tk_tensor* Vh, void* vh, tk_stream stream);

/* ---------------------------------------------------------- partial trace */
/* C = alpha * permute(trace(A, (pt, qt)), (p, q)) + beta * C (Alg. 3, Alg. 7 P:1225-1257,
 * fusion-tree traces P:1880-1904). nt pairs (1..4): leg pt[i] of A, read as a codomain leg (Alg. 3's
 * "(a_1 ...; b_1^* ...)"), is contracted with leg qt[i], read as a domain leg; they must be a ket/bra pair
 * of one space (else TK_ERR_SPACE_MISMATCH). (p, q) arrange the remaining legs (indices of A's legs);
 * C's spaces follow the Alg. 2 selection rule (tk_trace_output). Planar kinds (Fib, Ising) need the pairs
 * nested in the cyclic leg order; fermionic kinds -> TK_ERR_UNSUPPORTED; Float64 and ComplexF64. Workspace:
 * tk_trace_workspace bytes (A permuted so the pairs close at the tree ends), 256-byte aligned. */
tk_status tk_trace_output(const tk_tensor* A, const int32_t* pt, const int32_t* qt, int32_t nt, const int32_t* p,
                          int32_t np, const int32_t* q, int32_t nq, tk_tensor** C);
tk_status tk_trace_workspace(const tk_tensor* A, const int32_t* pt, const int32_t* qt, int32_t nt, const int32_t* p,
                             int32_t np, const int32_t* q, int32_t nq, const tk_tensor* C, size_t* bytes);
tk_status tk_trace(const tk_tensor* A, const void* a, const int32_t* pt, const int32_t* qt, int32_t nt,
                   const int32_t* p, int32_t np, const int32_t* q, int32_t nq, const tk_tensor* C, void* c,
                   double alpha, double beta, void* ws, size_t ws_bytes, tk_stream stream);
/* Host transfer matrix of the trace on tree pairs (A subblocks x C subblocks); tests / §4.3 example. */
tk_status tk_trace_transfer(const tk_tensor* A, const int32_t* pt, const int32_t* qt, int32_t nt, const int32_t* p,
                            int32_t np, const int32_t* q, int32_t nq, const tk_tensor* C, double* out);

/* --------------------------------------------------------------- instrumentation */
/* Per-phase CUDA-event timing of the NEXT tk_contract call(s) on the same thread: when
 * enabled, tk_contract records events around each launch on its stream; tk_phase_times
 * (after the stream is synchronized) returns milliseconds of [permute A, permute B, GEMM,
 * permute C] for the most recent call, and per-phase algorithmic bytes / flops. */
tk_status tk_profile_enable(int32_t on);
tk_status tk_phase_times(float* ms4, double* bytes4, double* flops);
/* Number of kernel launches issued by the most recent tk_contract / tk_permute call. */
int32_t tk_last_launch_count(void);
/* Roofline terms of one tk_contract through its plan; host only, no launch. out4 =
 * [useful flops sum_c 2 M_c K_c N_c (8 M_c K_c N_c for ComplexF64, reading C21), the GEMM phase's
 * minimum HBM bytes sum_c s (M_c K_c + K_c N_c + M_c N_c), the permute phase's algorithmic bytes
 * (every permuted operand / output element read once and written once, s = 8 or 16 B), the roofline
 * time in seconds sum_c max(flops_c / peak_flops, bytes_c / peak_bytes_per_s) + permute_bytes /
 * peak_bytes_per_s]. Blocks with K_c = 0 count their zero fill (s M_c N_c bytes). */
tk_status tk_contract_roofline(const tk_tensor* A, const int32_t* labA, const tk_tensor* B, const int32_t* labB,
                               const tk_tensor* C, const int32_t* labC, double peak_flops, double peak_bytes_per_s,
                               double* out4);
/* FP64 tensor-pipe probe, so a caller can measure the GEMM phase's roofline denominator in its own
 * process: launches `blocks` CTAs of 256 threads on `stream`; every warp issues iters x 8 independent
 * DMMA m8n8k4 (mma.sync .f64, no memory traffic). *flops = the launch's flop count; the caller times
 * it (CUDA events on `stream`). */
tk_status tk_dmma_probe(int32_t blocks, int64_t iters, tk_stream stream, double* flops);

/* ------------------------------------------------------- topological data (host) */
/* F^{abc}_d[e,f] (e = a(x)b inner, f = b(x)c inner) and R^{ab}_c of the planner's tables,
 * exported so tests can pin them against the oracle. */
tk_status tk_fsymbol(const char* kind, const int32_t* a, const int32_t* b, const int32_t* c,
                     const int32_t* d, const int32_t* e, const int32_t* f, double* out);
tk_status tk_rsymbol(const char* kind, const int32_t* a, const int32_t* b, const int32_t* c,
                     double* out);

/* Transfer matrix of a permute on tree pairs: for A -> permute(A,(p,q)) = C, writes the dense
 * (nsub_A x nsub_C) coefficient matrix (row = A subblock, col = C subblock, subblock order of
 * tk_tensor_subblocks) into out. Host only; for tests and the paper's §4.3 examples. */
tk_status tk_permute_transfer(const tk_tensor* A, const int32_t* p, int32_t np, const int32_t* q,
                              int32_t nq, const tk_tensor* C, double* out);

/* As tk_permute_transfer, but through the planar route (cyclic rotations and bends only, Alg. 1/5
 * P:398-415) that kinds without braiding use; (p, q) must be a cyclic transpose, else
 * TK_ERR_BRAIDING_UNAVAILABLE. kappa_mode < 0 keeps the library's convention (test hook). */
tk_status tk_permute_transfer_planar(const tk_tensor* A, const int32_t* p, int32_t np, const int32_t* q,
                                     int32_t nq, const tk_tensor* C, int32_t kappa_mode, double* out);

const char* tk_last_error(void);
/* Frees every memoised plan (contraction, fused pair, network, permute, trace, SVD) and its device tables. */
void tk_cache_clear(void);
/* Number of memoised plans currently held (all caches; each cache is a bounded LRU). */
int64_t tk_cache_size(void);
const char* tk_version(void);

#ifdef __cplusplus
}
#endif
#endif /* TK_H_ */
