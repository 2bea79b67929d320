/*
 * spx.h -- C-ABI of libspx.so, the B200 (sm_100a) backend for the scheduled
 * sparse tensor algebra kernels of arXiv 2001.00532 (reference package
 * `spindle`, mounted read-only at /root/reference/pkg/src/spindle).
 *
 * The reference ships no FFI and no lowering/execution modules: SPEC.md
 * specifies them (`lower`, `interpret`, `emit_c`) and the
 * only binary contract it fixes is the emitted-C entry point
 *
 *     void compute(double* out, const double** vals, const int32_t** pos,
 *                  const int32_t** crd, const int32_t* dims);
 *
 * with the parameter order of `Manifest` (ir.py:237-263): one `vals` array
 * per tensor in `Assignment.tensors` order (notation.py:202-209), one
 * (pos, crd) pair per compressed level enumerated tensor-major then
 * level-major (`Manifest.sparse_levels`, ir.py:257-263), and the input
 * dimensions concatenated per tensor (`Manifest.dim_index`, ir.py:249-255).
 *
 * spx_launch() replaces that entry point.  It keeps the Manifest ordering
 * for vals/pos/crd/dims and adds what a GPU launch needs: the selected
 * kernel and its schedule constants (spx_plan), a caller-provided workspace
 * and a CUDA stream.  All array arguments are DEVICE pointers; the pointer
 * tables themselves (vals/pos/crd) and dims live in host memory.
 *
 * Ownership: every buffer is allocated and owned by the caller; the library
 * never allocates or frees device memory.  Launches are asynchronous on the
 * given stream.  The library is reentrant; the only global state is the
 * per-thread error string and a launch counter.
 *
 * Error convention: every entry point returns an int status (0 = OK).
 * The Python host maps the codes onto the reference hierarchy
 * (errors.py:56-77):
 *   SPX_E_ARG          -> SpindleError          (bad argument)
 *   SPX_E_UNSUPPORTED  -> LoweringError         (errors.py:64-65)
 *   SPX_E_CONTRACT     -> ContractViolation     (MaxExact, errors.py:76-77)
 *   SPX_E_BOUNDS       -> OutOfBoundsError      (errors.py:72-73)
 *   SPX_E_CUDA         -> ExecutionError        (errors.py:68-69)
 *   SPX_E_WORKSPACE    -> ExecutionError        (workspace too small)
 */
#ifndef SPX_H_
#define SPX_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SPX_ABI_VERSION 1

/* status codes */
#define SPX_OK 0
#define SPX_E_ARG 1
#define SPX_E_UNSUPPORTED 2
#define SPX_E_CONTRACT 3
#define SPX_E_BOUNDS 4
#define SPX_E_CUDA 5
#define SPX_E_WORKSPACE 6

/* value types (the reference is fp64 everywhere, tensors.py:253; the
 * BASELINE configs 2-4 are fp32) */
#define SPX_F64 0
#define SPX_F32 1
#define SPX_I32 2 /* collectives only */

/*
 * Kernel ids -- one per row of the schedule-shape selection table
 * (DESIGN.md "Kernel table").  params[] carries the
 * schedule constants of the matched shape:
 *
 *  id  kernel                    expression               params
 *  1   SpMV row-split            y(i)=A(i,j)*x(j)  A:ds   [0]=ROWS_PER_TB
 *  2   SpMV warp-per-row         "                        [0]=ROWS_PER_TB [1]=WARPS_PER_TB
 *  3   SpMV nnz-split            "                        [0]=NNZ_PER_TB [1]=NNZ_PER_WARP [2]=NNZ_PER_THREAD
 *                                                         [5]=output strategy: 0 = Atomics (default; y zeroed, red.add), 1 = deterministic carry fix-up
 *  4   SpMM nnz-split            C(i,k)=A(i,j)*B(j,k)     [0]=NNZ_PER_TB [1]=NNZ_PER_WARP [2]=WARP_SIZE [3]=bound (0 = none)
 *                                                         [5]=B-row transport: 0 = default (staged-register path), >0 = cp.async row ring of that depth, <0 = staged-register path
 *  5   SpMM warp-per-row         "                        [0]=ROWS_PER_TB [1]=WARPS_PER_TB [2]=WARP_SIZE [3]=bound
 *                                                         [4]=1: rows longer than max(512, nnz/131072) positions get a whole
 *                                                         CTA, partials folded in range order (workspace: a row list)
 *  6   SDDMM nnz-split           A(i,j)=B(i,j)*C(i,k)*D(j,k)  [0]=NNZ_PER_TB [1]=NNZ_PER_WARP [2]=WARP_SIZE [3]=bound [7]=dense_out
 *  7   TTV fiber-split           A(i,j)=B(i,j,k)*c(k) B:sss   [0]=FIBERS_PER_TB [1]=FIBERS_PER_WARP
 *  8   MTTKRP nnz-split          A(i,j)=B(i,k,l)*C(k,j)*D(l,j) [0]=NNZ_PER_TB [1]=NNZ_PER_WARP [2]=WARP_SIZE [3]=bound
 *  9   MTTKRP slice-split        "                        [0]=SLICES_PER_TB [1]=WARPS_PER_TB
 *                                                         [2]=1: cut slices heavier than max(4096, nnz/8192) leaves into
 *                                                         leaf ranges, partial rows folded in range order (workspace);
 *                                                         0: one warp per slice (a GPU schedule's warp-per-slice)
 *  10  SDDMM row-split           A(i,j)=B(i,j)*C(i,k)*D(j,k)  [0]=ROWS_PER_TB [1]=WARPS_PER_TB [2]=WARP_SIZE [3]=bound [7]=dense_out
 *  11  TTV nnz-split             A(i,j)=B(i,j,k)*c(k) B:sss   [0]=NNZ_PER_TB [1]=NNZ_PER_WARP [2]=NNZ_PER_THREAD
 *                                                         [3]=1: fibers spanning warp chunks folded in chunk order
 *                                                         (deterministic; workspace slots) instead of red.add
 *
 * Operand roles: the kernels address operands by role, and slot[role] gives
 * the role's index in the Manifest tensor order (vals[]/dims[] layout):
 *   SpMV   role 0 = A (ds),  role 1 = x (d)            out = y[M]
 *   SpMM   role 0 = A (ds),  role 1 = B (dd, K x N)    out = C[M x N]
 *   SDDMM  role 0 = B (ds),  role 1 = C (dd, M x K), role 2 = D (dd, N x K)
 *          out = nnz-aligned values [nnz]  (params[7]=1: dense M x N)
 *   TTV    role 0 = B (sss), role 1 = c (d)            out = A[I x J]
 *   MTTKRP role 0 = B (sss), role 1 = C (dd, K x R), role 2 = D (dd, L x R)
 *          out = A[I x R]
 * pos[]/crd[] hold the sparse operand's compressed levels in level order
 * (exactly Manifest.sparse_levels for these expressions).
 *
 * level_sizes[] are the sparse operand's stored slot counts per level
 * (Tensor.level_sizes(), tensors.py:135-145): CSR {M, nnz}; CSF {S, F, nnz}.
 * They are passed so a launch never reads pos[] back to the host.
 */
#define SPX_K_SPMV_ROW 1
#define SPX_K_SPMV_WARP 2
#define SPX_K_SPMV_NNZ 3
#define SPX_K_SPMM_NNZ 4
#define SPX_K_SPMM_ROW 5
#define SPX_K_SDDMM_NNZ 6
#define SPX_K_TTV_FIBER 7
#define SPX_K_MTTKRP_NNZ 8
#define SPX_K_MTTKRP_SLICE 9
#define SPX_K_SDDMM_ROW 10
#define SPX_K_TTV_NNZ 11

typedef struct spx_plan {
  int32_t kernel_id;
  int32_t dtype;
  int32_t params[8];
  int32_t slot[4];
  int64_t level_sizes[4];
} spx_plan;

/* Replaces SPEC.md:447 `compute(out, vals, pos, crd, dims)`. */
int spx_launch(const spx_plan* plan, void* out, const void* const* vals,
               const int32_t* const* pos, const int32_t* const* crd,
               const int32_t* dims, void* workspace, size_t ws_bytes,
               void* stream);

/* Workspace bytes spx_launch needs for this plan (0 if none). */
size_t spx_workspace_size(const spx_plan* plan, const int32_t* dims);

/* Thread-local message describing the last non-zero status. */
const char* spx_last_error(void);

/* Library ABI version (SPX_ABI_VERSION). */
int spx_version(void);

/* Total kernel launches issued by this library since load (all threads). */
uint64_t spx_launch_count(void);

/*
 * Multi-GPU nnz-balanced segment partition -- the `divide` semantics of
 * SPEC.md:248-256 on the fused position variable, snapped to segment
 * boundaries:
 *     chunk    = ceil(nnz / ndev)
 *     target_g = min(g * chunk, nnz)
 *     R_g      = first s in [0, nseg) with seg_start[s] >= target_g
 *     R_0 = 0, R_ndev = nseg
 * seg_start is a HOST array of nseg nondecreasing leaf offsets (CSR: pos[0..M)
 * of the compressed level; CSF slices: pos2[pos1[s]]).  bounds_out receives
 * ndev+1 entries.  Device g owns segments [R_g, R_{g+1}).
 */
int spx_partition(const int32_t* seg_start, int64_t nseg, int64_t nnz,
                  int32_t ndev, int64_t* bounds_out);

/* Same partition computed on the device from a DEVICE seg_start array
 * (CSR pos of the compressed level, length >= nseg).  bounds_out is a DEVICE
 * int64 array of ndev+1 entries. */
int spx_partition_device(const int32_t* seg_start, int64_t nseg, int64_t nnz,
                         int32_t ndev, int64_t* bounds_out, void* stream);

/*
 * Multi-GPU collectives (SURVEY.md §8(b) "spx_comm_init / spx_gather /
 * spx_reduce_rows"; §8(e)): NCCL over NVLink on caller streams, opened with
 * dlopen (libnccl.so.2) so the library has no link-time NCCL dependency and
 * shares the process's NCCL when the host runtime has already loaded it.  The
 * reference has no multi-GPU path; these carry the data-path gathers.
 *
 * spx_comm_available: 1 when libnccl could be opened.
 * spx_comm_unique_id: 128-byte ncclUniqueId into id_out (rank 0; the host
 *   broadcasts it over its own process-group store).
 * spx_comm_init: one communicator per process (rank = global rank; the
 *   current CUDA device is the rank's GPU).
 * spx_comm_init_all: ndev communicators in one process (comms_out[ndev]);
 *   issue their collectives between spx_comm_group(1) and spx_comm_group(0).
 * spx_gather: all-gather of `count` elements per rank (each rank's row shard
 *   padded to the largest), rank-major into recv[nranks*count].
 * spx_reduce_rows: element-wise sum over ranks (in place when send == recv),
 *   for the partial outputs of leaf-exact CSF shards (MTTKRP/TTV).
 * dtype: SPX_F64, SPX_F32 or SPX_I32.
 */
int spx_comm_available(void);
int spx_comm_unique_id(void* id_out);
int spx_comm_init(int nranks, int rank, const void* id, void** comm_out);
int spx_comm_init_all(int ndev, const int* devs, void** comms_out);
int spx_comm_destroy(void* comm);
int spx_comm_info(void* comm, int* nranks, int* rank);
int spx_comm_group(int begin);
int spx_gather(void* comm, const void* send, void* recv, size_t count, int dtype, void* stream);
int spx_reduce_rows(void* comm, const void* send, void* recv, size_t count, int dtype, void* stream);

/* Device self-test: writes the createpolicy.fractional L2::evict_last /
 * evict_first descriptors of this GPU and the constants the kernels use in
 * their place (DEVICE uint64_t[4]).  Parity tests require them equal. */
int spx_selftest(uint64_t* out4, void* stream);

/*
 * Device-side pack: COO on the device -> the
 * reference's coordinate hierarchy, bit-exact with spindle.tensors.pack
 * (tensors.py:212-258) including CooTensor.normalized's duplicate folding
 * (tensors.py:83-90).  The reference has no FFI for pack; these replace the
 * body of `pack` for device-resident inputs and are driven phase by phase
 * by formats.pack_device(), which allocates every output between phases
 * from the counts the previous phase reports.
 *
 * spx_pack_sort: coords_host = host table of `order` DEVICE int32 arrays of
 *   n coordinates; dims = host int64[order]; vals = DEVICE fp64[n].  Writes
 *   ucoords (DEVICE int32[order][n], level-major, first nu entries of each
 *   row used) and uvals (DEVICE fp64[n]) for the nu sorted unique entries,
 *   and info (DEVICE int64[2]) = {nu, first out-of-bounds input index or -1}.
 *   Workspace: spx_pack_workspace_size(n, order) bytes.
 * spx_pack_level: one level of the hierarchy over the nu unique entries.
 *   diff (DEVICE int64[nu], zero before level 0) accumulates the
 *   prefix-change flags; slot (DEVICE int64[nu], zero before level 0) holds
 *   the parent slots on entry and this level's slots on exit.  Dense levels
 *   finish here; compressed levels also write the exclusive scan of diff
 *   into ex and the level's stored count into *count_out (DEVICE int64),
 *   then spx_pack_level_fill writes crd (count entries), pos
 *   (parent_count + 1 entries) and moves slot to this level.
 * spx_pack_vals: vals_out[slot[i]] = uvals[i] (the caller zero-fills
 *   vals_out; dtype SPX_F64 or SPX_F32).
 */
/*
 * Native tensor-file ingest, host-side, for
 * spindle.fileio's formats (fileio.py:66-162): fmt 0 = Matrix Market,
 * 1 = FROSTT.  spx_text_scan reports order, entry count and dims (FROSTT:
 * the last '# dims:' comment, or -1 = infer); spx_text_parse writes 0-based
 * int32 coordinates (level-major, coords[l*n + i]) and fp64 values in file
 * order into HOST buffers and fills inferred FROSTT dims.  Malformed files
 * return SPX_PARSE_ERROR; spx_text_error then gives the reference's error
 * class (1 TensorFileError, 2 HeaderError, 3 EntryBoundsError,
 * 4 EntryValueError, errors.py:28-45), 1-based line and message -- the
 * first error in file order, as fileio.py:66-162 raises it.  Only
 * non-ASCII text, integers past 18 digits, orders outside 1..8 and
 * dimensions past int32 return SPX_PARSE_DEFER (the host runs the
 * reference parser).
 */
/*
 * Runtime compilation for the generic lowering fallback (generic.py): NVRTC
 * for the current device, driver-API launch.  libnvrtc / libcuda are opened
 * with dlopen on first use (nvrtc_path may name the library; NULL = search).
 * spx_jit_launch takes the kernel arguments as a host array of pointers to
 * the argument values (cuLaunchKernel's convention).
 */
int spx_jit_compile(const char* src, const char* kernel, const char* nvrtc_path,
                    void** fn_out);
int spx_jit_launch(void* fn, uint32_t grid, uint32_t block, void** args,
                   void* stream);
const char* spx_jit_log(void);

#define SPX_PARSE_DEFER 1
#define SPX_PARSE_ERROR 2
int spx_text_scan(const char* text, int64_t len, int32_t fmt, int32_t* order_out,
                  int64_t* n_out, int64_t* dims_out);
int spx_text_parse(const char* text, int64_t len, int32_t fmt, int32_t order,
                   int64_t n, int64_t* dims, int32_t* coords, double* vals);
int spx_text_error(int32_t* kind, int64_t* line, char* msg, int64_t cap);

size_t spx_pack_workspace_size(int64_t n, int32_t order);
int spx_pack_sort(const int32_t* const* coords_host, int32_t order,
                  const int64_t* dims, int64_t n, const double* vals,
                  void* ws, size_t ws_bytes, int32_t* ucoords, double* uvals,
                  int64_t* info, void* stream);
/* Same, with level l's i-th coordinate at coords_host[l][i * coord_stride]
 * (coord_stride = order for one row-major (n, order) array, no copies). */
int spx_pack_sort_strided(const int32_t* const* coords_host, int64_t coord_stride,
                          int32_t order, const int64_t* dims, int64_t n,
                          const double* vals, void* ws, size_t ws_bytes,
                          int32_t* ucoords, double* uvals, int64_t* info,
                          void* stream);
size_t spx_pack_level_workspace_size(int64_t nu);
int spx_pack_level(const int32_t* ucoord, int64_t nu, int32_t compressed,
                   int64_t dim, int64_t parent_count, int64_t* diff,
                   int64_t* slot, int64_t* ex, void* ws, size_t ws_bytes,
                   int64_t* count_out, void* stream);
int spx_pack_level_fill(const int32_t* ucoord, int64_t nu,
                        const int64_t* diff, const int64_t* ex, int64_t* slot,
                        int64_t count, int64_t parent_count, int32_t* crd_out,
                        int32_t* pos_out, int64_t* cpar, void* stream);
int spx_pack_vals(const int64_t* slot, const double* uvals, int64_t nu,
                  void* vals_out, int32_t dtype, void* stream);

/*
 * Device-resident COO / hierarchy checks and conversions (formats.DeviceCoo,
 * formats.DeviceTensor), csrc/spx_coo.cu.  Orders 1..8; every array DEVICE
 * unless marked host.
 * spx_coo_check: *first_bad = first input index i (input order) whose
 *   coordinate lies outside [0, dims) -- CooTensor.validate's bounds check
 *   (tensors.py:75-81) -- or UINT64_MAX.  coords_host/dims as spx_pack_sort_strided.
 * spx_unpack: coords_out[l*nleaves + q] = level-l coordinate of stored leaf
 *   slot q, storage order -- Tensor.walk_stored (tensors.py:190-206).
 *   levels = host "ds.." string, pos_host/crd_host = host tables of device
 *   pointers (NULL for dense levels), level_sizes = host int64[order].
 * spx_check_invariants: one compressed level of Tensor.check_invariants
 *   (tensors.py:147-163): *result = min over violations of
 *   (level << 40) | (code << 36) | segment, code 1 malformed pos, 2 pos not
 *   nondecreasing, 3 segment not strictly increasing; UINT64_MAX if none.
 * spx_scatter_dense: out[row-major linearised coords[i]] = vals[i]
 *   (Tensor.to_dense, tensors.py:181-188); dtype SPX_F64 / SPX_F32.
 */
int spx_coo_check(const int32_t* const* coords_host, int64_t coord_stride,
                  int32_t order, const int64_t* dims, int64_t n,
                  uint64_t* first_bad, void* stream);
int spx_unpack(int32_t order, const char* levels, const int64_t* dims,
               const int32_t* const* pos_host, const int32_t* const* crd_host,
               const int64_t* level_sizes, int64_t nleaves, int32_t* coords_out,
               void* stream);
int spx_check_invariants(const int32_t* pos, const int32_t* crd, int64_t count,
                         int64_t ncrd, int32_t level, uint64_t* result,
                         void* stream);
int spx_scatter_dense(const int32_t* const* coords_host, int64_t coord_stride,
                      int32_t order, const int64_t* dims, int64_t n,
                      const void* vals, int32_t dtype, void* out, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* SPX_H_ */
