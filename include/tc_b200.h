/*
 * tc_b200.h — C ABI of the B200-native TensorCommitments prover (libtcb200.so).
 *
 * The reference (/root/reference/pkg) has no FFI: its prover entry points are Python
 * functions, and the commit / open / tree ones exist only as contracts in SPEC.md.  Each
 * entry point below is the native body of one of those Python functions; the Python
 * package paper_2602_12630_b200 binds them with ctypes and keeps the
 * reference's names, argument meaning and exception types.
 *
 * Conventions
 *   - Plain pointers and sizes only.  "d_" pointers are CUDA device pointers (e.g. a torch
 *     tensor's data_ptr()), everything else is host memory.
 *   - Field elements cross the ABI in CANONICAL little-endian form (never Montgomery):
 *     as 6 x uint32 limbs on the device (24 B), or as the reference's 21-byte
 *     encode_scalar layout on the host (backend.py:335-336).
 *   - Group elements cross as the reference's 43-byte encode_elem layout
 *     (0x04 || x LE21 || y LE21, infinity = 43 zero bytes; backend.py:309-317).
 *   - A context is bound to one device and one CUDA stream; calls on a context are
 *     stream-ordered, not re-entrant.  SRS handles are read-only after creation and may be
 *     shared by contexts on the same device.
 *   - Every call returns a status; TC_OK = 0.  The message of the last failure on a
 *     context is tc_ctx_last_error().  No exceptions cross the ABI.
 *   - No CPU fallback: every compute entry point launches CUDA kernels and fails with
 *     TC_ERR_CUDA when no device is usable.
 */
#ifndef TC_B200_H
#define TC_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TC_ABI_VERSION 1
#define TC_MAX_AXES 16

/* status codes -> Python exception types of the reference */
enum {
  TC_OK = 0,
  TC_ERR_VALUE = 1,          /* ValueError        (mvpoly.py:30-37, backend.py:319-333) */
  TC_ERR_INDEX = 2,          /* IndexError        (mvpoly.py:57) */
  TC_ERR_ZERO_DIVISION = 3,  /* ZeroDivisionError (field.py:41-42) */
  TC_ERR_BACKEND = 4,        /* BackendError      (backend.py:26-27) */
  TC_ERR_OVERFLOW = 5,       /* OverflowError     (mvpoly.py:546-547) */
  TC_ERR_CUDA = 10,          /* RuntimeError: CUDA failure / no device */
  TC_ERR_MEMORY = 11,        /* MemoryError */
  TC_ERR_ARGUMENT = 12       /* ValueError: malformed call (null pointer, bad dtype) */
};

/* input element types */
enum {
  TC_DTYPE_F16 = 1,
  TC_DTYPE_BF16 = 2,
  TC_DTYPE_F32 = 3,
  TC_DTYPE_F64 = 4,
  TC_DTYPE_FP_LIMBS = 16 /* already field elements: canonical 6 x u32 LE, < p */
};

/* SRS contents */
enum {
  TC_SRS_MONOMIAL = 1,
  TC_SRS_LAGRANGE = 2,
  /* (export / has only) the sub-grid Lagrange sets g^{prod_{j>=i} L_{j,w_j}(tau_j)} for the
   * axis suffixes i = 1..m-1, concatenated in order of i (prod_{j>=i} d_j elements each) */
  TC_SRS_SUBGRID = 4
};

/* commit / open routes (all produce identical bytes: the commitment g^{f_T(tau)} is unique) */
enum {
  TC_ROUTE_AUTO = 0,      /* Lagrange route when the SRS has Lagrange elements */
  TC_ROUTE_MONOMIAL = 1,  /* interpolate -> MSM over monomial SRS (SPEC.md:279 verbatim) */
  TC_ROUTE_LAGRANGE = 2   /* MSM of grid values over g^{L_i(tau)} */
};

typedef struct tc_ctx tc_ctx;
typedef struct tc_srs tc_srs;

int tc_abi_version(void);

/* ---- context ---------------------------------------------------------------------- */
int tc_ctx_create(int device, void* cuda_stream, tc_ctx** out);
int tc_ctx_destroy(tc_ctx* ctx);
int tc_ctx_set_stream(tc_ctx* ctx, void* cuda_stream);
/* Mark a context as one of a forward pipeline's (its own stream, several launches in
 * flight): tc_commit_tree_launch then runs each forward's post-accumulation tail on a
 * low-priority stream so the next forward's MSM blocks are scheduled first. */
int tc_ctx_set_pipelined(tc_ctx* ctx, int on);
int tc_ctx_synchronize(tc_ctx* ctx);
const char* tc_ctx_last_error(const tc_ctx* ctx);
uint64_t tc_ctx_launch_count(const tc_ctx* ctx);
/* per-kernel CUDA-event timing on the ctx stream (bench roofline); clears the stats.
 * "msm.accumulate": Pippenger bucket accumulation, units = bucket entries (mixed adds). */
int tc_ctx_set_profiling(tc_ctx* ctx, int on);
int tc_ctx_kernel_stats(const tc_ctx* ctx, const char* name, double* ms, uint64_t* launches,
                        double* units);
/* Debug: with TC_SCRATCH_GUARD=1 in the environment when the context is created, every
 * scratch buffer gets a 256-byte canary right after its requested size; this checks them
 * all (after synchronising the stream) and returns how many were overwritten (their names
 * in tc_ctx_last_error).  An out-of-bounds-write detector for the kernels' work buffers. */
int tc_ctx_check_guards(tc_ctx* ctx, uint64_t* bad_buffers);

/* ---- setup_srs (Srs SPEC.md:44-50) ----------------------------------
 * Monomial elements g^{prod_j tau_j^{i_j}} in lex order (mvpoly.py:3-5) and, with
 * TC_SRS_LAGRANGE, the grid-Lagrange elements g^{prod_j L_{j,i_j}(tau_j)} on the default
 * grid 1..d_j (mvpoly.py:130-133).  taus_le21: m x 21 bytes (canonical, < p). */
int tc_srs_generate(tc_ctx* ctx, const uint32_t* shape, int m, const uint8_t* taus_le21,
                    int flags, tc_srs** out);
/* SRS from public points (TCSR payload): monomial43 N x 43 B, axis43 m x 43 B.
 * The Lagrange elements and sub-grid sets are derived from the monomial ones on the device
 * (tc_srs_derive_lagrange), so a loaded SRS takes the same fast routes as a generated one. */
int tc_srs_load(tc_ctx* ctx, const uint32_t* shape, int m, const uint8_t* monomial43,
                const uint8_t* axis43, tc_srs** out);
/* Trapdoor-free Lagrange SRS (trapdoors stay with the trusted setup):
 * g^{prod_j L_{j,w_j}(tau_j)} computed from the monomial elements alone by the transpose of
 * the per-axis Newton interpolation applied to group elements.  No-op when present. */
int tc_srs_derive_lagrange(tc_ctx* ctx, tc_srs* srs);
/* export elements [offset, offset+count) as count x 43 B (which = TC_SRS_MONOMIAL |
 * TC_SRS_LAGRANGE), or the m axis elements */
int tc_srs_export(tc_ctx* ctx, const tc_srs* srs, int which, uint64_t offset, uint64_t count,
                  uint8_t* out43);
int tc_srs_export_axis(const tc_srs* srs, uint8_t* out43);
int tc_srs_has(const tc_srs* srs, int which);
/* Build the lazily built tables of an SRS up front (setup, not per commit): for fp16 inputs
 * at scale_bits, the exponent table 2^g G_i of the Lagrange basis (g < scale_bits + 6) the
 * fp16 commit plan reads; a no-op for other dtypes or when it does not fit in memory. */
int tc_srs_prepare(tc_ctx* ctx, tc_srs* srs, int dtype, int scale_bits);
/* device bytes held by the SRS: exponent table, fixed-base window tables, and the bases
 * (affine + Edwards copies of the monomial, Lagrange and sub-grid elements) */
int tc_srs_table_bytes(const tc_srs* srs, uint64_t* exptab_bytes, uint64_t* wintab_bytes,
                       uint64_t* basis_bytes);
uint64_t tc_srs_size(const tc_srs* srs);
int tc_srs_destroy(tc_srs* srs);

/* ---- quantize: RNE(v * 2^scale_bits), negatives -> p - |q| ------------
 * TC_ERR_VALUE when a value is not finite or |v| * 2^scale_bits >= p/2. */
int tc_quantize(tc_ctx* ctx, const void* d_in, int dtype, uint64_t n, int scale_bits,
                uint32_t* d_out_limbs);

/* ---- mvpoly.interpolate_lagrange (mvpoly.py:233-247), default grid, in place ---------- */
int tc_interpolate(tc_ctx* ctx, uint32_t* d_limbs, const uint32_t* shape, int m);

/* ---- mvpoly.evaluate (mvpoly.py:140-161) of a coefficient array at a point ------------- */
int tc_evaluate(tc_ctx* ctx, const uint32_t* d_coeffs, const uint32_t* shape, int m,
                const uint8_t* point_le21, uint8_t* out_y21);

/* ---- mvpoly.open_quotients (mvpoly.py:521-534) ----------------------------------------
 * d_quotients: m x N canonical limbs (each quotient keeps f's shape, mvpoly.py:455-456). */
int tc_open_quotients(tc_ctx* ctx, const uint32_t* d_coeffs, const uint32_t* shape, int m,
                      const uint8_t* omega_le21, uint32_t* d_quotients, uint8_t* out_y21);

/* ---- multi-exponentiation prod_k G_k^{a_k} ---------------------
 * over the SRS's monomial or Lagrange elements (which), scalars canonical device limbs. */
int tc_msm(tc_ctx* ctx, const tc_srs* srs, int which, const uint32_t* d_scalars, uint64_t n,
           uint8_t* out43);

/* ---- tc_commit ----------------------------------------------------------
 * d_in holds N = prod(shape) values of dtype (float dtypes are quantised at scale_bits). */
int tc_commit(tc_ctx* ctx, const tc_srs* srs, const void* d_in, int dtype, int scale_bits,
              int route, uint8_t* out43);
/* count tensors of the SRS's shape (protocol.prover_commit's per-layer loop) */
int tc_commit_batch(tc_ctx* ctx, const tc_srs* srs, const void* const* d_ins, int count,
                    int dtype, int scale_bits, int route, uint8_t* out43);
/* Same with HOST inputs (pinned for an asynchronous upload; pageable works, synchronously):
 * uploaded on a copy stream in groups of `group` (0 = one group) and committed as each
 * group becomes resident.  The entry point a reference-side caller holding numpy / CPU
 * activations binds (protocol.prover_commit). */
int tc_commit_batch_host(tc_ctx* ctx, const tc_srs* srs, const void* const* h_ins, int count,
                         int dtype, int scale_bits, int route, int group, uint8_t* out43);
/* Streaming host-input commits, one call per forward: commits h_cur and overlaps the upload
 * of h_next (the next forward's activations, or NULL) with this commit.  h_cur is taken
 * from the device slot a previous call prefetched it into when the pointers match, else
 * uploaded first.  Buffers passed as h_next must stay unchanged until they are committed. */
int tc_commit_stream(tc_ctx* ctx, const tc_srs* srs, const void* const* h_cur,
                     const void* const* h_next, int count, int dtype, int scale_bits, int route,
                     uint8_t* out43);

/* Forget any upload a previous tc_commit_stream* call prefetched (the caller abandoned its
 * stream of forwards, e.g. a consumer stopped early): the next call uploads h_cur afresh. */
int tc_commit_stream_reset(tc_ctx* ctx);

/* ---- tc_open: y = f_T(omega), pi_i = g^{q_i(tau)} ----------------------- */
int tc_open(tc_ctx* ctx, const tc_srs* srs, const void* d_in, int dtype, int scale_bits,
            const uint8_t* omega_le21, int route, uint8_t* out_y21, uint8_t* out_pi43);
/* count openings (tensor d_ins[i] at point omegas_le21[i*m .. i*m+m)): the quotients of a
 * group of openings feed ONE batched MSM per axis (config 4's many challenges); outputs
 * y (count x 21 B) and pi (count x m x 43 B) in input order, bytes identical to tc_open. */
int tc_open_batch(tc_ctx* ctx, const tc_srs* srs, const void* const* d_ins, int count, int dtype,
                  int scale_bits, const uint8_t* omegas_le21, int route, uint8_t* out_y21,
                  uint8_t* out_pi43);

/* Slice commitments of the opening route for often-challenged tensors (config 4), split so
 * several GPUs can share them: H[c', c] = sum_rest T[c', rest] L_{c, rest} for the tensor
 * slices c' in [row_lo, row_hi) over every SRS slice c of the first axis (d0 each), written
 * as (row_hi - row_lo) x d0 43-byte encodings into the DEVICE buffer d_out43.  Once the d0 x
 * d0 encodings are assembled (e.g. all-gathered), tc_open_batch_sliced opens `count` points
 * of that one tensor from them (pi_0 as a d0^2-point MSM, the other quotients as usual);
 * same bytes as tc_open. */
int tc_open_slices(tc_ctx* ctx, const tc_srs* srs, const void* d_in, int dtype, int scale_bits,
                   uint32_t row_lo, uint32_t row_hi, uint8_t* d_out43);
int tc_open_batch_sliced(tc_ctx* ctx, const tc_srs* srs, const void* d_in, const uint8_t* d_h43,
                         int count, int dtype, int scale_bits, const uint8_t* omegas_le21,
                         uint8_t* out_y21, uint8_t* out_pi43);

/* Commitments of `count` device tensors AND their Terkle tree in one call, all on the device
 * (protocol.prover_commit): the batched commit, the leaves
 * hash_to_scalar(encode_elem(C_l), b"terkle/leaf") hashed on the device, the tree levels
 * (as tc_terkle_build, Lagrange node SRS of <= 64 points), one readback.  Outputs: count x 43
 * B commitments; node commitments level by level (bottom first, capacity *inout_node_count);
 * every level's child values as canonical 24-byte LE limbs (leaves zero-padded to B^L first,
 * then each upper level's; capacity *inout_value_count).  Replaces the reference-side
 * sequence tc_commit per layer + leaf hashing + build. */
int tc_commit_tree(tc_ctx* ctx, const tc_srs* srs, const void* const* d_ins, int count,
                   int dtype, int scale_bits, int route, const tc_srs* node_srs,
                   uint8_t* out_comms43, uint8_t* out_nodes43, uint64_t* inout_node_count,
                   uint8_t* out_values24, uint64_t* inout_value_count);

/* tc_commit_tree in two halves, for pipelining forwards over several contexts: _launch
 * enqueues the commitments, the leaf hashing, the tree and the result readback on ctx's
 * stream and returns (it waits only for the MSM's bucket sizes midway); _finish waits for
 * that readback and writes the outputs of tc_commit_tree.  One launch in flight per ctx.
 * tc_commit_stream_tree_launch is the same for HOST inputs (uploaded on ctx's copy
 * stream).  The ctx stream must be ordered after the producers of d_ins. */
int tc_commit_tree_launch(tc_ctx* ctx, const tc_srs* srs, const void* const* d_ins, int count,
                          int dtype, int scale_bits, int route, const tc_srs* node_srs);
int tc_commit_stream_tree_launch(tc_ctx* ctx, const tc_srs* srs, const void* const* h_ins,
                                 int count, int dtype, int scale_bits, int route,
                                 const tc_srs* node_srs);
int tc_commit_tree_finish(tc_ctx* ctx, uint8_t* out_comms43, uint8_t* out_nodes43,
                          uint64_t* inout_node_count, uint8_t* out_values24,
                          uint64_t* inout_value_count);

/* tc_commit_stream + the device tree of tc_commit_tree, one call per forward
 * (protocol.prover_commit_stream). */
int tc_commit_stream_tree(tc_ctx* ctx, const tc_srs* srs, const void* const* h_cur,
                          const void* const* h_next, int count, int dtype, int scale_bits, int route,
                          const tc_srs* node_srs, uint8_t* out_comms43, uint8_t* out_nodes43,
                          uint64_t* inout_node_count, uint8_t* out_values24,
                          uint64_t* inout_value_count);

/* ---- multi-GPU building blocks (dist.py) ------------------------------------
 * tc_commit_points_launch: commit `count` device tensors (whole layers, or a layer's chunk
 * as a zero-masked copy: a Lagrange-route commitment is linear in the samples, so a chunk's
 * MSM is a partial sum of the layer's commitment) and write their 43-byte encodings into
 * the DEVICE buffer d_out43 — stream-ordered, nothing read back.  Every rank's encodings
 * are then exchanged with one all-gather (NCCL over NVLink), and
 * tc_tree_from_points_launch sums the gathered parts per layer (layer_of: host array, the
 * layer of each part, grouped by ascending layer; NULL = one part per layer), hashes the
 * leaves and builds the Terkle tree on the device; tc_commit_tree_finish collects the
 * per-layer commitments, node points and level values as for tc_commit_tree_launch. */
int tc_commit_points_launch(tc_ctx* ctx, const tc_srs* srs, const void* const* d_ins, int count,
                            int dtype, int scale_bits, int route, uint8_t* d_out43);
int tc_tree_from_points_launch(tc_ctx* ctx, const tc_srs* node_srs, const uint8_t* d_parts43,
                               const uint32_t* layer_of, uint64_t nparts, int n_layers);

/* ---- Terkle build ------------------------------------
 * leaves: n x 21 B field elements.  Pads with zeros to B^L (B = node SRS size,
 * L = max(1, ceil(log_B n))) and commits every node bottom-up; a child node enters its
 * parent as hash_to_scalar(encode_elem(C), b"terkle/node") (backend.py:346-348).
 * out_nodes43 receives all node commitments level by level (bottom first);
 * capacity in nodes is *inout_count, the number written is returned in it. */
int tc_terkle_build(tc_ctx* ctx, const tc_srs* node_srs, const uint8_t* leaves_le21,
                    uint64_t n, uint8_t* out_nodes43, uint64_t* inout_count);

/* ---- host-side verifier primitive (backend.py:219-291), CPU only ------------------------ */
int tc_pairing(const uint8_t* a43, const uint8_t* b43, uint8_t* out_f2_42);

/* tc_verify in the product-of-pairings form, CPU only:
 * e(C * g^-y, g) == prod_i e(pi_i, axis_i * g^-omega_i).  *ok = 1 accept / 0 reject. */
int tc_verify_host(int m, const uint8_t* axis43, const uint8_t* c43, const uint8_t* omega_le21,
                   const uint8_t* y21, const uint8_t* proofs43, int* ok);
/* hash_to_scalar (backend.py:346-348) */
int tc_host_hash_to_scalar(const uint8_t* data, uint32_t n, const uint8_t* tag, uint32_t tn,
                           uint8_t* out21);

/* ---- self-test hooks (host arithmetic of the shared __host__ __device__ core) ----------- */
/* the Terkle child value hash_to_scalar(encode_elem(P), b"terkle/node" | b"terkle/leaf") as
 * the device kernels compute it (register-assembled SHA-256 message), on the host */
int tc_host_hash_point(const uint8_t* p43, int node, uint8_t* out21);
/* canonical a^-1 in F_q (field 0) or F_p (field 1) by method 0 = safegcd (Bernstein-Yang),
 * 1 = Fermat, 2 = binary Euclid — the shared __host__ __device__ code, run on the host */
int tc_host_field_inv(int field, int method, const uint32_t* a, uint32_t* out);
int tc_host_fq_mul(const uint32_t* a, const uint32_t* b, uint32_t* out);   /* canonical */
int tc_host_fp_mul(const uint32_t* a, const uint32_t* b, uint32_t* out);   /* canonical */
int tc_host_g_mul(const uint8_t* k_le21, uint8_t* out43);                  /* k * g */
/* measured mad.lo.u32 throughput of the device at current clocks, in 10^12 ops/s */
int tc_measure_imad_peak(tc_ctx* ctx, double* tops);
/* device field-op check: op 0 = Fq mul, 1 = Fp mul, 2 = Fq add, 3 = Fq sub, 4 = Fq inv */
int tc_debug_field(tc_ctx* ctx, int op, const uint32_t* d_a, const uint32_t* d_b,
                   uint32_t* d_out, uint64_t n);

#ifdef __cplusplus
}
#endif
#endif /* TC_B200_H */
