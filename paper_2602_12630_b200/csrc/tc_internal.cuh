// Host-side runtime shared by all kernels: per-device context bound to one CUDA stream,
// grow-only stream-ordered scratch buffers, status codes and last-error text.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <map>
#include <mutex>
#include <set>
#include <tuple>
#include <string>
#include <vector>

#include "../../include/tc_b200.h"
#include "ec.cuh"

struct tc_ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  int num_sms = 148;
  std::string err;
  struct Buf {
    void* p = nullptr;
    size_t n = 0;
  };
  std::map<std::string, Buf> scratch;
  uint32_t* d_flags = nullptr;   // device status word (quantize overflow / NaN ...)
  uint32_t* h_flags = nullptr;   // pinned mirror
  void* h_stage = nullptr;       // pinned staging for small host<->device transfers
  size_t h_stage_bytes = 0;
  uint64_t launches = 0;         // kernels launched by this ctx (bench accounting)
  // optional per-kernel timing (CUDA events on the ctx stream) for the roofline report
  bool prof = false;
  struct Stat {
    double ms = 0;
    uint64_t launches = 0;
    double units = 0;   // kernel-specific work units (e.g. bucket entries accumulated)
  };
  std::map<std::string, Stat> stats;
  cudaEvent_t ev[2] = {nullptr, nullptr};
  cudaEvent_t ev_mid = nullptr;   // MSM pipeline: entry counts read back (host waits on it)
  // host-input pipeline (tc_commit_batch_host): a copy stream and one event per group
  cudaStream_t copy_stream = nullptr;
  std::vector<cudaEvent_t> copy_ev;
  // streaming commits (tc_commit_stream): two device slots; a slot remembers which host
  // buffers it was filled from so the next call can consume a prefetched upload
  struct Slot {
    std::vector<const void*> host;
    int dtype = 0;
    uint64_t n = 0;
    bool valid = false;
    cudaEvent_t ready = nullptr;
  };
  Slot slot[2];
  // asynchronous commit + tree (tc_commit_tree_launch / _finish): the points and level
  // values are copied into this pinned buffer on the ctx stream, `res_ev` marks completion
  void* h_res = nullptr;
  size_t h_res_bytes = 0;
  cudaEvent_t res_ev = nullptr;
  bool res_pending = false;
  uint64_t res_count = 0, res_nodes = 0, res_values = 0;
  void* h_off = nullptr;   // pinned per-layer part offsets of tc_tree_from_points_launch
  size_t h_off_bytes = 0;
  // TC_SCRATCH_GUARD=1: a canary after the requested size of every scratch buffer, checked
  // by tc_ctx_check_guards (out-of-bounds writes; compute-sanitizer is closed on this pool)
  bool guard = false;
  // deferred MSM finish (commit + tree): with defer_req set, a single-pipeline MSM batch on
  // the block window-sum path leaves its L x nwin prescaled window sums in defer_wsum and
  // does not write the points; the caller's fused tail kernel sums and converts them
  bool defer_req = false;
  // commit + tree launches of a pipeline context: everything after the level-0 bucket
  // accumulation (reduction levels, window sums, tree, readback) runs on a LOW-priority
  // stream, so the next forward's count / scatter / accumulation blocks are dispatched
  // first and this forward's latency-bound tail fills the gaps
  bool tail_split = false;
  bool pipelined = false;   // set by tc_ctx_set_pipelined (the forward pipeline's contexts)
  cudaStream_t tail_stream = nullptr, main_stream = nullptr;
  cudaEvent_t ev_tail = nullptr;
  tc::Ext* defer_wsum = nullptr;
  int defer_nwin = 0, defer_L = 0;
  std::map<std::string, std::pair<void*, size_t>> guards;
};

struct tc_srs {
  int device = 0;
  int m = 0;
  uint32_t shape[TC_MAX_AXES] = {0};
  uint64_t n = 0;
  tc::Aff* monomial = nullptr;   // N affine points, Montgomery form, lex order
  tc::Aff* lagrange = nullptr;   // N affine points g^{L_i(tau)} (optional)
  tc::Aff axis[TC_MAX_AXES];     // g^{tau_j} (host copy)
  tc::EdAff* small_tab[2] = {nullptr, nullptr};   // byte-window tables (monomial, Lagrange), n <= 64
  // sub-grid Lagrange elements g^{prod_{j>=i} L_{j,a_j}(tau_j)} for suffixes i = 1..m-1
  // (commitments of the Lagrange-route opening quotients q_i, which live on axes i..m-1)
  tc::Aff* sublag = nullptr;
  // twisted Edwards copies (x, y, xy) of the bases the Pippenger MSM reads (lazily built)
  tc::EdPk* ed_monomial = nullptr;
  tc::EdPk* ed_lagrange = nullptr;
  tc::EdPk* ed_sublag = nullptr;
  // fixed-base window tables for full-scalar MSMs (openings): for a base range B (key:
  // its first point), FB_NDIG copies 2^(FB_C w) B, w = 0..FB_NDIG-1 (built on first use)
  std::map<const tc::EdPk*, tc::EdPk*> wintab;
  uint64_t wintab_bytes = 0;   // device bytes held by the window tables
  // exponent table of the Lagrange basis for fp16 / bf16 commits (WinPlan mode 3):
  // exptab[k n + i] = 2^k G_i, k < exptab_depth (built on first use, grown on demand)
  tc::EdPk* exptab = nullptr;
  int exptab_depth = 0;
  std::vector<tc::EdPk*> retired;   // superseded (shallower) exponent tables, freed on destroy
  // guards the lazily built tables above when several contexts (threads) share the SRS
  std::mutex mu;
  uint64_t sublag_off[TC_MAX_AXES] = {0};
};

// SRS sizes up to this many points use the fixed-base small-MSM kernel (small_msm.cu)
constexpr uint64_t SMALL_MSM_MAX = 64;

namespace tcrt {

int fail(tc_ctx* ctx, int code, const char* fmt, ...);

#define TC_CUDA(ctx, call)                                                                 \
  do {                                                                                     \
    cudaError_t e_ = (call);                                                               \
    if (e_ != cudaSuccess)                                                                 \
      return tcrt::fail((ctx), TC_ERR_CUDA, "%s failed: %s (%s:%d)", #call,                \
                        cudaGetErrorString(e_), __FILE__, __LINE__);                       \
  } while (0)

#define TC_LAUNCHED(ctx)                                                                   \
  do {                                                                                     \
    (ctx)->launches++;                                                                     \
    cudaError_t e_ = cudaGetLastError();                                                   \
    if (e_ != cudaSuccess)                                                                 \
      return tcrt::fail((ctx), TC_ERR_CUDA, "kernel launch failed: %s (%s:%d)",            \
                        cudaGetErrorString(e_), __FILE__, __LINE__);                       \
  } while (0)

#define TC_TRY(call)          \
  do {                        \
    int s_ = (call);          \
    if (s_ != TC_OK) return s_; \
  } while (0)

// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) for `func` on the calling thread's
// current device, once per (device, kernel, size): the attribute is per device, so a
// process driving several GPUs sets it on each
int func_smem(tc_ctx* ctx, const void* func, int bytes);

// grow-only scratch buffer named `name` of at least `bytes` (stream ordered)
int scratch(tc_ctx* ctx, const char* name, size_t bytes, void** out);
constexpr uint32_t GUARD_BYTES = 256;   // canary size (scratch always allocates >= 256 B of slack)

template <class T>
int scratch_t(tc_ctx* ctx, const char* name, size_t count, T** out) {
  void* p = nullptr;
  int s = scratch(ctx, name, count * sizeof(T) + 16, &p);
  *out = (T*)p;
  return s;
}

inline unsigned blocks_for(uint64_t n, unsigned threads) {
  uint64_t b = (n + threads - 1) / threads;
  return (unsigned)(b ? b : 1);
}

// ---- MSM entry used by commit/open/terkle ----------------------------------------------
enum ScalarKind { SCALAR_FP_CANON = 0, SCALAR_I64 = 1 };

// result = sum_k scalars[k] * bases[k]; bases are device affine points.  out_aff on device
// (one Aff) receives the canonical-Montgomery affine result.
int msm_device(tc_ctx* ctx, ScalarKind kind, const void* d_scalars, const tc::EdPk* d_bases,
               uint64_t n, tc::Aff* d_out);

// L MSMs over the same n bases in one pipeline: d_out[l] = sum_k s_l[k] * bases[k].
// h_ptrs: L device pointers (host array) to n scalars of `dtype` (TC_DTYPE_FP_LIMBS =
// canonical limbs; float dtypes are quantised at scale_bits inside the digit kernel).
// h_boff (optional, host, L entries): MSM l reads the bases d_bases + h_boff[l] (batches of
// MSMs over different slices of one SRS, e.g. the opening slice commitments)
// fbw > 0: d_bases is a fixed-base window table of digit width fbw (srs_window_table,
// fb_ndig(fbw) * n points) and the scalars are canonical F_p: every digit window shares ONE
// set of buckets (no Horner).
// exp_srs (optional): d_bases is exp_srs's full Edwards Lagrange basis; fp16 / bf16 batches
// may then take the exponent-table plan (mode 3, srs_exp_table)
int msm_batch_device(tc_ctx* ctx, int dtype, int scale_bits, const void* const* h_ptrs, int L,
                     const tc::EdPk* d_bases, uint64_t n, tc::Aff* d_out, const uint32_t* h_boff = nullptr,
                     int fbw = 0, tc_srs* exp_srs = nullptr);

// the exponent table of srs's Edwards Lagrange basis `bases` (n points) with >= depth levels
// 2^k G_i (k < depth), or TC_ERR_MEMORY when it does not fit the device-memory budget
int srs_exp_table(tc_ctx* ctx, tc_srs* srs, const tc::EdPk* bases, uint64_t n, int depth, const tc::EdPk** out);

// fixed-base windowed MSMs over canonical F_p scalars: digit windows of c bits, ndig(c) =
// ceil(163 / c) of them (162 bits + the final carry); see WinPlan mode 2 in msm.cu.
// c = 15 (2^14 buckets, 11 windows) for large ranges, 11 (2^10 buckets, 15 windows) for
// small ones, whose MSMs are latency-bound: their one bucket window then fits the
// single-launch block weighting
constexpr int FB_C_LARGE = 15, FB_C_SMALL = 11;
constexpr uint64_t FB_SMALL_N = 1ull << 16;   // config 4 (65536-point quotient ranges): 2^18 -> 119.8 ms, 2^16 -> 118.2 ms
inline int fb_width(uint64_t n) {
  static const uint64_t small_n = getenv("TC_FB_SMALL_N") ? strtoull(getenv("TC_FB_SMALL_N"), nullptr, 10) : FB_SMALL_N;
  return n >= small_n ? FB_C_LARGE : FB_C_SMALL;
}
inline int fb_ndig(int c) { return (163 + c - 1) / c; }
// the window table of the n bases starting at `bases` (fb_ndig(c) * n points, c = fb_width(n)),
// built once per SRS range
int srs_window_table(tc_ctx* ctx, tc_srs* srs, const tc::EdPk* bases, uint64_t n, const tc::EdPk** out);

// Terkle tree on the device over cap = B^L zero-padded canonical leaves (Lagrange node SRS):
// node points level by level (bottom first) into d_pts, no host round trip between levels
// d_levels (optional): receives every level's child values (cap + cap/B + ... + B entries,
// bottom level first) — the tree's `values` without a host recomputation
int terkle_device(tc_ctx* ctx, tc_srs* srs, tc::Fe* d_vals, uint64_t cap, int L, tc::Aff* d_pts,
                  tc::Fe* d_levels = nullptr);
// commit + tree tail in ONE single-block kernel: the count MSMs' window sums (count x nwin
// prescaled Ext, msm_batch_device's deferred finish) -> canonical affine commitments
// (d_pts[0..count)), leaves hash_to_scalar(encode_elem(C), "terkle/leaf") padded to cap,
// every tree level (node points after the commitments, level values in d_levels)
int tree_tail_device(tc_ctx* ctx, tc_srs* node_srs, const tc::Ext* wsum, int count, int nwin, uint64_t cap, int L,
                     tc::Aff* d_pts, tc::Fe* d_levels);
// Terkle leaves hash_to_scalar(encode_elem(C_i), "terkle/leaf") of count device points,
// zero-padded to cap
int leaf_hash_device(tc_ctx* ctx, const tc::Aff* d_comms, int count, uint64_t cap, tc::Fe* d_vals);

// Montgomery affine points -> twisted Edwards affine (x, y, t = x y), batched inversion
int to_edwards_device(tc_ctx* ctx, const tc::Aff* d_in, uint64_t n, tc::EdPk* d_out);
// the Edwards copy of an SRS basis for the Pippenger pipeline (built on first use):
// which = TC_SRS_MONOMIAL | TC_SRS_LAGRANGE, or 0 for the sub-grid Lagrange elements
int srs_edwards(tc_ctx* ctx, tc_srs* srs, int which, const tc::EdPk** out);

// L MSMs over a small SRS (n <= SMALL_MSM_MAX) with canonical F_p scalars, via per-point
// byte-window tables built once per SRS (`which` = TC_SRS_MONOMIAL | TC_SRS_LAGRANGE)
int small_msm_device(tc_ctx* ctx, tc_srs* srs, int which, const void* const* h_ptrs, int L, tc::Aff* d_out);

// trapdoor-free Lagrange elements of `shape` from the Edwards monomial elements of the same
// shape (derive.cu): canonical Montgomery-curve affine points into d_out (n of them)
int derive_lagrange_device(tc_ctx* ctx, const tc::EdPk* d_mono, const uint32_t* shape, int m, tc::Aff* d_out);

// fixed-base batch: out[i] = e_i * g for canonical F_p exponents e (device arrays)
int fixed_base_g(tc_ctx* ctx, const tc::Fe* d_exps, uint64_t n, tc::Aff* d_out);

// quantize n values of dtype into canonical F_p limbs (device -> device)
int quantize_device(tc_ctx* ctx, const void* d_in, int dtype, uint64_t n, int scale_bits,
                    tc::Fe* d_out);

// e_i = prod_j tabs_j[i_j] for the lex index i (per-axis tables concatenated, canonical)
int srs_exponents(tc_ctx* ctx, const std::vector<tc::Fe>& tabs_host, const uint32_t* shape,
                  int m, uint64_t n, tc::Fe* d_exps);

// per-axis Lagrange->monomial interpolation in place (canonical limbs in / out)
int interpolate_device(tc_ctx* ctx, tc::Fe* d_vals, const uint32_t* shape, int m);

// mvpoly.evaluate on device (per-axis Horner), y returned on the host
int evaluate_device(tc_ctx* ctx, const tc::Fe* d_coeffs, const uint32_t* shape, int m,
                    const tc::Fe* point_canon, tc::Fe* h_y);

// Lagrange-route quotients on the grid (no interpolation): r_0 = grid values (consumed);
// per axis a: r_{a+1} = contraction of r_a with lam[a] (Montgomery L_k(omega_a)), and
// q_a[k, rest] = (r_a[k, rest] - r_{a+1}[rest]) * inv[a][k] (Montgomery 1/(z_k - omega_a)).
// q_a is written at d_quotients + a*N (only its first prod_{j>=a} d_j entries); y on host.
// Per-axis weights of a Lagrange-route opening at omega (Montgomery form, axes concatenated):
// lam[k] = L_k(omega_a); inv[k] = 1 / (x_k - omega_a) for x_k != omega_a.  When omega_a is the
// grid node x_j (sj[a] = j, else -1) the quotient's value on that node is the derivative of the
// fibre interpolant, sum_i r[i] L_i'(x_j): der[i] = L_i'(x_j) (zero when sj[a] < 0).
struct LagW {
  std::vector<tc::Fe> lam, inv, der;
  std::vector<int> sj;
};
int open_quotients_lagrange_device(tc_ctx* ctx, tc::Fe* d_vals, const uint32_t* shape, int m, const LagW& W,
                                   tc::Fe* d_quotients, tc::Fe* h_y, bool skip_q0 = false);
// the same for `cnt` openings in one launch per axis (opening o: vals[o], Ws[o], quotients at
// qouts + o m n); h_y receives cnt values
int open_quotients_lagrange_batch(tc_ctx* ctx, const tc::Fe* const* vals, int cnt, const uint32_t* shape, int m,
                                  const std::vector<LagW>& Ws, tc::Fe* qouts, tc::Fe* h_y, bool skip_q0,
                                  const uint64_t* qoff = nullptr, const uint64_t* qstride = nullptr);
// s[o][c' d + c] = (delta_{c c'} - lam_o[c']) inv_o[c], or der_o[c'] in the column c = sj_o,
// for `count` openings (tabs: per opening lam[d] ++ inv[d] ++ der[d], Montgomery form; sj per
// opening, -1 off the grid) — the scalars of pi_0 over slice commitments
int slice_scalars_device(tc_ctx* ctx, const std::vector<tc::Fe>& tabs_host, const std::vector<int>& sj, uint32_t d,
                         uint32_t count, tc::Fe* d_out);

// open_quotients on device: coefficient array (canonical) -> m quotient arrays + y
int open_quotients_device(tc_ctx* ctx, const tc::Fe* d_coeffs, const uint32_t* shape, int m,
                          const tc::Fe* omega_canon, tc::Fe* d_quotients, tc::Fe* h_y, tc::Fe* d_y = nullptr);

}  // namespace tcrt
