/*
 * glr_b200.h — C ABI of the B200-native GLR hot path (libglr_b200.so).
 *
 * This is the drop-in boundary for the data-parallel core of the reference
 * package `glr` (/root/reference/pkg/src/glr). The reference has no native
 * code of its own: every entry point below replaces a numpy/scipy call site
 * of the reference, cited as file:line. The Python package
 * `paper_2301_03047_b200` (the reference-facing host layer) is the only
 * in-tree caller; INTEGRATION.md shows the ctypes binding a maintainer of the
 * reference would add.
 *
 * Conventions
 *  - Every pointer argument named *_d is a DEVICE pointer owned by the caller.
 *    The library never allocates in a hot call; scratch comes from the caller
 *    through an explicit workspace pointer sized by the matching *_workspace
 *    query.
 *  - `stream` is a cudaStream_t passed as void*; all work is stream-ordered.
 *  - Images are (H, W, C) row-major, channels last, float64 — the reference
 *    layout (glr/__init__.py:3-4). Anchors/positions are int32 (row, col)
 *    pairs of patch top-left corners (glr/patches.py:5-6).
 *  - Return value: GLR_OK or an error code; glr_last_error() gives a
 *    thread-local message. Validation happens before any launch.
 */
#ifndef GLR_B200_H
#define GLR_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
  GLR_OK = 0,
  GLR_ERR_INVALID = 1,     /* bad shape / argument (reference raises ValueError) */
  GLR_ERR_BOUNDS = 2,      /* anchor out of bounds (glr/patches.py:36-40)        */
  GLR_ERR_NONFINITE = 3,   /* non-finite group entries (glr/lowrank.py:54-55)     */
  GLR_ERR_CUDA = 4,        /* CUDA runtime / driver failure                        */
  GLR_ERR_UNSUPPORTED = 5, /* shape outside what the kernels support               */
  GLR_ERR_WORKSPACE = 6    /* workspace too small                                  */
};

/* ---- library ------------------------------------------------------------ */

const char* glr_last_error(void);
int glr_version(void);
/* Number of SMs and compute capability of the current device (sanity probe). */
int glr_device_info(int* sm_count, int* cc_major, int* cc_minor);

/* ---- (1) edges: glr/edges.py:53-85 ---------------------------------------
 * glr_sobel: per-channel 3x3 Sobel correlation with edge-replicate borders,
 * fp64 with scipy.ndimage.correlate's accumulation order (edges.py:53-64).
 * x_d (H,W,C) -> gh_d, gv_d (H,W,C).                                         */
int glr_sobel(const double* x_d, int H, int W, int C, double* gh_d, double* gv_d, void* stream);

/* glr_edge_stack: sign-split thresholding (edges.py:67-85) of gh/gv into
 *  - maps_d  (optional, may be NULL): u8 {0,1} (4,H,W,C) in the order
 *            h_pos, h_neg, v_pos, v_neg (EdgeMaps.as_tuple, edges.py:33-34);
 *  - stack_d (optional): the im2col-friendly "expanded" stack used by the
 *            heat-map GEMM: (H,W,e*4C) elements with element p*4C+m*C+ch of
 *            pixel (r,c) = map_m[r+p][c][ch] for p<e (0 past the last row),
 *            each an E2M1 (fp4) 1.0 / 0.0 code packed two per byte (element
 *            2j in the low nibble of byte j): H*W*e*2C bytes.
 * th is relative to max|g| when relative != 0 (edges.py:79-80).
 * ws_d: 2 doubles of scratch (the two maxima).                              */
int glr_edge_stack(const double* gh_d, const double* gv_d, int H, int W, int C, double th,
                   int relative, int expand, uint8_t* maps_d, uint8_t* stack_d, double* ws_d,
                   void* stream);

/* glr_stack_from_maps: same expanded stack from caller-provided binary maps
 * (4,H,W,C) u8 — the similarity_heatmap(EdgeMaps, ...) entry (matching.py:140). */
int glr_stack_from_maps(const uint8_t* maps_d, int H, int W, int C, int expand, uint8_t* stack_d,
                        void* stream);

/* ---- (1) exemplars: glr/edges.py:88-162, solvers.py:154-167 ---------------
 * glr_corner_response: channel-mean gradient magnitude -> Shi-Tomasi
 * min-eigenvalue response (edges.py:88-97, 110-112), bitwise equal to the
 * reference's fp64 evaluation order. resp_d (H,W). ws: glr_corner_workspace. */
size_t glr_corner_workspace(int H, int W, int C);
int glr_corner_response(const double* x_d, int H, int W, int C, double* resp_d, void* ws_d,
                        void* stream);

/* glr_corner_response_grad: the same response from the Sobel gradients
 * glr_sobel already produced (gh_d, gv_d (H,W,C)): mag = mean_c
 * sqrt(gh^2 + gv^2) is bit-identical to the x-based entry, one Sobel pass
 * fewer when the edge stack needs the gradients anyway. ws as above.       */
int glr_corner_response_grad(const double* gh_d, const double* gv_d, int H, int W, int C,
                             double* resp_d, void* ws_d, void* stream);

/* glr_corners: threshold >= quality*max, order (score desc, row, col), greedy
 * Chebyshev NMS, at most max_n picks (edges.py:113-128).
 * out_rc_d: 2*max_n int32; out_n_d: 1 int32. ws: glr_nms_workspace.          */
size_t glr_nms_workspace(int H, int W);
int glr_corners(const double* resp_d, int H, int W, int max_n, int nms_radius, double quality,
                int32_t* out_rc_d, int32_t* out_n_d, void* ws_d, size_t ws_bytes, void* stream);

/* glr_select_anchors: corners -> clamped top-left anchors, deduplicated in
 * order, then the row-major uniform grid if grid_interval > 0
 * (edges.py:131-162). anchors_d: 2*max_anchors int32; tags_d: u8 per anchor
 * (0 corner, 1 uniform); n_d: 1 int32. ws: glr_anchor_workspace.            */
size_t glr_anchor_workspace(int H, int W);
int glr_select_anchors(const int32_t* corners_rc_d, const int32_t* n_corners_d, int max_corners,
                       int H, int W, int P, int grid_interval, int max_anchors,
                       int32_t* anchors_d, uint8_t* tags_d, int32_t* n_d, void* ws_d,
                       void* stream);

/* ---- (2) global similarity heat map: glr/matching.py:140-167 ---------------
 * heat[n][u*ow+v] = sum_{p,q,ch<4C} E[u+p][v+q][ch] * E[r_n+p][c_n+q][ch],
 * exact integer overlap counts on tcgen05 tensor cores (kind::mxf4: packed
 * fp4 0/1 operands, unit UE8M0 scale factors, f32 accumulation).
 * Exemplar-major u16 output heat[n*stride + u*ow + v], stride =
 * glr_heat_stride(H,W,P) (oh = H-P+1, ow = W-P+1). n_dev_d (optional) caps the exemplar count on device.
 * ws: glr_heat_workspace (the packed exemplar operand).                     */
int glr_heat_expand_factor(int C, int P);
/* Row stride (entries) of the heat map: (H-P+1)*(W-P+1) rounded up to 8.  */
int64_t glr_heat_stride(int H, int W, int P);
size_t glr_heat_workspace(int C, int P, int n_max);
int glr_heat_map(const uint8_t* stack_d, int H, int W, int C, int P, int expand,
                 const int32_t* anchors_d, int n_max, const int32_t* n_dev_d, uint16_t* heat_d,
                 void* ws_d, size_t ws_bytes, void* stream);

/* glr_heat_topk: heat map + top-K fused (matching.py:140-231) without
 * materialising the heat map: the GEMM epilogue appends, per exemplar n, every
 * position whose score reaches |E_n|/4 (a quarter of the exemplar's
 * self-score, the row maximum) to a list of capacity `cap`; the exact top-K
 * (same semantics as glr_topk) then runs on the lists. An exemplar whose cut
 * falls below that floor, whose list overflows, or with more than 4096 ties
 * at the cut gets fallback_d[n] = 1 and untouched positions/padded: the
 * caller runs glr_heat_map + glr_topk for it. ws: glr_heat_topk_workspace.  */
size_t glr_heat_topk_workspace(int C, int P, int n_max, int cap);
int glr_heat_topk(const uint8_t* stack_d, int H, int W, int C, int P, int expand,
                  const int32_t* anchors_d, int n_max, int K, int sep, int cap,
                  int32_t* positions_d, int32_t* padded_d, uint8_t* fallback_d, void* ws_d,
                  size_t ws_bytes, void* stream);

/* ---- (3) top-K selection: glr/matching.py:170-231 ---------------------------
 * Exact tie-ordered greedy selection per exemplar: slot 0 = anchor, then
 * (score desc, flat index asc) skipping Chebyshev <= sep of any chosen,
 * relaxed to sep = 0, then padded with the anchor.
 * positions_d: n*K*2 int32; padded_d: n int32. ws (optional, may be NULL):
 * glr_topk_workspace bytes let the histogram pass record the high-score
 * entries so each heat row is read once instead of twice.                  */
size_t glr_topk_workspace(int n_max, int K, int sep);
int glr_topk(const uint16_t* heat_d, int n_max, const int32_t* n_dev_d, int oh, int ow,
             int max_score, const int32_t* anchors_d, int K, int sep, int32_t* positions_d,
             int32_t* padded_d, void* ws_d, size_t ws_bytes, void* stream);

/* ---- (3) gather: glr/patches.py:43-54 ---------------------------------------
 * groups_d: (G, K, m) fp64, column j of group g = x[r:r+P, c:c+P, :].ravel()
 * (m = P*P*C).                                                              */
int glr_gather(const double* x_d, int H, int W, int C, int P, const int32_t* positions_d, int G,
               int K, double* groups_d, void* stream);

/* ---- (3b) block matching + pixel re-rank --------------------
 * glr_block_match: glr/matching.py:256-283 (`block_match`, the "nlr-*"
 * regularizers, solvers.py:154-164,199-200). For each of the n anchors the
 * window rows/cols [max(0, a - window), min(H - P, a + window)] at `stride`,
 * squared pixel distance to the anchor patch (numpy's pairwise order, bit
 * identical), the K-1 nearest by (distance, row, col) after the anchor
 * itself, anchor padding. positions_d (n, K, 2), padded_d (n).
 * glr_rerank_pixel: glr/matching.py:243-249 (`MatchConfig.rerank_pixel`):
 * in place, slot 0 kept, slots 1..K-1 ordered by (pixel L2 distance to the
 * slot-0 patch, (row, col)).                                                */
int glr_block_match(const double* x_d, int H, int W, int C, int P, const int32_t* anchors_d,
                    int n, int window, int stride, int K, int32_t* positions_d,
                    int32_t* padded_d, void* stream);
/* glr_xcorr_valid: matching.py:116-137 (`xcorr2_valid_batch`, any float
 * input): out_d (H-P+1, W-P+1, N) fp64 valid cross-correlation of x_d
 * (H,W,C) with N kernels k_d (N,P,P,C), channels summed, accumulated in
 * (dr, dc, ch) order with rounded products (bit-identical to the reference
 * tests' loop oracle; the reference's own backends agree with it exactly on
 * binary inputs).                                                          */
int glr_xcorr_valid(const double* x_d, int H, int W, int C, const double* k_d, int N, int P,
                    double* out_d, void* stream);
int glr_rerank_pixel(const double* x_d, int H, int W, int C, int P, int32_t* positions_d, int n,
                     int K, void* stream);

/* ---- (3c) TV baseline regularizer: glr/solvers.py:101-139 -------------------
 * glr_tv_denoise: anisotropic TV prox by `iters` dual projected-gradient
 * steps (tau = 1/8) on every channel, bit-identical to the reference's numpy
 * arithmetic; weight <= 0 copies x. out_d must not alias x_d; workspace
 * glr_tv_workspace(H, W, C) bytes (the dual pair, double-buffered).       */
size_t glr_tv_workspace(int H, int W, int C);
int glr_tv_denoise(const double* x_d, int H, int W, int C, double weight, int iters,
                   double* out_d, void* ws_d, size_t ws_bytes, void* stream);

/* ---- (4) WNNM: glr/lowrank.py:46-65 ------------------------------------------
 * Batched weighted singular-value shrinkage of G groups (K columns of m
 * rows each, column-major per group) via an fp64 Gram matrix, a cyclic
 * Jacobi eigensolver and out = M * V diag(f(s)/s) V^T. Any K >= 1 (like the
 * reference): K <= 64 runs the fast kernels (block Jacobi, eigenvector
 * cache, split-integer apply), wider groups a generic path (cold, no cache).
 * sigma: noise level (WnnmParams.noise_sigma); uniform_weight < 0 = unused.
 * nonfinite_d (optional): set to 1 when a group holds a non-finite value.   */
size_t glr_wnnm_workspace(int G, int K);
int glr_wnnm(const double* groups_d, int G, int m, int K, double sigma, double c_weight,
             double eps, double uniform_weight, double* out_d, int32_t* nonfinite_d, void* ws_d,
             size_t ws_bytes, void* stream);

/* ---- (4)+(5) fused regularizer: glr/lowrank.py:68-87 + patches.py:57-70 ----
 * For every group g < n: gather from x, WNNM, and scatter-add the denoised
 * patches into acc_d, an int64 fixed-point numerator (value * 2^frac_bits),
 * so aggregation is deterministic and rank-count invariant. The Gram is fp64
 * (DMMA); the product M * Wm runs on the int8 tensor cores as an exact
 * split-integer product (six base-256 digit slices per operand, levels
 * k + l <= 5), within ~2^-40 max|x| of the fp64 product per entry.
 * ws: glr_wnnm_workspace(n_max, K) bytes.
 * vcache_d (optional, n_max*64*64 doubles) keeps each group's eigenvectors;
 * warm != 0 starts the Jacobi sweeps from them (valid while the group's
 * positions are unchanged, i.e. between matching refreshes).              */
int glr_wnnm_scatter(const double* x_d, int H, int W, int C, int P, const int32_t* positions_d,
                     int n_max, const int32_t* n_dev_d, int K, double sigma, double c_weight,
                     double eps, int frac_bits, int64_t* acc_d, double* vcache_d, int warm,
                     const uint8_t* warm_flags_d, void* ws_d, size_t ws_bytes, void* stream);

/* glr_eig_work: measurement aid (no reference counterpart). The eigen step of
 * glr_wnnm_scatter / glr_wnnm (K <= 64) is iterative, so its work is data
 * dependent; the library counts, per device, [0] groups processed, [1] 4x4
 * block super-rounds run (one line of the Jacobi schedule = 1/21 of a sweep),
 * [2] groups finished by the first-order correction. Copies the three
 * counters to out3_host (host memory, may be NULL) after a device
 * synchronisation and clears them when reset != 0.                          */
int glr_eig_work(uint64_t* out3_host, int reset);

/* glr_vcache_remap: carry cached eigenvectors across a matching refresh —
 * new group g in [new_lo, new_hi) whose anchor was old group i in
 * [old_lo, old_hi) gets vc_new[g] = vc_old[i] and flags[g] = 1 (else 0), for
 * warm = 2 in glr_wnnm_scatter. With old_pos_d / new_pos_d ((n, K, 2) group
 * positions, both or neither) the eigenvector coordinates are re-indexed so
 * each kept patch position keeps its coordinate (an orthogonal row
 * permutation). map_d: H*W int32 scratch that must hold -1 everywhere on
 * entry (it is restored on exit).                                          */
int glr_vcache_remap(const int32_t* old_anchors_d, int old_lo, int old_hi,
                     const int32_t* new_anchors_d, int new_lo, int new_hi, int H, int W,
                     const double* vc_old_d, double* vc_new_d, uint8_t* flags_d, int32_t* map_d,
                     const int32_t* old_pos_d, const int32_t* new_pos_d, int K, void* stream);

/* glr_scatter_count: cnt[r][c] += 1 for every pixel covered by every patch
 * (channel-invariant form of scatter_group's counter, patches.py:70).      */
int glr_scatter_count(const int32_t* positions_d, int n_max, const int32_t* n_dev_d, int K,
                      int P, int H, int W, int32_t* cnt_d, void* stream);

/* glr_scatter_add_f64: exact-API scatter_group (patches.py:57-70) of fp64
 * groups into fp64 acc/cnt, deterministic (one thread per output pixel).  */
int glr_scatter_add_f64(const double* groups_d, const int32_t* positions_d, int G, int K, int P,
                        int H, int W, int C, double* acc_d, double* cnt_d, void* stream);

/* glr_scatter_fixed: fixed-point scatter-add of explicit fp64 groups (G,K,m)
 * into acc_d (the glr_regularize(x, groups, params) entry, lowrank.py:80-83). */
int glr_scatter_fixed(const double* groups_d, const int32_t* positions_d, int G, int K, int P,
                      int H, int W, int C, int frac_bits, int64_t* acc_d, void* stream);

/* glr_normalize: z = acc/cnt where cnt > 0 else x (lowrank.py:84-87).
 * The numerator is CONSUMED: covered entries are reset to 0 after the read
 * (read-and-clear), so the next scatter starts from zero without a memset.
 * The same holds for glr_gap_masksum / glr_gap_fourier.                    */
int glr_normalize(int64_t* acc_d, const int32_t* cnt_d, const double* x_d, int H, int W,
                  int C, int frac_bits, double* z_d, void* stream);

/* ---- (6) sensing operators + GAP update: glr/operators.py, solvers.py:298-301
 * Mask-sum family (CACTI operators.py:35-59, MSFA operators.py:160-185):
 *   A x = sum_t M_t x_t,  A^T y = M_t y,  gram = sum_t M_t^2.
 * glr_gap_masksum fuses normalize + z + A^T(safe_div(y - A z, gram)),
 * clip [lo, hi], and the per-block partial residual ||y - A x||^2; with
 * rho > 0 the divisor is rho + gram (the ADMM x-update, solvers.py:329).
 * acc_d/cnt_d may be NULL (then z = x_in). x_out may alias x_in.
 * resid_d: 1 double (deterministic reduction).                              */
int glr_masksum_forward(const double* x_d, const double* masks_d, int H, int W, int T,
                        double* y_d, void* stream);
int glr_masksum_adjoint(const double* y_d, const double* masks_d, int H, int W, int T,
                        double* x_d, void* stream);
size_t glr_gap_workspace(int H, int W);
int glr_gap_masksum(int64_t* acc_d, const int32_t* cnt_d, int frac_bits,
                    const double* x_in_d, const double* masks_d, const double* y_d,
                    const double* gram_d, int H, int W, int T, double lo, double hi,
                    double rho, double* x_out_d, double* resid_d, void* ws_d, void* stream);

/* Masked unitary 2-D DFT (operators.py:65-89): real (C=1, adjoint keeps the
 * real part) or complex (C=2, (re,im) channels) images. y is complex128
 * interleaved (H,W,2). glr_gap_fourier fuses normalize + projection + clip
 * + residual like glr_gap_masksum. ws: glr_fft_workspace.                  */
size_t glr_fft_workspace(int H, int W);
int glr_fourier_forward(const double* x_d, const double* mask_d, int H, int W, int C,
                        double* y_d, void* ws_d, void* stream);
int glr_fourier_adjoint(const double* y_d, const double* mask_d, int H, int W, int C,
                        double* x_d, void* ws_d, void* stream);
int glr_gap_fourier(int64_t* acc_d, const int32_t* cnt_d, int frac_bits,
                    const double* x_in_d, const double* mask_d, const double* y_d, int H, int W,
                    int C, int clip, double lo, double hi, double rho, double* x_out_d,
                    double* resid_d, void* ws_d, void* stream);

/* init="interp" (solvers.py:237-254). glr_interp_msfa: per channel
 * gaussian_filter(xt) / gaussian_filter(mask) (0 where the latter <= 1e-12),
 * bit-identical to scipy's symmetric correlate1d with mode "reflect";
 * weights: the 2*radius+1 host-computed taps (HOST pointer), ws: 4*H*W*C
 * doubles. glr_interp_cacti: xt / max(gram, 1e-12).                        */
int glr_interp_msfa(const double* xt_d, const double* masks_d, int H, int W, int C,
                    const double* weights, int radius, double* out_d, void* ws_d, void* stream);
int glr_interp_cacti(const double* xt_d, const double* gram_d, int H, int W, int C,
                     double* out_d, void* stream);

/* f3 -- on-device SSIM (metrics.py:40-78 + the clip of solvers.py:262-264):
 * *out_d = SUM over channels and valid window positions of the SSIM map
 * (divide by C*(H-S+1)*(W-S+1) for the reference's mean); window = the S
 * normalised 1-D Gaussian taps (HOST pointer), the 2-D window being their
 * outer product; clip != 0 clips x to [0, peak] first.
 * ws: glr_ssim_workspace(H, W, C) bytes.                                     */
size_t glr_ssim_workspace(int H, int W, int C);
int glr_ssim(const double* x_d, const double* ref_d, int H, int W, int C, double peak, int clip,
             const double* window, int win_size, double* out_d, void* ws_d, void* stream);

/* glr_lincomb: out = clip((a*x + b*y) + c*z) elementwise, y/z optional (NULL),
 * in that evaluation order (the ADMM bookkeeping of solvers.py:327-334). */
int glr_lincomb(const double* x_d, double a, const double* y_d, double b, const double* z_d,
                double c, int64_t n, int clip, double lo, double hi, double* out_d, void* stream);

/* Squared-error sum vs a reference for PSNR (metrics.py:26-37), of
 * clip(x, 0, peak) (no clip when peak <= 0), deterministic. out_d: 1 double. */
int glr_sq_err(const double* x_d, const double* ref_d, int n, double peak, double* out_d,
               void* ws_d, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* GLR_B200_H */
