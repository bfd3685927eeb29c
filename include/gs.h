/*
 * gs.h -- C ABI of the B200 (sm_100a) 3D Gaussian Splatting forward rasterizer,
 * the data-parallel hot path of Hi^2-GSLoc (arXiv 2507.15683).
 *
 * Citations: P:<n> = PAPER.md line n (section / equation / algorithm named),
 * S:<n> = SPEC.md line n, Q<n> = reading n in DESIGN.md §2.
 *
 * The hot path is four calls, each batched over poses and pyramid levels
 * ("views"):
 *
 *   gs_project     -> per (view, Gaussian): camera transform, cull, EWA 2D
 *                     covariance + conic + radius, tile rectangle, SH colour
 *                     (Alg. 1 l.9-12; "tile-based rasterization";
 *                     P:134 Theta_i).
 *   gs_bin_sort    -> duplicate records into (16x16 tile, depth) pairs, order
 *                     each tile's list by (depth_bits, gid), tile ranges
 *                     ("Tile size 16x16; front-to-back sort by
 *                     primitive depth per tile with stable index tiebreak").
 *   gs_rasterize   -> per pixel front-to-back alpha compositing of colour,
 *                     depth (sum w z), accumulated opacity A = 1 - T and an
 *                     optional D-channel feature ("alpha blending",
 *                     "identical rasterization"; "render dense feature and
 *                     depth maps").
 *   gs_backproject -> rendered depth -> world points for 2D-3D constraints
 *                     ("fully leverage the depth information from
 *                     Gaussian rendering for 3D constraints"; S:519 drop
 *                     accum_alpha < 0.5).
 *
 * Conventions common to every call
 * --------------------------------
 * - All data pointers are DEVICE pointers unless the name ends in _host.
 * - `stream` is a cudaStream_t passed as void* (NULL = legacy default stream).
 *   All work is enqueued asynchronously on it; no call synchronises the host.
 * - The caller allocates and frees every buffer (outputs and workspaces).
 *   The library never allocates device memory, never frees, and keeps no
 *   pointer after a call returns.  Calls are stateless and re-entrant:
 *   concurrent calls on different streams with distinct outputs/workspaces
 *   are safe.  Inputs and outputs must not alias.
 * - Return value: host-side validation result.  GS_OK means the work was
 *   enqueued.  Validation never reads device memory.  On error nothing is
 *   enqueued and gs_last_error() (thread-local) names the bad argument.
 * - Data-dependent conditions are NOT errors: degenerate / near / transparent /
 *   off-screen Gaussians are skipped and counted; capacity overflow
 *   sets bits in the device status word and the required sizes, and every
 *   later call of the batch that sees the bit writes nothing.  The caller
 *   reads the status once per batch and re-runs with larger buffers.
 * - Views of one batch own disjoint, contiguous slices of a flat pixel space
 *   (pix_offset) and a flat tile space (tile_offset); gs_views_layout() fills
 *   both.  Per view, images are planar: rgb [3][H][W] at 3*pix_offset,
 *   depth/alpha [H][W] at pix_offset, feat [D][H][W] at D*pix_offset.
 */
#ifndef GS_H_
#define GS_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define GS_ABI_VERSION 2
#define GS_TILE 16           /* tile edge in pixels */
#define GS_MAX_FEAT_DIM 64   /* D in [0, 64], D % 4 == 0 */
#define GS_MAX_VIEWS 65535   /* view index is stored in 16 bits of a record */

typedef enum gs_status {
    GS_OK = 0,
    GS_INVALID_ARG = 1,          /* NULL pointer, bad size, inconsistent layout */
    GS_UNSUPPORTED = 2,          /* sh_degree > 3, D % 4 != 0, D > 64, too many views */
    GS_WORKSPACE_TOO_SMALL = 3,  /* ws_bytes < the matching *_workspace_bytes() */
    GS_CUDA_ERROR = 4            /* a launch failed; gs_last_error() has cudaGetErrorString */
} gs_status;

/* Device status word bits (gs_projected.status). */
#define GS_STATUS_RECORD_OVERFLOW 0x1u  /* some view had > rec_capacity visible Gaussians */
#define GS_STATUS_PAIR_OVERFLOW 0x2u    /* the batch had > pair_capacity tile pairs */

/*
 * Pinhole camera + pose.  R, t map WORLD points to CAMERA points:
 * p = R x + t (Alg. 1 l.10 applies T_wc to world points; reading Q1).
 * Camera axes: x right, y down, z forward.  Pixel (px, py) is centred at the
 * integer coordinates (px, py) (Q4; S:44 maps (0,0,5) to pixel (50,50)).
 */
typedef struct gs_view {
    float R[9];            /* row-major world->camera rotation */
    float t[3];
    float fx, fy, cx, cy;  /* K (pixels) */
    int32_t width, height; /* image size (pixels), each in [1, 65535*16] */
    int64_t pix_offset;    /* first pixel of this view in the batch pixel space */
    uint32_t tile_offset;  /* first tile of this view in the batch tile space */
    uint32_t reserved;     /* must be 0 */
} gs_view;                 /* 88 bytes */

/*
 * Scene G: SoA planes of N Gaussians Theta_i = {mu, q, s, alpha, c, f}
 * (P:134).  q is (w,x,y,z), normalised inside (Q2).  scale and
 * opacity are linear, already-activated values (Q3).  Colour is real
 * SH of degree 0..3 ([3DGS] basis; flat RGB c is degree 0 with
 * k0 = (c - 0.5)/0.28209479177387814, Q23).  Features f are view-independent
 * and blended unnormalised (Q18).
 * Optional block partition (the cells of P:134, "divided into multiple
 * cells"): Gaussians stored block-major; block b owns [block_offsets[b],
 * block_offsets[b+1]); block_bounds[b] = {min x,y,z of centres, max x,y,z of
 * centres, max scale component, 0}.  gs_project uses them only for a
 * conservative per-(view, block) cull; results are identical with
 * n_blocks = 0.  gs_scene_block_bounds() computes block_bounds.
 */
typedef struct gs_scene {
    int64_t n;
    int32_t sh_degree;             /* 0..3 */
    int32_t feat_dim;              /* D: 0..64, multiple of 4 */
    const float* pos;              /* [3][n] */
    const float* quat;             /* [4][n] */
    const float* scale;            /* [3][n] */
    const float* opacity;          /* [n] */
    const float* sh;               /* [(deg+1)^2 * 3][n]; row k*3+c = coefficient k of channel c */
    const float* feat;             /* [n][D] row-major (NULL iff D == 0) */
    int32_t n_blocks;              /* 0 = no partition */
    int32_t reserved;
    const int64_t* block_offsets;  /* [n_blocks + 1] */
    const float* block_bounds;     /* [n_blocks][8] */
    const void* feat_h;            /* [n][D] IEEE binary16 copy of feat (round to nearest even), or
                                      NULL; filled by gs_scene_features_f16().  When present and
                                      D is 16, 32, 48 or 64, gs_rasterize gathers these rows and
                                      runs the feature contraction on tcgen05 (the features are
                                      rounded to fp16 either way) */
} gs_scene;                        /* 96 bytes */

/* Readings Q5, Q7, Q6, Q14, Q15; gs_default_params() returns these. */
typedef struct gs_params {
    float z_near;        /* 0.2   near cull, scene units (Q5) */
    float dilation;      /* 0.3   px^2 added to the 2D covariance diagonal (Q7) */
    float clamp_margin;  /* 0.15  off-screen Jacobian guard, fraction of W/H (Q6) */
    float alpha_min;     /* 1/255 skip threshold (Q14) */
    float alpha_max;     /* 0.99  opacity clamp (Q14) */
    float t_min;         /* 1e-4  stop before blending when T(1-alpha) < t_min (Q15) */
} gs_params;

/*
 * One projected (view, Gaussian) record, 64 bytes.  u, v, z, the exponent
 * coefficients, rect, radius are computed in IEEE fp32 in the operation order
 * of DESIGN.md §4.1 (bit-identical to the oracle); rgb is SH colour
 * (tolerance only).  The Gaussian exponent at offset d = mean - pixel is, in
 * log2 units (reading Q29), p(d) = dx (ea dx + eb dy) + ec dy dy =
 * log2(e) * (-1/2) d^T conic d, with ea = k conic_a, eb = 2k conic_b,
 * ec = k conic_c and k = fp32(-log2(e)/2) -- power-of-two multiples of one
 * rounded constant, so conic = (ea, eb/2, ec)/k.  e_cut (reading Q30) =
 * -((k' + (m - 0.9135)) 1.05 + 0.0075) for opacity / alpha_min = m 2^k',
 * m in [1, 2): an exactly reproducible bound with p(d) < e_cut implying
 * alpha < alpha_min with margin (used by the tight binning mode and the
 * rasterizer's cull to skip provably-zero work).
 */
typedef struct gs_record {
    float u, v;                       /* pixel-space mean */
    float ea, eb, ec;                 /* exponent coefficients, log2 units (see above) */
    float opacity;
    float e_cut;
    uint32_t tile_mask;               /* N3: bit (ty-y0)*nx + (tx-x0) set iff tile (tx, ty) of the
                                         rectangle is reached by the alpha >= alpha_min ellipse
                                         (reading Q30), rectangles of <= 31 tiles; bit 31 set =
                                         larger rectangle (decided per tile when binning) */
    float rgb[3];
    float z;                          /* camera-space depth (depth key = its bits, O9) */
    uint32_t gid;                     /* Gaussian index in the scene */
    uint32_t view_radius;             /* view (low 16 bits) | min(radius, 65535) << 16 */
    uint16_t x0, x1, y0, y1;          /* inclusive tile rectangle in the view's tile grid */
} gs_record;

typedef struct gs_projected {
    gs_record* rec;          /* [n_views * rec_capacity]; view v owns slots [v*cap, v*cap + n_rec[v]) */
    int64_t rec_capacity;    /* records per view */
    uint32_t* n_rec;         /* [n_views] visible count (may exceed cap: = required capacity) */
    uint64_t* diag;          /* [4] += near, transparent, degenerate, off-screen (Gaussians
                                skipped by the block cull are not visited and not counted) */
    uint32_t* status;        /* [1] GS_STATUS_* bits; caller zeroes before the batch */
    unsigned long long* contrib; /* optional [n_views * rec_capacity]: per record, the sum over all
                                    pixels of its blend weight w (N1, the forward visibility criterion
                                    of SPEC S:180), in units of 2^-32; zeroed and written by
                                    gs_rasterize when non-NULL (order-independent fixed point, so
                                    run-to-run deterministic) */
} gs_projected;

typedef struct gs_bins {
    uint32_t* ranges;        /* [total_tiles][2]: [start, end) into sorted_rec (lower bound, Q13) */
    uint32_t* sorted_rec;    /* [pair_capacity] record slot of each pair, ordered by
                                (tile in batch, depth_bits, gid) (Q12, Q22) */
    int64_t pair_capacity;
    uint64_t* n_pairs;       /* [1] pairs in the batch (= required capacity on overflow) */
    uint64_t* sorted_key;    /* optional [pair_capacity]: (tile in batch << 32) | depth_bits */
    uint32_t* sorted_gid;    /* optional [pair_capacity]: gid of each pair (lets gs_rasterize fetch
                                feature rows without a dependent record load) */
    uint32_t* tile_sched;    /* optional [1]: scratch counter of gs_rasterize's dynamic tile
                                scheduler (zeroed by gs_rasterize on its stream); NULL = static */
    int32_t mode;            /* GS_BIN_SQUARE: every tile of the 3-sigma rectangle (O8);
                                GS_BIN_TIGHT (N3, reading Q30): only the rectangle's tiles whose
                                pixel centres the alpha >= alpha_min ellipse p(d) >= e_cut can
                                reach (pinned fp32 test, bit-exact with the oracle's tight mode).
                                Both modes render bit-identical RGB, depth, opacity and
                                contributions; features agree up to fp32 summation grouping. */
    int32_t reserved;        /* must be 0 */
} gs_bins;
#define GS_BIN_SQUARE 0
#define GS_BIN_TIGHT 1

typedef struct gs_images {
    float* rgb;     /* [3 * total_pixels] */
    float* depth;   /* [total_pixels]  sum of w z (un-normalised, Q16) */
    float* alpha;   /* [total_pixels]  A = 1 - T_final */
    float* feat;    /* [D * total_pixels] or NULL when D == 0 */
} gs_images;

/* ---------------------------------------------------------------------- */

/* Library ABI version (GS_ABI_VERSION). */
int32_t gs_abi_version(void);

/* Thread-local description of the last non-OK status (never NULL). */
const char* gs_last_error(void);

/* Defaults of the readings Q5-Q7, Q14, Q15. */
gs_params gs_default_params(void);

/*
 * Fill pix_offset / tile_offset of views_host[0..n_views) contiguously in view
 * order and return the batch totals.  Host only; no device access.
 * Errors: GS_INVALID_ARG for NULL pointers, n_views < 1 or bad image sizes;
 * GS_UNSUPPORTED if n_views > GS_MAX_VIEWS or total tiles >= 2^31.
 */
gs_status gs_views_layout(gs_view* views_host, int32_t n_views, int64_t* total_pixels,
                          int64_t* total_tiles);

/*
 * block_bounds_out[b] = {min centre xyz, max centre xyz, max scale, 0} for
 * every block of `scene` (its block_bounds field is ignored).  Not on the
 * hot path: call once after loading a partitioned scene.
 */
gs_status gs_scene_block_bounds(const gs_scene* scene, float* block_bounds_out, void* stream);

/*
 * feat_h_out[i][c] = (binary16, round to nearest even) scene->feat[i][c] for
 * the n x D feature matrix of `scene` (its feat_h field is ignored); device
 * buffer of n * D * 2 bytes, 16-byte aligned, owned by the caller.  Not on the
 * hot path: call once after loading a scene with features, then set
 * scene->feat_h.  Errors: GS_INVALID_ARG if D == 0 or a pointer is NULL or
 * misaligned.
 */
gs_status gs_scene_features_f16(const gs_scene* scene, void* feat_h_out, void* stream);

/*
 * gs_validate_scene -- debug check of SPEC's Gaussian invariants over
 * the whole scene, reporting the first offending Gaussian ("naming the
 * offending record index").  Not on the hot path; the hot path never rejects
 * data (degenerate Gaussians are counted in diag).
 *   first_bad (device, 1 x int64): smallest index i violating an invariant,
 *     or -1 when the scene is valid; used as scratch during the call.
 *   reason (device, 1 x int32): the smallest GS_BAD_* code violated by
 *     Gaussian first_bad (GS_BAD_NONE when valid).
 *   unit_quat: 1 = also require | |q| - 1 | <= 1e-6; 0 = only
 *     a finite, non-zero q (gs_project normalises q, reading Q2).
 * Asynchronous on `stream`.  Errors: GS_INVALID_ARG for NULL pointers.
 */
#define GS_BAD_NONE 0
#define GS_BAD_POSITION 1   /* non-finite mean */
#define GS_BAD_QUAT 2       /* non-finite or zero quaternion */
#define GS_BAD_QUAT_NORM 3  /* | |q| - 1 | > 1e-6 (unit_quat = 1 only) */
#define GS_BAD_SCALE 4      /* scale not finite or <= 0 */
#define GS_BAD_OPACITY 5    /* opacity outside [0, 1] or NaN */
#define GS_BAD_SH 6         /* non-finite SH coefficient */
#define GS_BAD_FEATURE 7    /* non-finite feature */
gs_status gs_validate_scene(const gs_scene* scene, int32_t unit_quat, int64_t* first_bad, int32_t* reason,
                            void* stream);

/*
 * gs_sanitize_scene -- N4 training helper: after an optimizer step on the raw
 * parameter planes (Eq. 1-3 update Theta_i), project every Gaussian
 * back onto the set gs_project renders (readings Q3, Q19): opacity clamped to
 * [opacity_min, 1] (opacity_min >= alpha_min keeps it from being culled as
 * transparent and never receiving a gradient again), each scale to a finite
 * value >= scale_min (a scale <= 0 is degenerate, Q19), and a zero or
 * non-finite quaternion reset to identity.  Scene planes are modified in place
 * (device); changed (device, 1 x uint64) is incremented by the number of
 * Gaussians changed.  Errors: GS_INVALID_ARG for a bad scene, NULL changed,
 * opacity_min outside [0, 1] or scale_min <= 0.
 */
gs_status gs_sanitize_scene(const gs_scene* scene, float opacity_min, float scale_min, uint64_t* changed,
                            void* stream);

/*
 * N2 -- coarse-to-fine probabilistic mutual matching (Eq. 11 at
 * P:312-316; readings Q31-Q34).  For each of n_pairs (query,
 * rendered) feature-map pairs of equal size, planar [D][H][W] f32 (the layout
 * of gs_images.feat), H and W multiples of w = 8:
 *   coarse: w x w average pooling, cosine similarity M over the
 *   (H/8 W/8)^2 cell pairs, P = softmax_row(M/tau) (.) softmax_col(M/tau),
 *   mutual nearest neighbours with P > p_min (ties to the lowest index);
 *   fine: for every coarse match, the same between the 64 pixels of the two
 *   cells, then a 3 x 3 soft-argmax of P around the peak, clipped to the
 *   window; optionally the peak's back-projected point (gs_backproject
 *   output of the rendered view, [n_pairs][3][H][W] + [n_pairs][H][W]).
 * All outputs are dense and fully overwritten; pixel index = py * W + px.
 */
typedef struct gs_matches {
    int32_t* coarse;      /* [n_pairs][Nc], Nc = (H/8)(W/8): rendered cell matched to query cell, or -1 */
    float* coarse_prob;   /* [n_pairs][Nc]: P of the coarse match (0 if none) */
    int32_t* peak;        /* [n_pairs][H*W]: rendered pixel matched to each query pixel, or -1 */
    float* prob;          /* [n_pairs][H*W]: P of the fine match (0 if none) */
    float* ref;           /* [n_pairs][2][H*W]: sub-pixel rendered position (x, y) (0 if none) */
    float* xyz;           /* optional [n_pairs][3][H*W]: back-projected point at the peak (0 if none) */
    uint8_t* valid;       /* optional [n_pairs][H*W]: matched and the peak's depth is valid */
} gs_matches;

/* Workspace of gs_match (0 for invalid sizes). */
size_t gs_match_workspace_bytes(int32_t n_pairs, int32_t D, int32_t H, int32_t W);

/*
 * gs_match -- N2 as above on `stream`.  D in {16, 32, 48, 64}; tau > 0
 * (SPEC default 0.1), p_min (default 0.05).  rend_xyz / rend_valid may be
 * NULL (then out->xyz / out->valid are written as 0 when present).  ws: device,
 * 256-byte aligned, >= gs_match_workspace_bytes.  Errors: GS_INVALID_ARG
 * (NULL / misaligned pointers, sizes not multiples of 8, tau <= 0),
 * GS_UNSUPPORTED (D), GS_WORKSPACE_TOO_SMALL.
 */
gs_status gs_match(const float* query_feat, const float* rend_feat, int32_t n_pairs, int32_t D, int32_t H,
                   int32_t W, float tau, float p_min, const float* rend_xyz, const uint8_t* rend_valid, void* ws,
                   size_t ws_bytes, gs_matches* out, void* stream);

/*
 * N2 pose stage -- Eq. 10 on the dense correspondences of
 * gs_match: for problem b, correspondence = query pixel p = (px, py) with
 * valid[b][p] != 0 and world point xyz[b][:, p] (gs_matches.valid / .xyz;
 * in pixel order; with n > cap of them every k-th, k = ceil(n / cap), is used).  Reading Q35: RANSAC over n_hyp
 * minimal 3-point samples (counter-based hash of (seed, hypothesis, draw)),
 * each fitted exactly by 8 Gauss-Newton steps from the pose of views_in[b]
 * (the pose the rendered view was made at), scored by inlier count
 * (||p - pi(K[R|t]X)|| <= tau_px, z > 0); the best (or the start pose if none
 * has more inliers) refined by 10 damped Gauss-Newton steps on
 * rho(e) = min(e^2, tau^2).  fp64 arithmetic.
 * views_out[b] = views_in[b] with R, t replaced (ready for the next
 * gs_project of the refinement loop); stats[b] as below.  Device pointers,
 * asynchronous.  ws >= gs_pnp_workspace_bytes(n_problems, cap), 16-B aligned.
 */
typedef struct gs_pnp_stats {
    int32_t n_corr;          /* correspondences used (<= cap) */
    int32_t n_inliers;       /* |I*| under the returned pose */
    float mean_err;          /* mean reprojection error of the inliers, pixels */
    int32_t best_hypothesis; /* winning RANSAC sample, -1 = the start pose */
} gs_pnp_stats;

size_t gs_pnp_workspace_bytes(int32_t n_problems, int32_t cap);
gs_status gs_pnp(const uint8_t* valid, const float* xyz, int32_t n_problems, int32_t H, int32_t W,
                 const gs_view* views_in_dev, float tau_px, int32_t n_hyp, uint32_t seed, int32_t cap, void* ws,
                 size_t ws_bytes, gs_view* views_out_dev, gs_pnp_stats* stats_dev, void* stream);

/*
 * Algorithm 2 over a refinement trace trace_dev[i][b]
 * (n_iters poses per problem): angle_deg[b][i] = arccos((clamp(tr(R_i R_{i+1}^T),
 * -1, 3) - 1)/2) in degrees, dtrans[b][i] = |t_i - t_{i+1}| (computed, not
 * gated -- as in the algorithm); verdict[b] = -1 reliable (return T_n), i = the
 * first consecutive pair over tau_deg (unreliable), -2 when n_iters < 2.
 */
gs_status gs_verify_consistency(const gs_view* trace_dev, int32_t n_iters, int32_t n_problems, float tau_deg,
                                float* angle_deg, float* dtrans, int32_t* verdict, void* stream);

/*
 * N4 -- feature-field backward of Eq. 2 with the geometry frozen
 * (DESIGN.md §4.8): for the batch rendered by gs_project / gs_bin_sort (same
 * proj, bins, views), grad_feat[g][c] += sum over the batch's pixels of
 * w_g(px) * grad_image[c][px], where w are the forward blend weights and
 * grad_image is dL/dF in the layout of gs_images.feat ([D][H][W] per view at
 * D * pix_offset).  grad_feat [n][D] f32 is accumulated (caller zeroes).  The
 * per-pixel walk is the forward's (same cull, exponent, stop rule).
 * D must be a multiple of 8 (8..64).  Asynchronous; device pointers.
 */
gs_status gs_feature_backward(const gs_scene* scene, const gs_projected* proj, const gs_bins* bins,
                              const gs_view* views_host, const gs_view* views_dev, int32_t n_views,
                              const gs_params* params, const float* grad_image, float* grad_feat, void* stream);

/*
 * N4 radiance backward: for the batch rendered with proj /
 * bins / views (fwd = its gs_images), the gradient of
 * L = sum_px gC . C + gD Dz + gA A  (grad_out = dL/d{rgb, depth, alpha} in the
 * gs_images layout; its feat is ignored) w.r.t. each record's
 * {u, v, ea, eb, ec, opacity, r, g, b, z}: grad_rec [n_views * rec_capacity][10]
 * f32, accumulated (caller zeroes), indexed by record slot like proj->contrib.
 * The skip / stop decisions are the forward's (zero gradient through them);
 * an alpha clamped at alpha_max has no opacity / exponent gradient.
 */
gs_status gs_radiance_backward(const gs_projected* proj, const gs_bins* bins, const gs_view* views_host,
                               const gs_view* views_dev, int32_t n_views, const gs_params* params,
                               const gs_images* fwd, const gs_images* grad_out, float* grad_rec, void* stream);

/*
 * gs_appearance_l1_grad -- N4, Eq. 3's L1 term between the ground truth I and the
 * appearance-varied rendering I^a (reading Q38: per view and channel an
 * affine transform I^a = a I^r + b of the direct rendering, trained jointly).
 * n_planes planes of plane_pixels pixels each (a run of equal-size views: plane
 * 3 v + c), plane p uses a[p], b[p].  Writes grad_image = scale sign(I^a - I) a
 * (dL/dI^r), accumulates grad_a[p] += scale sum sign(I^a - I) I^r,
 * grad_b[p] += scale sum sign(I^a - I) and loss += scale sum |I^a - I| (fp64).
 * All device pointers.  Errors: GS_INVALID_ARG for NULL pointers or sizes out of
 * range (n_planes > 65535).
 */
gs_status gs_appearance_l1_grad(const float* rendered, const float* target, int32_t n_planes, int64_t plane_pixels,
                                const float* a, const float* b, float scale, float* grad_image, float* grad_a,
                                float* grad_b, double* loss, void* stream);

/*
 * gs_joint_backward -- N4, Eq. 1's joint loss: gs_radiance_backward
 * plus Eq. 2's feature term through the blend weights.  grad_out->feat
 * ([D][H][W] per view, the gs_images layout) is dL/dF of the rendered feature
 * map; F = sum_k w_k f_k enters like a colour channel, so each record's
 * {u, v, ea, eb, ec, opacity} gradient also receives
 * sum_px dL/dalpha_k with dF/dalpha_k = T_k f_k - (F - F_<=k)/(1 - alpha_k)
 * (scene->feat: the fp32 feature rows; fwd->feat: the forward's feature map).
 * The gradient w.r.t. the features themselves is gs_feature_backward's.
 * grad_out->feat == NULL or D == 0: exactly gs_radiance_backward.
 * Errors: as gs_radiance_backward; GS_UNSUPPORTED for D not in
 * {8, 16, 24, 32, 48, 64}.
 */
gs_status gs_joint_backward(const gs_scene* scene, const gs_projected* proj, const gs_bins* bins,
                            const gs_view* views_host, const gs_view* views_dev, int32_t n_views,
                            const gs_params* params, const gs_images* fwd, const gs_images* grad_out,
                            float* grad_rec, void* stream);

/*
 * N4 projection backward: chains grad_rec (from gs_radiance_backward, same
 * proj) through O1-O7 -- pinhole u, v and depth z, the clamped EWA Jacobian
 * (Q6), the 2D covariance, its inverse and e = k conic (Q29) -- to the
 * Gaussians' 3D means: grad_pos [3][n] (the layout of gs_scene.pos) +=
 * dL/dmu, fp64 arithmetic, f32 atomics.  Alg. 1's literal render-gradient
 * visibility test is ||dL/dmu|| > 0 for a loss on the render.
 * Includes the path through O10's SH view direction d = (mu - c)/|mu - c|
 * (colour of degree >= 1; zero for a channel clamped at 0).
 */
gs_status gs_mean_backward(const gs_scene* scene, const gs_projected* proj, const gs_view* views_host,
                           const gs_view* views_dev, int32_t n_views, const gs_params* params,
                           const float* grad_rec, float* grad_pos, void* stream);

/*
 * N4 projection backward, the other parameters of Theta_i: chains
 * grad_rec through O4-O7 and O10 to the Gaussians' scale, rotation, opacity
 * and SH coefficients.  With G = dL/dSigma' (Sigma' = [[a, b], [b, c]]),
 * dL/dSigma = T^T G T (T = J R), Sigma = M M^T -> dL/dM = 2 dL/dSigma M,
 * M = R(q) diag(s) -> dL/ds and dL/dR(q); the normalised quaternion's R(q) is
 * differentiated and projected, dL/dq = (I - q^ q^T)/|q| dL/dq^;
 * dL/df_kc = b_k(d) dL/drgb_c [rgb_c > 0]; dL/do from grad_rec directly.
 * Outputs in the layouts of gs_scene: grad_scale [3][n], grad_quat [4][n],
 * grad_opacity [n], grad_sh [(deg+1)^2 * 3][n]; each optional (NULL = skip);
 * accumulated over records and views (caller zeroes), fp64 arithmetic, f32
 * atomics.  Errors as gs_mean_backward.
 */
gs_status gs_param_backward(const gs_scene* scene, const gs_projected* proj, const gs_view* views_host,
                            const gs_view* views_dev, int32_t n_views, const gs_params* params,
                            const float* grad_rec, float* grad_scale, float* grad_quat, float* grad_opacity,
                            float* grad_sh, void* stream);

/* Eq. 2's L1 feature loss: grad_image[i] = scale * sign(rendered[i] - target[i]);
 * *loss (device double, accumulated) += scale * sum |rendered - target|. */
gs_status gs_feature_l1_grad(const float* rendered, const float* target, int64_t n, float scale,
                             float* grad_image, double* loss, void* stream);

/* Eq. 3's D-SSIM term (reading Q37: 1 - SSIM with an
 * 11 x 11 Gaussian window, sigma 1.5, zero padding, C1 = 0.01^2, C2 = 0.03^2)
 * over n_planes contiguous fp32 planes of height x width (row-major; e.g. the
 * [3][H][W] RGB planes of one view of gs_images, or several equal-size views).
 * *loss (device double, accumulated) += scale * sum over planes and pixels of
 * (1 - S); grad_image (same layout, ACCUMULATED: the caller zeroes it or lets it
 * hold the L1 gradient of gs_feature_l1_grad) += scale * d sum(1 - S) / d rendered.
 * With scale = lambda / (C H W) this is lambda * L_D-SSIM and its gradient.
 * workspace: device, >= gs_dssim_workspace_bytes(...) bytes, caller-owned
 * scratch (three fp32 partial-derivative planes per input plane).
 * Errors: GS_INVALID_ARG for negative sizes, n_planes > 65535 or NULL pointers
 * (when the size is non-zero); GS_WORKSPACE_TOO_SMALL; empty input is a no-op. */
size_t gs_dssim_workspace_bytes(int32_t n_planes, int32_t height, int32_t width);
gs_status gs_dssim_grad(const float* rendered, const float* target, int32_t n_planes, int32_t height, int32_t width,
                        float scale, float* grad_image, float* workspace, size_t workspace_bytes, double* loss,
                        void* stream);

/* feat[i] -= lr * grad_feat[i] over n floats; refreshes the fp16 copy (gs_scene.feat_h) when feat_h != NULL. */
gs_status gs_feature_sgd(float* feat, const float* grad_feat, int64_t n, float lr, void* feat_h, void* stream);

/* One Adam step over n floats (the optimiser of 3DGS-style training, N4):
 * m = b1 m + (1 - b1) g; v = b2 v + (1 - b2) g^2;
 * param -= lr (m / (1 - b1^step)) / (sqrt(v / (1 - b2^step)) + eps), step >= 1.
 * m, v: caller-owned state (zero-initialised), fp32; param_h as in gs_feature_sgd.
 * Errors: GS_INVALID_ARG for NULL pointers, n < 0 or step < 1. */
gs_status gs_adam(float* param, const float* grad, float* m, float* v, int64_t n, float lr, float beta1,
                  float beta2, float eps, int32_t step, void* param_h, void* stream);

/* Workspace of gs_project: a (view x block) visibility bitmask. */
size_t gs_project_workspace_bytes(int32_t n_blocks, int32_t n_views);

/*
 * gs_project -- O1-O10 for every (view, Gaussian) of the batch.
 * views_host and views_dev hold identical contents (host copy for
 * validation/launch sizing, device copy for the kernels).  Writes the
 * visible records of view v to out->rec[v*cap ...] in an unspecified order
 * (the sort makes the result canonical), n_rec[v], diag; sets
 * GS_STATUS_RECORD_OVERFLOW if a view has more than rec_capacity.
 * out->n_rec and out->diag are overwritten (zeroed by this call).
 */
gs_status gs_project(const gs_scene* scene, const gs_view* views_host, const gs_view* views_dev,
                     int32_t n_views, const gs_params* params, gs_projected* out, void* ws,
                     size_t ws_bytes, void* stream);

/* Workspace of gs_bin_sort for a batch of total_tiles tiles and pair_capacity pairs. */
size_t gs_bin_sort_workspace_bytes(int64_t pair_capacity, int64_t total_tiles);

/*
 * gs_bin_sort -- O11: one pair per tile of each record's rectangle, each
 * tile's pairs ordered by (depth_bits, gid) ascending (Q12), lower-bound
 * ranges (Q13).  The pair list and ranges are bit-identical to the oracle's
 * and run-to-run deterministic.  Sets GS_STATUS_PAIR_OVERFLOW (and n_pairs)
 * if the batch needs more than pair_capacity pairs.
 */
gs_status gs_bin_sort(const gs_projected* proj, const gs_view* views_host, const gs_view* views_dev,
                      int32_t n_views, gs_bins* out, void* ws, size_t ws_bytes, void* stream);

/*
 * gs_rasterize -- O12: for every pixel of every view, front to back over its
 * tile's list: power = -0.5(ca dx^2 + cc dy^2) - cb dx dy, skip if > 0;
 * alpha = min(alpha_max, o exp(power)), skip if < alpha_min;
 * Tn = T(1 - alpha), stop before blending if Tn < t_min;
 * C += w rgb, Dz += w z, F += w f with w = alpha T; T = Tn.  A = 1 - T.
 * Every output pixel is written (background 0).  `scene` supplies feat / D.
 */
gs_status gs_rasterize(const gs_scene* scene, const gs_projected* proj, const gs_bins* bins,
                       const gs_view* views_host, const gs_view* views_dev, int32_t n_views,
                       const gs_params* params, gs_images* out, void* stream);

/*
 * gs_rasterize_backproject -- gs_rasterize with O13 (gs_backproject below) fused
 * into its per-pixel epilogue: the same outputs as gs_rasterize followed by
 * gs_backproject(out, ..., a_min, xyz, valid), without re-reading depth and
 * alpha.  P:278 (rendered depth for the 2D-3D constraints).  xyz [3][H][W] and
 * valid [H][W] per view as gs_backproject (no alignment requirement).
 * Errors: those of gs_rasterize; GS_INVALID_ARG for NULL xyz / valid or NaN a_min.
 */
gs_status gs_rasterize_backproject(const gs_scene* scene, const gs_projected* proj, const gs_bins* bins,
                                   const gs_view* views_host, const gs_view* views_dev, int32_t n_views,
                                   const gs_params* params, gs_images* out, float a_min, float* xyz,
                                   uint8_t* valid, void* stream);

/*
 * gs_pack_images -- the compact transport of SURVEY.md §8(e) (reading Q39): RGB + A as
 * fp16 and the depth plane sum(w z) as fp32, 12 B per pixel instead of 20, for moving
 * rendered batches off the GPU (device -> host, or a gather).  Per view v the packed
 * block starts at byte 12 * pix_offset(v): planes R, G, B, A (fp16, hw each) then
 * Sigma w z (fp32, hw).  fp16 rounding changes a colour / opacity value c <= 2 by
 * <= 2^-11 |c| <= 9.8e-4, inside the 1e-3 image tolerance; depth is exact.
 * format: GS_PACK_COMPACT or GS_PACK_DENSE11 (below).  out: device,
 * gs_pack_bytes(total_pixels, format) bytes,
 * 16-byte aligned.  Errors: GS_UNSUPPORTED for another format, GS_INVALID_ARG for
 * NULL / misaligned pointers or a bad view batch.
 */
#define GS_PACK_COMPACT 1
/*
 * GS_PACK_DENSE11 (r2, Q39): 11 B per pixel, batch-planar (TP = total_pixels):
 * bytes [0, 6 TP) the R, G, B planes (fp16, plane c at 2 c TP, pixel pix_offset(v) + i of
 * view v at index pix_offset(v) + i), [6 TP, 8 TP) A as unorm16 round(65535 A)
 * (error <= 7.7e-6), [8 TP, 11 TP) sum(w z) as the upper 24 bits of its fp32 pattern
 * (round half up on the dropped byte; decode: bits << 8; relative error <= 2^-16,
 * inside the 1e-4 depth tolerance), 3 bytes little-endian per pixel.  Requires 16-byte
 * aligned input planes.
 */
#define GS_PACK_DENSE11 2
size_t gs_pack_bytes(int64_t total_pixels, int32_t format);
gs_status gs_pack_images(const gs_images* in, const gs_view* views_host, const gs_view* views_dev, int32_t n_views,
                         int32_t format, void* out, void* stream);

/*
 * gs_probe_alpha -- debug: alpha_out[i] = o_i 2^{p_i} evaluated exactly as
 * gs_rasterize's walk evaluates it (the unclamped alpha of O12 step 4, P:136
 * "alpha blending" with alpha = o exp(power) in log2 units, reading Q29), for
 * checking the kernel's deviation from the oracle's fp64 2^p against the O14
 * alpha band (reading Q20).  opacity, power, alpha_out: device
 * float arrays of n elements (caller-owned; alpha_out must not alias).
 * Errors: GS_INVALID_ARG for n < 0 or NULL pointers with n > 0.
 */
gs_status gs_probe_alpha(const float* opacity, const float* power, int64_t n, float* alpha_out, void* stream);

/*
 * gs_backproject -- O13: valid iff A >= a_min and Dz/A > 0;
 * X = R^T(((px - cx)/fx zbar, (py - cy)/fy zbar, zbar) - t), zbar = Dz/A.
 * xyz is planar [3][H][W] per view at 3*pix_offset; invalid pixels get
 * X = 0 and valid = 0.
 */
gs_status gs_backproject(const gs_images* in, const gs_view* views_host, const gs_view* views_dev,
                         int32_t n_views, float a_min, float* xyz, uint8_t* valid, void* stream);

/*
 * gs_visibility_score -- N1: Alg. 1 render-visibility check with
 * projection filtering and significance scoring (Eq. 4-6,
 * P:174-185) for every record of the batch.  Needs out->contrib from
 * gs_rasterize.
 *   M^r = contrib > eps (the forward criterion; eps default 1e-6),
 *   M^i = 0 <= u < W and 0 <= v < H (Alg. 1 l.17), visible = M^i and M^r;
 *   visible[slot] = 1/0 for each record slot (the (U', V') of Alg. 1 are the
 *   records' u, v where visible), n_visible[v] = count per view;
 *   count[gid] += 1 per view in which gid is visible (Eq. 6's M);
 *   if fmaps != NULL: score_sum[gid] += cos(f_gid, F^t_v(cell)) (Eq. 4-5) as
 *   signed 2^-32 fixed point (two's complement in a u64), with F^t_v the view's
 *   target feature map [D][ceil(H/stride)][ceil(W/stride)] (maps of all views
 *   concatenated in view order) sampled at the nearest cell
 *   (floor((u + 0.5)/stride), floor((v + 0.5)/stride)) (reading Q27); the
 *   cosine of a zero vector is 0 (Q28).  S(g) = score_sum / count (Eq. 6) is
 *   formed by the caller.  n_visible is overwritten; count and score_sum
 *   accumulate (the caller zeroes them once for a multi-batch pass).
 *   ws (optional, >= gs_visibility_workspace_bytes()) receives a channels-last
 *   copy of the maps so each sample reads one contiguous feature row; with
 *   ws == NULL the planar maps are sampled channel by channel (slower).
 */
size_t gs_visibility_workspace_bytes(const gs_view* views_host, int32_t n_views, int32_t feat_dim, int32_t stride);

gs_status gs_visibility_score(const gs_projected* proj, const gs_view* views_host, const gs_view* views_dev,
                              int32_t n_views, float eps, const float* feat /* scene [N][D] */, int32_t feat_dim,
                              const float* fmaps, int32_t stride, void* ws, size_t ws_bytes, uint8_t* visible,
                              uint32_t* n_visible, unsigned long long* score_sum, uint32_t* count, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* GS_H_ */
