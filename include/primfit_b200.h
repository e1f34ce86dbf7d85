/*
 * primfit_b200.h — C ABI of the B200 (sm_100a) differentiable bitmap compositor.
 *
 * This is the drop-in boundary for the hot path of the reference package
 * `primfit` (arxiv 2602.22625, DiffBMP): one optimisation step of
 * fit.run_loop (pkg/src/primfit/fit.py:448-505) =
 *     bin_tiles -> render_forward(save=True) -> loss_mse -> backward -> adam_step -> psnr
 *
 * The reference has no FFI; its native layer is four numba kernels with flat
 * positional array arguments (pkg/src/primfit/_kernels.py:76-363) driven by the
 * L2 Python API (raster.py, grad.py, fit.py).  Each entry point below names the
 * reference unit it replaces.  Conventions, identical for every entry point:
 *
 *   - every pointer argument is a DEVICE pointer unless the comment says "host";
 *   - every output buffer is caller-allocated (reference ownership model,
 *     raster.py:327-342 allocates before calling the kernels);
 *   - every call is stream-ordered on `stream` (a cudaStream_t, passed as void*
 *     so the header has no CUDA dependency) and never synchronises;
 *   - the return value is 0 (PF_OK) or a nonzero code: a cudaError_t value from
 *     the launch, or one of the PF_ERR_* codes below.  No exceptions cross the ABI.
 *
 * Parameter layout (scene.py:36, PARAM_GROUPS): params is float64 [n][8] with
 * columns x, y, scale, rotation, opacity_logit, c0, c1, c2 (primitive-major,
 * exactly the reference's packed vector from pack_params, scene.py:183-191).
 *
 * Template atlas (raster.py:63-96, PackedScene.tex/toff/tw/th): float64,
 * PLANAR [4][texels] (R plane, G plane, B plane, A plane); template t occupies
 * texels [tpl_base[t], tpl_base[t] + tpl_w[t]*tpl_h[t]) of every plane,
 * row-major (texel index base + v*w + u, _kernels.py:40).
 *
 * Canvas tiles are row-major (t = ty*ntx + tx, _kernels.py:88-89).  A "row band"
 * [ty_begin, ty_end) restricts binning/rendering to those tile rows (multi-GPU
 * row-band sharding); band-local tile index tb = (ty - ty_begin)*ntx + tx.
 * The full canvas is ty_begin = 0, ty_end = ceil(H / tile).
 */
#ifndef PRIMFIT_B200_H
#define PRIMFIT_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PF_OK 0
#define PF_ERR_ARG 1001      /* bad argument (null pointer, negative size, ...) */
#define PF_ERR_SCRATCH 1002  /* scratch buffer smaller than pf_bin_scratch_bytes */
#define PF_ERR_TILE 1003     /* render kernels support tile == 16 only */

/* Loss kinds fused into pf_forward (fit.py:112-171 evaluate_loss). */
#define PF_LOSS_NONE 0
#define PF_LOSS_MSE 1        /* loss_mse, fit.py:112-116 */
#define PF_LOSS_SPATIAL 2    /* loss_spatial, fit.py:128-151 */
#define PF_LOSS_COMBINED 3   /* mse_w * loss_mse + gray_l1_w * loss_grayscale_l1, fit.py:119-125, 162-168 */
#define PF_LOSS_EXTERN 4     /* pf_fit_step only: dL/dI, dL/dA given per pixel in tgt4 (a torch loss
                                upstream: the autograd Function's backward), no loss sums */
#define PF_LOSS_RENDER 5     /* pf_fit_step only (ABI 7, CSR lists): render only -- img4 written, no
                                loss, no gradients; tgt4 / part / grads may be NULL (the autograd
                                Function's forward) */

/* ABI version; bumped on any signature change. */
int pf_abi_version(void);  /* 8 */

/* Diagnostics: the PF_* environment switches (A/B variants, profiling) are read
 * once at load; this re-reads them (tests that flip a switch at run time). */
int pf_diag_reload(void);

/* Bytes of the per-primitive device record written by pf_preprocess
 * (replaces PackedScene, raster.py:45-96, as the kernels' view of a scene). */
size_t pf_record_bytes(void);

/* Render tile edge the forward/backward kernels are built for (16). */
int pf_render_tile(void);

/* Scratch bytes pf_preprocess + pf_bin need for n primitives, n_tiles band
 * tiles and `capacity` (tile, primitive) bin entries. Host-only query. */
size_t pf_bin_scratch_bytes(int n, int n_tiles, int capacity);

/* Saved-forward entry capacity for `capacity` bin entries (256 per entry). */
long long pf_saved_capacity(int capacity);

/* Bytes of the saved-forward buffer for `capacity` bin entries:
 * pf_saved_capacity(capacity) entries x 16 bytes (list position, texel cell,
 * fp32 bilinear weights, fp32 incoming transmittance). */
size_t pf_saved_bytes(int capacity);

/*
 * Alpha "quad atlas": for every texel (u, v) of the planar atlas `tex`, the four
 * bilinear taps of the alpha plane (a[v][u], a[v][u+1], a[v+1][u], a[v+1][u+1])
 * with the reference's zero padding (_kernels.py:35-40) applied.  quad out:
 * float32 [texels][4] (16-byte aligned).  Build once per atlas; pass it to
 * pf_forward / pf_backward (which re-take the m < eps_skip decision on the
 * float64 plane whenever the fp32 taps leave it within rounding).
 */
int pf_atlas_quad(const double* tex, int texels, const int32_t* tpl_base, const int32_t* tpl_w,
                  const int32_t* tpl_h, int n_tpl, float* quad, void* stream);

/*
 * One-time setup of a binning scratch buffer for a scene structure: zero it,
 * copy the static z order, and build the static per-primitive structure
 * (template geometry, z rank) that K1 reads with one load per primitive.
 *   template_id [n]   PrimitiveParams.template_id (scene.py:70-87)
 *   zorder      [n]   primitive indices in ascending z (PackedScene.order, raster.py:92)
 *   tpl_base / tpl_pbase / tpl_w / tpl_h [n_tpl]  atlas base, padded-atlas base
 *                     (pf_atlas_pad; may be NULL), template width / height
 *   tpl_q   [n_tpl]   aspect q used for primitives of that template (th/tw when
 *                     preserve_aspect, else 1.0; raster.py:88-91)
 *   tpl_hyp [n_tpl]   hypot(1, max(1, q)) (host-computed, bit-identical to
 *                     math.hypot in bbox_half_side, raster.py:222-224)
 */
int pf_scratch_init(void* scratch, size_t scratch_bytes, const int32_t* template_id,
                    const int32_t* zorder, int n, const int32_t* tpl_base,
                    const int32_t* tpl_pbase, const int32_t* tpl_w, const int32_t* tpl_h,
                    const double* tpl_q, const double* tpl_hyp, int n_tpl, int capacity,
                    void* stream);

/*
 * K1 — per-primitive preprocess + bin rects.
 * Replaces: the per-pair inline transform/sigmoid math of every numba kernel
 * (_kernels.py:106-123), pack_scene (raster.py:63-96) and the bbox part of
 * bin_tiles (raster.py:246-257, bbox_half_side raster.py:222-224).
 *   params   float64 [n][8]
 *   padding  bbox padding (fit.effective_padding, fit.py:338-341)
 *   rec      out   n * pf_record_bytes() bytes
 *   scratch  pf_bin_scratch_bytes(n, n_band_tiles, capacity) bytes, set up by
 *            pf_scratch_init; receives the band-clipped tile rect of every
 *            primitive at its z rank
 */
int pf_preprocess(const double* params, int n, double alpha_max, double mu_blend, double padding,
                  int W, int H, int tile, int ty_begin, int ty_end, int capacity,
                  void* rec, void* scratch, size_t scratch_bytes, void* slots, int slot_m,
                  int32_t* tile_classes, void* stream);

/*
 * Slot binning (the fit step's tile lists without pf_bin).  With `slots` set
 * (pf_slot_bytes(n_band_tiles, slot_m, capacity) bytes; NULL = CSR mode), every
 * K1 launch (pf_preprocess, pf_preprocess_sync, pf_adam_preprocess with rec)
 * also appends each of its primitives' (tile, z rank) pairs to the tile's slot
 * list (arrival order; past slot_m slots to an overflow list sized from
 * `capacity`), writes the K34-only records at the z rank, and (except
 * pf_preprocess_sync) rebuilds the tile cost classes from the costs the last
 * pf_fit_step measured.  pf_fit_step then sorts each tile's list by z rank
 * (= bin_tiles' z-ascending list, raster.py:227-265) before staging it, and
 * empties the slots for the next K1.  pf_slot_reset empties them (and the class
 * counts) before a full pf_preprocess; pf_preprocess_sync re-scatters only
 * edited primitives and flags the step, whose lists are then validated against
 * the current rects and de-duplicated.  The render tile (16) is required.
 */
size_t pf_slot_bytes(int n_tiles, int slot_m, int capacity);
int pf_slot_reset(void* slots, int n_tiles, int slot_m, int capacity, int32_t* tile_classes,
                  void* stream);

/*
 * K1, incremental: the parameters are taken from `src` (e.g. the caller's
 * pinned host vector, read in place over the host link); only primitives whose
 * 8 values differ bitwise from `params` (the device copy) are copied into
 * `params` and get new records / rects -- the others' are current from the
 * pf_adam_preprocess launch that wrote `params` (and mirrored them to `src`).
 * The per-step H2D of a host-driven fit loop.
 */
int pf_preprocess_sync(double* params, const double* src, int n, double alpha_max,
                       double mu_blend, double padding, int W, int H, int tile, int ty_begin,
                       int ty_end, int capacity, void* rec, void* scratch, size_t scratch_bytes,
                       void* slots, int slot_m, int32_t* tile_classes, void* stream);

/*
 * K5+K1 fused: one Adam step (fit.py:195-238) on every parameter, then the
 * records / tile rects of the NEXT step from the updated parameters (as
 * pf_preprocess) -- one launch between two renders.  Gradients are zeroed.
 * The learning rate and bias corrections come from host tables indexed by the
 * iteration counter kept in `scratch` (zeroed by pf_scratch_init; the Adam
 * launch marks the iteration done and the next pf_bin advances the counter).
 *   sums       this step's loss sums (after a cross-rank allreduce), or NULL
 *   part       pf_fit_step's n_part per-warp loss partials, or NULL
 *   hist_part  [iterations][pf_adam_blocks(n)][3] float64: this step's loss sums
 *              per launch block (fixed-order fold of `part`, or `sums` in block
 *              0 and zeros elsewhere); summing the blocks in order gives the
 *              HistoryEntry loss of the iteration (fit.py:502-505), or NULL
 *   last_part  [pf_adam_blocks(n)][3]: the same sums of the latest step only (a
 *              fixed address a per-step host read can use), or NULL
 *   rec        the records of the next step, or NULL for Adam only (no records,
 *              no rects: the caller runs pf_preprocess before the next pf_bin)
 *   mirror     the updated parameters are also written here (e.g. the caller's
 *              pinned host vector: the per-step D2H of a host-driven loop), or NULL
 */
int pf_adam_blocks(int n);
int pf_adam_preprocess(double* params, double* grads, double* m, double* v, const uint8_t* frozen,
                       const double* gains8, const double* lr_table, const double* bc1_table,
                       const double* bc2_table, int clamp, double s_min, double s_max,
                       const double* sums, const double* part, int n_part, double* hist_part,
                       double* last_part, int n, double alpha_max, double mu_blend, double padding, int W, int H,
                       int tile, int ty_begin, int ty_end, int capacity, void* rec, void* scratch,
                       size_t scratch_bytes, double* mirror, void* slots, int slot_m,
                       int32_t* tile_classes, void* stream);

/*
 * K2 — tile binning from the rects of pf_preprocess: one block per tile row,
 * a two-digit (row, column) stable radix bucketing of the z-ordered primitive
 * stream (block-wide stable compactions and ballots; no sort scratch, no
 * atomics, no host sync).  Output is bit-identical to bin_tiles
 * (raster.py:227-265): primitive indices ascending in z inside each tile.
 *   bin_off  out [n_band_tiles + 1]   (TileBins.offsets)
 *   bin_idx  out [capacity]           (TileBins.indices; first K valid)
 *   status   out int32[4]: [0] = K (total entries), [1] = overflow flag (K > capacity;
 *            nothing else is written then)
 *   tile_classes  optional int32 [16 + 65 * n_band_tiles] (NULL to skip): the
 *            band tiles grouped by cost class for pf_fit_step's longest-first
 *            schedule -- [0..16) counts (accumulated: zero before the first
 *            pf_bin; pf_fit_step re-zeroes them), one list of int4 tile entries
 *            (tile, list offset, list length, tx | ty << 16) per class, then the
 *            per-tile costs pf_fit_step measured (consumed and cleared here; the
 *            list length stands in until a first fit step).
 *            Order inside a class is not deterministic; it only steers scheduling.
 */
/* Kernels one pf_bin call launches for this shape (1, or 4 on the two-level
 * path for many primitives x many rows: per-chunk row counts, their prefix over
 * chunks, a stable scatter into per-row lists, then the column pass); -1 on bad
 * arguments. */
int pf_bin_launches(int n, int W, int H, int tile, int ty_begin, int ty_end);

int pf_bin(int n, int W, int H, int tile, int ty_begin, int ty_end, int capacity,
           void* scratch, size_t scratch_bytes,
           int32_t* bin_off, int32_t* bin_idx, int32_t* status,
           int32_t* tile_classes, void* stream);

/*
 * K3 — tiled front-to-back forward (16x16 tiles), optionally saving the
 * per-pixel contribution lists for the backward and optionally fusing the loss.
 * Replaces: forward_nosave / count_entries + fill_entries (_kernels.py:76-255),
 * render_forward (raster.py:290-363), and (when loss_kind != NONE) loss_mse /
 * loss_spatial (fit.py:112-151).
 *   tex        [4][texels] planar float64 atlas (RGB planes read when mu_blend > 0)
 *   quad       float32 [texels][4] alpha quad atlas from pf_atlas_quad
 *   bg4        float32 [H*W][4] per-pixel background (rgb, unused), or NULL for
 *              the solid (bg_r, bg_g, bg_b)
 *   saved      saved state (NULL = render only): pf_saved_bytes(capacity) bytes
 *              holding saved_entries = pf_saved_capacity(capacity) 16-byte
 *              entries (list position j, texel cell, bilinear weights, incoming
 *              transmittance T -- the reference's Tbuf, _kernels.py:294-297);
 *              ent_n int32 [H*W] per-pixel contribution counts
 *   img4       out float32 [H*W][4] = (r, g, b, alpha) (band rows written)
 *   tgt4       float32 [H*W][4] = (target r, g, b, target alpha); alpha read by SPATIAL
 *   d4         out float32 [H*W][4] = (dL/dI r, g, b, dL/dA)
 *   w_mse, w_gray  LossSpec.mse_w / gray_l1_w (PF_LOSS_COMBINED only)
 *   part       out float64 [n_band_tiles * 8 * 3]: per-warp loss partials
 *              (sum (I-t)^2; sum ((I-t)*mask)^2 or, for COMBINED, sum |(I-t).gray|;
 *              sum (I_a - t_a)^2), reduced in
 *              fixed order by pf_backward (deterministic loss value)
 *   inv_3P, inv_P  1/(3*H*W), 1/(H*W) of the FULL canvas (band-independent)
 */
int pf_forward(const void* rec, int n, const double* tex, const float* quad, int texels,
               const int32_t* bin_off, const int32_t* bin_idx, const int32_t* status,
               int W, int H, int ty_begin, int ty_end,
               double eps_skip, double mu_blend,
               double bg_r, double bg_g, double bg_b, const float* bg4,
               void* saved, long long saved_entries, int32_t* ent_n, float* img4,
               int loss_kind, const float* tgt4, double alpha_w, double w_mse, double w_gray,
               double inv_3P, double inv_P, float* d4, double* part, void* stream);

/*
 * K4 — backward: back-to-front over each pixel's saved contributions,
 * warp-level (shfl_xor butterfly) reduction of the 8 per-primitive gradients
 * before float64 atomics into grads.
 * Replaces: backward_tiles + reduce_partials (_kernels.py:258-363,
 * grad.py:134-206).  grads is ACCUMULATED into (caller zeroes it).
 *   d4     float32 [H*W][4] = (dL/dI r, g, b, dL/dA)
 *   grads  float64 [n][8], columns as params
 *   part   the forward's per-warp loss partials (or NULL); when given, block 0
 *          also reduces them in fixed order into sums[3] (loss value + psnr input)
 */
int pf_backward(const void* rec, int n, const double* tex, const float* quad, int texels,
                const int32_t* bin_off, const int32_t* bin_idx, const int32_t* status,
                const void* saved, long long saved_entries, const int32_t* ent_n,
                const float* d4, double bg_r, double bg_g, double bg_b, const float* bg4,
                double mu_blend, int W, int H, int ty_begin, int ty_end,
                double* grads, const double* part, double* sums, void* stream);

/*
 * Zero-padded fp32 alpha plane for pf_fit_step: template t occupies
 * (tpl_w[t] + 1) x (tpl_h[t] + 1) texels from tpl_pbase[t] (row stride w + 1);
 * the extra column / row are the reference's zero padding (_kernels.py:35-40).
 * apad out: float32 [pad_texels]; pad_texels >= sum (w+1)(h+1), a multiple of 4.
 */
int pf_atlas_pad(const double* tex, int texels, const int32_t* tpl_base, const int32_t* tpl_pbase,
                 const int32_t* tpl_w, const int32_t* tpl_h, int n_tpl, int pad_texels,
                 float* apad, void* stream);

/*
 * K34 — the fit step's render -> loss -> backward in one persistent kernel
 * (mu_blend == 0).  Replaces: the run_loop body render_forward(save=True) ->
 * evaluate_loss -> backward (fit.py:486-492; raster.py:290-363, fit.py:112-151,
 * grad.py:134-187).  Same decisions, compositing, loss and gradients as
 * pf_forward(save, loss) + pf_backward, but the padded alpha atlas and the
 * tile's records live in shared memory, the per-pixel contribution stack stays
 * on chip (depth >= 2 spills to `spill`) and dL/dI never leaves registers.
 *   apad    padded alpha plane from pf_atlas_pad (pad_texels floats)
 *   apad64  the same plane as float64 (pad_texels doubles), or NULL; staged in
 *           shared memory when it fits (no fp32->fp64 conversions on the hot path)
 *   spill   device scratch of pf_step_spill_bytes(capacity) bytes
 *   img4    optional out float32 [H*W][4] (r, g, b, alpha); NULL skips it
 *   part    out float64 [n_band_tiles * 8][3] per-warp loss partials (sum (I-t)^2,
 *           sum ((I-t)*mask)^2, sum (I_a-t_a)^2); fold them with pf_fold_loss or
 *           pass them to pf_adam_preprocess
 *   grads   float64 [n][8] accumulated into (zeroed by pf_adam_preprocess)
 *   counters uint32[4] zeroed once at allocation (tile ticket, finished producers,
 *           slot-mode grid barrier; self-resetting)
 *   tile_classes  pf_bin's tile classes of this band (longest-first schedule; the
 *           counts are re-zeroed for the next pf_bin), or NULL (tile order)
 *   stage   list entries staged in shared memory per tile: 32, or 64 for scenes
 *           with long tile lists (a hint: entries beyond it are read from L2)
 *   scratch, scratch_bytes, capacity, slots, slot_m
 *           slot mode (slots != NULL, see pf_slot_bytes): the lists come from the
 *           slots K1 filled (bin_off / bin_idx unused, may be NULL), sorted here
 *           by z rank; `scratch` is the K1 scratch (rects, iteration counter);
 *           K of the step is published to status[0] (status[1]: list overflow).
 *           NULL: CSR mode, lists from pf_bin.
 */
size_t pf_step_spill_bytes(int capacity);
int pf_fit_step(const void* rec, int n, const double* tex, const float* apad,
                const double* apad64, int pad_texels, int texels, const int32_t* bin_off, const int32_t* bin_idx, const int32_t* status,
                int W, int H, int ty_begin, int ty_end, double eps_skip,
                double bg_r, double bg_g, double bg_b, const float* bg4,
                int loss_kind, const float* tgt4, double alpha_w, double w_mse, double w_gray,
                double inv_3P, double inv_P, void* spill, float* img4, double* part,
                double* grads, uint32_t* counters,
                const int32_t* tile_classes, int stage, void* scratch, size_t scratch_bytes,
                int capacity, void* slots, int slot_m, void* stream);

/* Upstream gradients for PF_LOSS_EXTERN: rgb float32 [P][3] (dL/dI) and alpha
 * float32 [P] (dL/dA, or NULL = 0) into out4 float32 [P][4], the per-pixel rows
 * pf_fit_step stages (the autograd Function's backward). */
int pf_pack_grad4(const float* rgb, const float* alpha, int P, float* out4, void* stream);

/* loss_mse (fit.py:110-115) on the autograd path (ABI 7).  img4: the renderer's
 * (r, g, b, alpha) float32 rows [P][4]; target float32 [P][3].  pf_mse4 writes
 * mean((I - t)^2) over P x 3 to loss[0] (float32; per-pixel error in float32,
 * float64 partials folded in a fixed order); scratch: PF_MSE4_SCRATCH zeroed
 * doubles owned by the caller (self-resetting; one launch at a time per scratch).
 * pf_mse4_grad writes grad_out[0] * 2 (I - t) / (3 P) as (r, g, b, 0) rows into
 * out4 [P][4] -- the rows pf_fit_step(PF_LOSS_EXTERN) reads, no pf_pack_grad4. */
#define PF_MSE4_SCRATCH 2048
int pf_mse4(const float* img4, const float* target, int P, double* scratch, float* loss,
            void* stream);
int pf_mse4_grad(const float* img4, const float* target, int P, const float* grad_out,
                 float* out4, void* stream);

/* Fixed-order fold of n_part partial triples into sums[3] (deterministic: the
 * order depends on n_part only), many blocks + a last-block fold (ABI 8).
 * scratch: pf_fold_scratch_bytes(n_part) bytes, zeroed once at allocation
 * (self-resetting); one fold at a time per scratch. */
size_t pf_fold_scratch_bytes(int n_part);
int pf_fold_loss(const double* part, int n_part, double* sums, void* scratch, void* stream);

/*
 * Cross-band gradient exchange (row-band split; replaces the
 * sequential tile-order sum of reduce_partials, grad.py:190-206, across bands):
 * for i in [begin, end): s = srcs[0][i] + srcs[1][i] + ... (fixed order), then
 * dsts[k][i] = s for every k.  srcs / dsts are HOST arrays of device pointers
 * (<= PF_MAX_BANDS each; in place is allowed): the band buffers of one device,
 * or NVLink-mapped peer buffers with [begin, end) = this rank's slice (one-shot
 * reduce-scatter + all-gather).  Every destination gets bit-identical values.
 */
#define PF_MAX_BANDS 16
int pf_sum_bands(const double* const* srcs, int nsrc, double* const* dsts, int ndst,
                 long long begin, long long end, void* stream);

/*
 * K5 — fused Adam step (+ loss/psnr history, + gradient zeroing for the next step).
 * Replaces: adam_step (fit.py:195-238), lr_schedule lookup (fit.py:174-186),
 * psnr (fit.py:241-247) and the HistoryEntry bookkeeping (fit.py:505).
 * Two modes:
 *   table mode (iter != NULL): it = *iter; lr = lr_table[it]; bias corrections
 *     bc1_table[it] = 1 - 0.9^t, bc2_table[it] = 1 - 0.999^t (host-computed);
 *     hist_loss[it], hist_psnr[it] written from sums; *iter incremented.
 *   scalar mode (iter == NULL): lr, bc1, bc2 given as scalars; no history.
 *   gains8   host pointer to 8 per-column gains (NULL = all 1)
 *   frozen   uint8 [n] or NULL (OptimState.frozen)
 *   clamp    nonzero: clip the scale column to [s_min, s_max] (all rows)
 *   zero_grads nonzero: grads[0..8n) set to 0 after use
 *   sums     float64[3] from pf_forward (after any allreduce); loss_kind/alpha_w
 *            select mse or spatial for the history value
 *   counter  uint32 zeroed once (last-block detection)
 */
int pf_adam(double* params, double* grads, double* m, double* v, const uint8_t* frozen,
            const double* gains8, int n,
            const double* lr_table, const double* bc1_table, const double* bc2_table, int32_t* iter,
            double lr, double bc1, double bc2,
            int clamp, double s_min, double s_max, int zero_grads,
            const double* sums, int loss_kind, double alpha_w, double inv_3P, double inv_P,
            double* hist_loss, double* hist_psnr, uint32_t* counter, void* stream);

/*
 * f4 layered export (exportio.py:272-346): every primitive alone over its own
 * pixel box of the rho-times denser canvas (scale_scene: x' = rho x + (rho-1)/2,
 * s' = rho s), premultiplied RGBA.
 *   pf_layer_bboxes: bbox out int32 [n][4] (x0, y0, x1, y1; -1 rows = fully off
 *   canvas, the reference's DegenerateBBox), area out int64 [n], offsets out
 *   int64 [n + 1] (exclusive scan; offsets[n] = total pixels).
 *   pf_render_layers: rgba out float32 [offsets[n]][4], layer i at offsets[i],
 *   row-major over its box.  tpl_q = aspect per template (as pf_scratch_init).
 */
int pf_layer_bboxes(const double* params, const int32_t* template_id, const double* tpl_hyp,
                    int n, int W, int H, int rho, int32_t* bbox, long long* area,
                    long long* offsets, void* stream);
int pf_render_layers(const double* params, const int32_t* template_id, const double* tex,
                     int texels, const int32_t* tpl_base, const int32_t* tpl_w,
                     const int32_t* tpl_h, const double* tpl_q, int n, double alpha_max,
                     double mu_blend, int rho, const int32_t* bbox, const long long* offsets,
                     float* rgba, void* stream);

/*
 * f3 video heuristics (dyn.py:86-177).
 *   pf_diff_mask: prev, cur float64 [H][W][3]; mask out uint8 [H][W] =
 *     max_c |prev - cur| > tau                                    (diff_mask)
 *   pf_freeze_flags: frozen out uint8 [n] = 1 iff the binning box (padding)
 *     holds no changed pixel                                      (freeze_flags)
 *   pf_remove_stuck: per (grid_rows x grid_cols) region, at most k primitives
 *     (not frozen, scale >= tau_scale * W, alpha >= tau_alpha, depth rank >=
 *     zeta * members; ordered by scale * alpha desc, index asc) get their
 *     opacity logit scaled by eta IN params; decayed out uint8 [n]  (remove_stuck)
 *     z int32 [n]; frozen uint8 [n] or NULL; scratch pf_stuck_scratch_bytes.
 */
int pf_diff_mask(const double* prev, const double* cur, int W, int H, double tau, uint8_t* mask,
                 void* stream);
int pf_freeze_flags(const double* params, const int32_t* template_id, const double* tpl_hyp,
                    int n, int W, int H, double padding, const uint8_t* mask, uint8_t* frozen,
                    void* stream);
size_t pf_stuck_scratch_bytes(int n, int regions);
int pf_remove_stuck(double* params, const int32_t* z, const uint8_t* frozen, int n, int W, int H,
                    int grid_rows, int grid_cols, int k, double tau_scale, double tau_alpha,
                    double zeta, double eta, double alpha_max, uint8_t* decayed, void* scratch,
                    size_t scratch_bytes, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* PRIMFIT_B200_H */
