/*
 * fcn.h -- C ABI of the B200-native homomorphic evaluation path
 * (Faster CryptoNets / reference package `hecnet`).
 *
 * The reference is pure Python + numpy and has no FFI of its own; the entry
 * points below are what its Python functions would bind through ctypes.
 * Each declaration cites the reference function it replaces.
 *
 * Conventions (all mirror the reference's ring/fv contracts):
 *  - residues are canonical uint64 in [0, q_i) at every boundary
 *    (reference ring.py:140-150);
 *  - a polynomial is `limbs` rows of n coefficients, limb-major; a
 *    ciphertext is [2][k][n] (c0 then c1) -- byte-identical to the body of
 *    the reference serialization after its 64-byte header (fv.py:610-619);
 *    a batch of B ciphertexts is [B][2][k][n];
 *  - device pointers are caller-owned device memory; `stream` is a
 *    cudaStream_t (NULL = legacy default stream); calls are asynchronous
 *    on that stream unless stated otherwise;
 *  - every function returns FCN_OK (0) or a negative error code, with a
 *    thread-local message from fcn_last_error().  The Python host maps
 *    FCN_ERR_ARG/PARAM to RingError/FVError (ring.py:28, fv.py:38).
 *  - compute is GPU-only: there is no CPU fallback in this library.
 */
#ifndef FCN_H_
#define FCN_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define FCN_OK 0
#define FCN_ERR_ARG (-1)   /* bad argument / shape mismatch            */
#define FCN_ERR_PARAM (-2) /* unsupported or invalid parameter set     */
#define FCN_ERR_CUDA (-3)  /* CUDA runtime failure                     */
#define FCN_ERR_STATE (-4) /* e.g. workspace too small                 */

typedef struct fcn_ring fcn_ring; /* RNS ring Z_q[x]/(x^n+1) with NTT tables */
typedef struct fcn_ctx fcn_ctx;   /* one FV parameter set                    */
typedef struct fcn_keys fcn_keys; /* device-resident relinearization keys   */

const char* fcn_last_error(void);
int fcn_version(void);
/* Number of kernels this library has launched in the process (bench evidence). */
long long fcn_launch_count(void);
/* Per-stage CUDA-event timing of fcn_mul_ct_ex / fcn_mul_ct_multi (bench and
 * profiling aid; no reference counterpart).  fcn_stage_timing(1) clears the
 * record and starts recording events around every stage of every chunk on
 * the call's stream (skipped while a stream is being captured);
 * fcn_stage_timing(0) clears and stops.  fcn_stage_times synchronises the
 * recorded events and writes the summed milliseconds per stage id:
 * 0 lift, 1 forward NTT (+ fused tensor), 2 tensor INTT, 3 exact rescale +
 * digits, 4 digit NTT, 5 key MAC, 6 final INTT + epilogue.                 */
int fcn_stage_timing(int enable);
int fcn_stage_times(double* ms_out, int n_stages);
/* Reduction schedule the FP64 NTT uses for a transform of size 2^logn whose
 * largest limb is qmax: 0 = reduce every third stage (any q < 2^51), 1 = once
 * per transform, 2 = never (host-only diagnostic; no reference counterpart). */
int fcn_ntt_f64_schedule(int logn, uint64_t qmax);

/* ---------------------------------------------------------------- rings */

/* RingContext.create(n, primes) (ring.py:104-125) with the tables of
 * ModulusLimb._build_limb (ring.py:67-101): root = primitive_2n_root
 * (modmath.py:136-149), psi^bitrev(i) / psi^-bitrev(i), Shoup quotients.
 * n: power of two in [4, 32768]; every prime < 2^62, prime, = 1 mod 2n. */
int fcn_ring_create(int device, int n, int count, const uint64_t* primes, fcn_ring** out);
int fcn_ring_destroy(fcn_ring* ring);
/* Copy the per-limb primitive 2n-th roots (host array of `count`). */
int fcn_ring_roots(const fcn_ring* ring, uint64_t* roots_out);

/* Rows: d_data is [n_rows][n]; row r uses limb (limb_offset + r % limb_period).
 * ring.ntt_forward (ring.py:242-247, CT over psis[m:2m], bit-reversed out).  */
int fcn_ntt_forward(const fcn_ring* ring, uint64_t* d_data, int64_t n_rows, int limb_period,
                    int limb_offset, void* stream);
/* ring.ntt_inverse (ring.py:250-255, GS over ipsis[h:m], then * n^-1).      */
int fcn_ntt_inverse(const fcn_ring* ring, uint64_t* d_data, int64_t n_rows, int limb_period,
                    int limb_offset, void* stream);

/* Elementwise ring ops over rows (ring.py:261-300).  op: 0 add, 1 sub,
 * 2 neg (b ignored), 3 pointwise mul (NTT domain, modmath.mul_mod).
 * b has b_rows rows and is broadcast: row r of a pairs with b row
 * (r % b_rows); b_rows must divide n_rows and be a multiple of the
 * limb period (b_rows == n_rows is the plain elementwise case).         */
#define FCN_OP_ADD 0
#define FCN_OP_SUB 1
#define FCN_OP_NEG 2
#define FCN_OP_MUL 3
int fcn_poly_binary(const fcn_ring* ring, int op, const uint64_t* d_a, const uint64_t* d_b,
                    int64_t b_rows, uint64_t* d_out, int64_t n_rows, int limb_period, int limb_offset,
                    void* stream);

/* RingPoly.from_int_coeffs / fv._signed_to_ringpoly (ring.py:156-168,
 * fv.py:220-225) batched: d_vals [count][n] signed -> d_out
 * [count][limbs][n] residues mod q_(offset + l).                         */
int fcn_lift_signed(const fcn_ring* ring, const int64_t* d_vals, int64_t count, uint64_t* d_out, int limbs,
                    int limb_offset, void* stream);

/* ring.scalar_mul (ring.py:282-288): out = a * c mod q_i with c given as
 * per-limb canonical residues (host array of limb_period values).          */
int fcn_scalar_mul(const fcn_ring* ring, const uint64_t* d_a, const uint64_t* c_res, uint64_t* d_out,
                   int64_t n_rows, int limb_period, int limb_offset, void* stream);

/* ring.poly_mul_monomial (ring.py:339-361): out = coeff * x^k * a with the
 * negacyclic wrap; coeff given as per-limb residues (host, limb_period).  */
int fcn_poly_mul_monomial(const fcn_ring* ring, const uint64_t* d_a, int k, const uint64_t* c_res,
                          uint64_t* d_out, int64_t n_rows, int limb_period, int limb_offset,
                          void* stream);

/* ------------------------------------------------------------ FV context */

/* EncryptionParams (fv.py:42-124): q-limbs, plaintext lanes, beta = 2^log2_beta.
 * Derives ell (fv.py:78-85), Delta = q // t (fv.py:87-88), the auxiliary
 * base and all exact-rescale constants.  The
 * reference's auxiliary base is find_ntt_primes(n, (bitlen(n)+bitlen(q)+1)
 * //54+1, 55, exclude=q) (fv.py:99-107); the result of mul_ct does not depend
 * on which base extends q as long as its product P exceeds 2nq, so the
 * context instead takes the first NTT primes in (2^50, 2^51) (ascending
 * scan, q-limbs excluded) with the smallest count giving P >= 8nq -- limbs
 * below 2^51 keep every mul_ct kernel on the exact FP64 path (csrc/fv.cu,
 * fcn_ctx_create).  When a q-limb is >= 2^51 the integer kernels run instead;
 * a set for which (2^50, 2^51) holds too few NTT primes is rejected with
 * FCN_ERR_PARAM.  fcn_ctx_aux_primes returns the base.                      */
int fcn_ctx_create(int device, int n, int k, const uint64_t* primes, int n_lanes,
                   const uint64_t* t_lanes, int log2_beta, fcn_ctx** out);
int fcn_ctx_destroy(fcn_ctx* ctx);
/* The ring over the extended base (q-limbs first, then aux): q-base ops
 * use it with limb_period = k, limb_offset = 0.                          */
int fcn_ctx_ring(const fcn_ctx* ctx, const fcn_ring** out);
/* what: 0 n, 1 k, 2 aux count m, 3 ell, 4 n_lanes, 5 log2_beta,
 * 6 whether mul_ct's lift/rescale run the exact-size FP64 kernels (1) or
 * the integer ones (0; a one-line notice goes to stderr at creation),
 * 7 whether squares relinearise through the shared prime pair (digits
 * transformed under q_0, q_1 only, the sums of the other limbs rebuilt by a
 * two-residue CRT; same bytes as the per-limb form, fv.py:524-537;
 * FCN_PAIR_RELIN=0 at creation turns it off).                             */
int fcn_ctx_query(const fcn_ctx* ctx, int what, int64_t* value);
int fcn_ctx_aux_primes(const fcn_ctx* ctx, uint64_t* out_m);

/* EvalKeys (fv.py:191-198): host arrays a, g of shape [ell+1][k][n] in the
 * coefficient domain (the eval-key serialization body, fv.py:660-664).
 * Copied to the device and NTT-transformed there.                         */
int fcn_keys_create(const fcn_ctx* ctx, const uint64_t* a, const uint64_t* g, fcn_keys** out);
int fcn_keys_destroy(fcn_keys* keys);

/* ---------------------------------------------------------- evaluation */

/* Sparse plaintext add (fv.add_pt, fv.py:418-431 via _delta_m :284-292):
 * for each term e: ct[ct_index[e]].c0[pos[e]] += coef[e] * Delta_lane
 * (mod q_i).  coef is the centered plaintext coefficient.  In place;
 * positions must be distinct within one ciphertext.                       */
int fcn_add_plain_terms(const fcn_ctx* ctx, int lane, uint64_t* d_cts, int64_t n_terms,
                        const int32_t* d_ct_index, const int32_t* d_pos, const int64_t* d_coef,
                        void* stream);

/* Fused sparse linear layer (engine.py:698-717 lin_out; per term
 * fv.mul_pt monomial path fv.py:449-453 + ring.poly_mul_monomial, chained
 * by fv.add_ct fv.py:394-403):
 *   out[o] = sum_{e in [rowptr[o], rowptr[o+1])} coef[e] * x^rot[e] * in[col[e]]
 * over both ciphertext polys and all k limbs.  Inputs are addressed as the
 * concatenation of d_in0 (n_in0 cts) and d_in1 (n_in1 cts, may be NULL).
 * coef: signed centered plaintext coefficient; rot in [0, n).  Rows with
 * no terms produce the all-zero ciphertext (Ciphertext.zero, fv.py:210). */
int fcn_linear_mac(const fcn_ctx* ctx, const uint64_t* d_in0, int64_t n_in0, const uint64_t* d_in1,
                   int64_t n_in1, const int32_t* d_rowptr, const int32_t* d_col, const int32_t* d_rot,
                   const int64_t* d_coef, uint64_t* d_out, int64_t n_out, void* stream);
/* Same, with host-known layer facts enabling the fast path: no_rot != 0
 * when every rot is 0 (constant plaintexts, the SIMD-batched encoding) and
 * max_abs_coef = max |coef| (0 = unknown).  Output is identical.          */
int fcn_linear_mac_ex(const fcn_ctx* ctx, const uint64_t* d_in0, int64_t n_in0, const uint64_t* d_in1,
                      int64_t n_in1, const int32_t* d_rowptr, const int32_t* d_col, const int32_t* d_rot,
                      const int64_t* d_coef, uint64_t* d_out, int64_t n_out, int no_rot, uint64_t max_abs_coef,
                      void* stream);

/* Output fan-out (sharded evaluation): the kernel's final
 * store writes the same n_out ciphertexts to each of the n_dst (1..8)
 * destinations -- this GPU's buffer and the peers' buffers mapped over
 * NVLink (torch symmetric memory) -- so the per-stage all-gather
 * (engine.py:682-690 merges independent outputs) happens inside the layer
 * kernel.  d_outs is a HOST array of device pointers.                     */
#define FCN_MAX_FANOUT 8
int fcn_linear_mac_multi(const fcn_ctx* ctx, const uint64_t* d_in0, int64_t n_in0, const uint64_t* d_in1,
                         int64_t n_in1, const int32_t* d_rowptr, const int32_t* d_col, const int32_t* d_rot,
                         const int64_t* d_coef, uint64_t* const* d_outs, int n_dst, int64_t n_out, int no_rot,
                         uint64_t max_abs_coef, void* stream);

/* The same linear layer on the tensor cores (csrc/mac_tc.cu) for plans whose
 * terms are signed constants |c| <= 127 without rotation (the SIMD-batched
 * encoding of engine.py:698-717's mul_pt + add_ct chain): every residue is
 * split into P = fcn_tc_planes(ctx) byte planes (limbs in [2^32, 2^64)), the
 * planes are multiplied by the int8 weights with tcgen05.mma kind::i8 into
 * exact int32 sums, and the epilogue folds them back mod q_l.  Bit-identical
 * to fcn_linear_mac_multi on the same plan.
 *   fcn_split_planes: d_in [count][2][k][n] u64 -> d_planes [count][P][2kn + 256]
 *     u8 (each plane row padded by 256 bytes: fcn_tc_planes_bytes gives the size).
 *   fcn_linear_mac_tc: d_groups [n_groups][8] int32 = {row_off, m, k_off,
 *     n_k, w_off, 0, 0, 0} (m <= 128 output rows d_rows[row_off..+m), inputs
 *     d_kidx[k_off..+n_k), weights: ceil(n_k/64) 8 KB tiles from tile w_off
 *     of d_wimg, int8, byte (m, kk) of a tile at (m/8)*512 + (kk/16)*128 +
 *     (m%8)*16 + kk%16, zero beyond m rows / n_k inputs).  Writes the output
 *     rows in [row_lo, row_hi) to every destination (row r at r - row_lo).
 * Returns 0 planes / FCN_ERR_PARAM when the limbs do not fit 5..8 bytes.     */
int fcn_tc_planes(const fcn_ctx* ctx);
size_t fcn_tc_planes_bytes(const fcn_ctx* ctx, int64_t count);
int fcn_split_planes(const fcn_ctx* ctx, const uint64_t* d_in, int64_t count, uint8_t* d_planes, void* stream);
int fcn_linear_mac_tc(const fcn_ctx* ctx, const uint8_t* d_planes, int64_t n_in, int64_t n_groups,
                      const int32_t* d_groups, const int32_t* d_kidx, const int32_t* d_rows, const int8_t* d_wimg,
                      uint64_t* const* d_outs, int n_dst, int64_t row_lo, int64_t row_hi, void* stream);

/* fv.mul_ct (fv.py:498-549): exact tensor in the extended base, exact
 * floor((t*T + q>>1)/q) mod q, base-beta digits of c2', key switching.
 * d_b == NULL computes the square a*a.  `count` ciphertexts [count][2][k][n].
 * Workspace: device scratch of fcn_mul_ct_workspace_bytes(ctx, chunk)
 * bytes; batches larger than the chunk the workspace allows are processed
 * in chunks.                                                              */
size_t fcn_mul_ct_workspace_bytes(const fcn_ctx* ctx, int64_t chunk);
int fcn_mul_ct(const fcn_ctx* ctx, const fcn_keys* keys, int lane, const uint64_t* d_a,
               const uint64_t* d_b, uint64_t* d_out, int64_t count, void* d_workspace,
               size_t workspace_bytes, void* stream);

/* fcn_mul_ct with an optional fused epilogue.  flags & FCN_MUL_ACT (squares
 * only, d_b == NULL): out = act_c2 * a^2 + act_c1 * a (mod q), i.e. the
 * reference's polynomial activation a2*x^2 + a1*x (engine.py:744-770:
 * mul_ct, two mul_pt of constant plaintexts, add_ct) evaluated in the last
 * kernel of the product;
 * identical to fcn_mul_ct followed by fcn_linear_mac over [a^2 ; a] with the
 * coefficients (act_c2, act_c1).  flags == 0: plain fcn_mul_ct.           */
#define FCN_MUL_ACT 1
int fcn_mul_ct_ex(const fcn_ctx* ctx, const fcn_keys* keys, int lane, const uint64_t* d_a,
                  const uint64_t* d_b, uint64_t* d_out, int64_t count, int flags, int64_t act_c2,
                  int64_t act_c1, void* d_workspace, size_t workspace_bytes, void* stream);
/* fcn_mul_ct_ex with output fan-out to n_dst destinations (see above).   */
int fcn_mul_ct_multi(const fcn_ctx* ctx, const fcn_keys* keys, int lane, const uint64_t* d_a,
                     const uint64_t* d_b, uint64_t* const* d_outs, int n_dst, int64_t count, int flags,
                     int64_t act_c2, int64_t act_c1, void* d_workspace, size_t workspace_bytes, void* stream);

/* Key-switching inner product of fv.mul_ct (fv.py:533-537) on NTT-domain
 * rows: acc[c][0] = sum_d g_d * D[c][d], acc[c][1] = sum_d a_d * D[c][d]
 * (mod q_l, pointwise), for digits [count][D][k][n] already forward-NTT'd
 * per limb; acc [count][2][k][n].  The kernel fcn_mul_ct runs between its
 * digit NTT and its final inverse NTT, exported for measurement.          */
int fcn_key_mac(const fcn_ctx* ctx, const fcn_keys* keys, const uint64_t* d_digits, uint64_t* d_acc,
                int64_t count, void* stream);

/* fv.decrypt core (fv.py:337-353): given w = [c0 + c1 s]_q as RNS rows
 * [count][k][n], write m = floor((w t + q>>1)/q) mod t as [count][n].     */
/* Noise budget (fv.noise_budget, fv.py:356-377) on the GPU: for each of the
 * `count` polynomials w = c0 + c1 s in d_w ([count][k][n] residues), every
 * one of `blocks` CTAs writes the largest |centred [t w]_q| of its share of
 * the coefficients as `out_words` little-endian u64 words (>= the words of
 * q) to d_out[count][blocks][out_words]; the host takes the maximum over
 * the blocks and the reference's log2(q) - 1 - log2(worst).               */
int fcn_noise_max(const fcn_ctx* ctx, int lane, const uint64_t* d_w, int64_t count, uint64_t* d_out, int blocks,
                  int out_words, void* stream);
int fcn_decrypt_round(const fcn_ctx* ctx, int lane, const uint64_t* d_w, uint64_t* d_m, int64_t count,
                      void* stream);

/* Diagnostics: number of coefficients that took the exact multiword
 * fallback of the fixed-point rescale since context creation.           */
int fcn_ctx_fallback_count(const fcn_ctx* ctx, int64_t* value);

#ifdef __cplusplus
}
#endif
#endif /* FCN_H_ */
