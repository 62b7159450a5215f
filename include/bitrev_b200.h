/*
 * bitrev_b200.h -- C ABI of libbitrev_sm100a.so, the B200 (sm_100a) bit-reversed
 * permutation library.
 *
 * The permutation: for an array a of length n = 2^b, element i moves to slot
 * rev_b(i) (rev_b reverses the low b bits of i).  It is an involution, so
 * "dst[rev(i)] = src[i]" and "dst[i] = src[rev(i)]" are the same map.
 *
 * Every entry point here replaces a numba kernel (or the Python wrapper that
 * validates and calls it) of the reference package `bitrev`
 * (/root/reference/pkg/src/bitrev, cited as src/ below).  Those kernels take
 * numpy arrays; the C ABI takes plain device pointers, sizes in ELEMENTS of
 * elem_bytes bytes, and a cudaStream_t passed as void* (NULL = legacy default
 * stream).  No torch types cross this boundary.
 *
 * Conventions (all entry points):
 *   - return 0 on success;
 *   - return a NEGATIVE BITREV_E* code for an invalid argument (nothing was
 *     launched; the Python layer has normally raised ValueError before);
 *   - return a POSITIVE cudaError_t value if a CUDA call failed.
 *   - Device entry points only ENQUEUE work on `stream`: they neither allocate
 *     nor synchronise.  The *_host entry points are synchronous (they return
 *     when the result is in host memory), like the reference functions.
 *   - Stateless apart from per-device caches of occupancy; safe to call from
 *     several host threads on distinct arrays (the reference's nogil contract,
 *     SPEC.md:253).
 *   - elem_bytes in {1, 2, 4, 8, 16}.  4/8/16-byte elements on 16-byte aligned
 *     pointers take the shared-memory tile kernels; anything else takes a
 *     correct but slower element-wise kernel.
 *   - Width domain b in [1, 48] (src/bits.py:15-23 MAX_BITS / check_width).
 */
#ifndef BITREV_B200_H
#define BITREV_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define BITREV_OK 0
#define BITREV_EWIDTH (-1)    /* b outside 1..48 (src/bits.py:21-23)            */
#define BITREV_EELEM (-2)     /* elem_bytes not in {1,2,4,8,16}                  */
#define BITREV_ENULL (-3)     /* NULL data pointer                               */
#define BITREV_EBATCH (-4)    /* batch < 1 or a batch stride < 2^b               */
#define BITREV_EOVERLAP (-5)  /* src/dst ranges overlap (src/permutations.py:305) */
#define BITREV_ESHARD (-6)    /* sharded plan needs 1 <= 2g <= b_local + g       */
#define BITREV_ETILE (-7)     /* tile-bits override not supported               */
#define BITREV_ESTAGES (-8)   /* FFT pre-pass: unsupported number of stages      */
#define BITREV_EALIGN (-9)    /* FFT pre-pass tiles: rows not 16-byte aligned    */

/* Library version string, e.g. "bitrev_b200 0.1.0 sm_100a". */
const char* bitrev_version(void);

/* Human-readable text for any return code above. */
const char* bitrev_strerror(int code);

/*
 * Out-of-place permutation dst[rev_b(i)] = src[i] for `batch` independent rows.
 * Row r of src starts at src + r*src_batch_stride elements (same for dst).
 * Replaces: cobra_out_of_place -> _cobra_copy (src/permutations.py:293-308,
 * 225-249); also serves oracle_permute (src/verify.py:34-39) and make_method
 * ("cobra") (src/bench.py:164-171).  batch > 1 is an extension for the batched
 * FFT pre-pass (BASELINE config 4); the reference handles one 1-D array.
 * src and dst must not overlap (BITREV_EOVERLAP otherwise).
 */
int bitrev_oop(const void* src, void* dst, int b, int elem_bytes, int64_t batch,
               int64_t src_batch_stride, int64_t dst_batch_stride, void* stream);

/*
 * In-place permutation of `batch` rows of a.  Each unordered tile pair
 * {y, rev(y)} of the middle index bits is swapped by exactly one CTA.
 * Replaces: cobra_in_place -> _cobra_swap (src/permutations.py:311-321,
 * 252-285), and (identical output) recursive_permute /
 * semi_recursive_permute (src/recursive.py:189-228),
 * parallel_semi_recursive_permute (src/parallel.py:95-156),
 * stockham_permute, naive_bitwise_permute, bytetable_permute, xor_permute,
 * pair_bitwise_permute (src/permutations.py:46-180) and apply_schedule with a
 * full schedule (src/schedule.py:124-130).
 */
int bitrev_inplace(void* a, int b, int elem_bytes, int64_t batch, int64_t batch_stride,
                   void* stream);

/*
 * Host-buffer variants: H2D copy into caller-provided device scratch, the
 * kernel, D2H copy back, then stream synchronisation.  host_* may be pageable
 * or pinned (pinned is faster).  dev_src/dev_dst (oop) and dev_buf (in-place)
 * must each hold batch * 2^b elements, or be NULL: the library then takes
 * stream-ordered scratch (cudaMallocAsync) and frees it before returning.
 * This is the call a numpy-array caller of the reference API lands on.
 */
int bitrev_oop_host(const void* host_src, void* host_dst, int b, int elem_bytes, int64_t batch,
                    void* dev_src, void* dev_dst, void* stream);
int bitrev_inplace_host(void* host_a, int b, int elem_bytes, int64_t batch, void* dev_buf,
                        void* stream);

/*
 * Stream `count` independent host arrays (each `batch` rows of 2^b elements)
 * through the GPU with the transfers overlapped: while array k is copied
 * host->device, array k-1 is permuted and array k-2 copied back, on three
 * internal streams (copy-in, compute, copy-out) over three device slots.
 * PCIe is full duplex, so with pinned host memory the per-array time tends
 * to max(H2D, D2H) instead of their sum.  host_dst[k] may equal host_src[k]
 * (in place on the host), and a host array may recur in the sequence: a copy
 * in waits for any in-flight copy out to the same host memory.  Ordered after
 * prior work on `stream`; synchronous.
 * dev_scratch: NULL (stream-ordered allocation) or 3 * batch * 2^b *
 * elem_bytes bytes.  No reference counterpart: the extension a caller with
 * many host arrays (the FFT pre-pass of BASELINE config 4) needs.
 */
int bitrev_host_pipeline(const void* const* host_src, void* const* host_dst, int64_t count, int b,
                         int elem_bytes, int64_t batch, void* dev_scratch, void* stream);

/*
 * Square in-place transpose of the 2^h x 2^h row-major matrix at a
 * (`batch` matrices, batch_stride elements apart).
 * Replaces: transpose_square_inplace -> _transpose_diag/_transpose_offdiag
 * (src/recursive.py:30-81).
 */
int bitrev_transpose_square(void* a, int h, int elem_bytes, int64_t batch, int64_t batch_stride,
                            void* stream);

/*
 * Even-odd split out of place: dst[j] = src[2j], dst[n/2 + j] = src[2j+1].
 * Replaces: even_odd_permute -> _even_odd (src/recursive.py:84-107); the
 * reference runs it in place through an n/2 scratch, the Python layer does
 * the same through a device scratch.
 */
int bitrev_even_odd(const void* src, void* dst, int b, int elem_bytes, int64_t batch,
                    int64_t src_batch_stride, int64_t dst_batch_stride, void* stream);

/*
 * Fill scratch[0 .. 2^b) with what the reference's stockham_permute leaves in
 * a caller-supplied scratch buffer (the last block's split of every level of
 * its buffered passes), gathered from the UNPERMUTED array a; call it before
 * permuting a.  Replaces: the side effect of _stockham on its scratch
 * argument (src/permutations.py:30-59); the permutation itself is
 * bitrev_inplace.  a and scratch must not overlap.
 */
int bitrev_stockham_scratch(const void* a, void* scratch, int b, int elem_bytes, void* stream);

/*
 * Swap a[pairs[2k]] <-> a[pairs[2k+1]] for k < npairs, pairs a device array of
 * int64 index pairs that must be pairwise disjoint (a swap schedule is).
 * Replaces: apply_schedule -> _apply_pairs (src/schedule.py:100-130) for a
 * caller-supplied pair list; a complete schedule takes bitrev_inplace instead.
 */
int bitrev_apply_pairs(void* a, const void* pairs, int64_t npairs, int elem_bytes, void* stream);

/*
 * FFT pre-pass: dst = the first `stages` radix-2 decimation-in-time butterfly
 * stages applied to bit-reversed src, per row (complex64: elem_bytes 8,
 * complex128: 16; forward twiddles exp(-2 pi i k / 2^s), or conjugated when
 * inverse != 0, no normalisation).  stages = 0 is the plain permutation;
 * stages = b is a complete unnormalised radix-2 FFT.  Rows of n*E <= 64 KB
 * (16-byte aligned; 32 KB otherwise) take any stages <= b; larger rows fuse
 * up to 7 (complex64) or 6 (complex128) stages into the drain of rectangular
 * tiles whose destination rows are the FFT blocks, at the permutation's HBM
 * traffic.
 * Serves the downstream step the reference's permutation exists for
 * (SURVEY.md 8(f) f2).  No reference counterpart.
 */
int bitrev_dit_prepass(const void* src, void* dst, int b, int elem_bytes, int64_t batch,
                       int64_t src_batch_stride, int64_t dst_batch_stride, int stages,
                       int inverse, void* stream);

/*
 * bitrev_dit_prepass over `count` host arrays with the transfers overlapped,
 * like bitrev_host_pipeline: array k's host->device copy runs beside array
 * k-1's kernel and array k-2's copy back.  host_dst[k] may equal
 * host_src[k].  Pinned host arrays overlap both copy directions; pageable
 * ones go one array at a time through pinned bounce buffers.  Ordered after
 * prior work on `stream`; synchronous.  dev_scratch: NULL (stream-ordered
 * allocation) or 6 * batch * 2^b * elem_bytes bytes (an input and an output
 * buffer for each of three slots).  No reference counterpart (SURVEY.md 8(f)
 * f2, the batched FFT pre-pass of BASELINE config 4 on host data).
 */
int bitrev_dit_prepass_host_pipeline(const void* const* host_src, void* const* host_dst,
                                     int64_t count, int b, int elem_bytes, int64_t batch,
                                     int stages, int inverse, void* dev_scratch, void* stream);

/*
 * Steps 1+2 of the top-bit sharded plan fused (no reference counterpart;
 * SURVEY.md 8(e)): rank `rank` of G = 2^g bit-reverses its local shard of
 * 2^b_local elements and stores each destination row straight into
 * peer_recv[d] (the receive buffer of rank d, G entries, G <= 8) at element
 * rank*C + k, C = 2^(b_local-g) -- i.e. what the all-to-all would deliver.
 * With peer pointers mapped over NVLink/NVSwitch (symmetric memory or CUDA
 * IPC) the stores cross the fabric from the SMs; after a cross-rank barrier
 * every rank runs bitrev_sharded_unpack on its receive buffer.  Requires
 * b_local - g >= the tile bits (rows never straddle two chunks).
 */
int bitrev_sharded_scatter(const void* local, void* const* peer_recv, int b_local, int g, int rank,
                           int elem_bytes, void* stream);

/*
 * apply_schedule with an explicit pair list whose pairs may share indices
 * (replaces _apply_pairs, src/schedule.py:100-107): the pairs are swapped one
 * after another in list order by a single device thread, so the result is
 * the reference's for any list.  Indices must lie in [0, 2^b) (the Python
 * layer checks).  Disjoint lists should use bitrev_apply_pairs.
 */
int bitrev_apply_pairs_ordered(void* a, const void* pairs, int64_t npairs, int elem_bytes,
                               void* stream);

/*
 * The complete swap schedule of width b in the reference's emission order
 * (generate_swap_schedule, src/schedule.py:77-91): swap_count(b) int64 pairs
 * (i, rev_b(i)), i < rev_b(i), written to the device array pairs_out
 * (2 * swap_count(b) int64).  Generated on the device, one thread per pair.
 */
int bitrev_swap_schedule(int b, void* pairs_out, void* stream);

/*
 * Step 1 of the top-bit sharded plan for an all-to-all in 2^chunk_bits
 * rounds (no reference counterpart): the local reversal of
 * the 2^b_local-element shard written to `send` in the layout
 * [sub-chunk c][destination d][k'], sub-chunk length S = 2^(b_local-g-chunk_bits),
 * for local output index u = d*C + c*S + k'.  Row c of `send` (G*S elements)
 * is then the equal-split input of one all-to-all round.  chunk_bits = 0 is
 * exactly bitrev_oop.  Requires b_local >= 2g + chunk_bits, G <= 8, and (for
 * chunk_bits > 0) S >= the scatter tile side (64 / 32 / 32 for 4 / 8 / 16 B).
 */
int bitrev_sharded_pack(const void* local, void* send, int b_local, int g, int chunk_bits,
                        int elem_bytes, void* stream);

/*
 * Step 3 of the top-bit sharded plan (no reference counterpart: the reference
 * has no multi-device path).  recv holds G = 2^g
 * chunks of C = 2^(b_local-g) elements, chunk r received from rank r;
 * writes dst[k*G + rev_g(r)] = recv[r*C + k].
 */
int bitrev_sharded_unpack(const void* recv, void* dst, int b_local, int g, int elem_bytes,
                          void* stream);

/*
 * Tile-bit parameter of the shared-memory kernels (the GPU analogue of
 * CobraConfig.q, src/permutations.py:187-216; tuned like tune_cobra,
 * src/bench.py:380-433).  Output never depends on it.  inplace selects the
 * in-place kernel family.  set returns BITREV_ETILE if q is not instantiated
 * for that element size; q = 0 restores the default.
 */
int bitrev_get_tile_bits(int elem_bytes, int inplace);
int bitrev_set_tile_bits(int elem_bytes, int inplace, int q);

/*
 * Staging path of the shared-memory kernels for (element size, family):
 * 0 = register staging (LDG.128 -> registers -> STS), 1 = TMA bulk ring
 * (cp.async.bulk row copies into a multi-stage shared-memory ring completing
 * on mbarriers), 2 = TMA tensor ring (one cp.async.bulk.tensor per tile),
 * 3 = rectangular register tiles (out of place only), 4 = element-granular
 * cp.async into the transposed layout (in place only), 5 = register loads +
 * TMA tensor stores from a swizzled staging buffer (in place only).  Output never depends
 * on it; a (q, path) pair that is not instantiated falls back to path 0.
 * Initial value from the environment (BITREV_B200_PATH_OOP /
 * BITREV_B200_PATH_IP), else the measured default.
 */
int bitrev_get_tile_path(int elem_bytes, int inplace);
int bitrev_set_tile_path(int elem_bytes, int inplace, int path);

/*
 * The (tile bits, staging path) of the calling thread's most recent
 * successful bitrev_oop / bitrev_inplace launch -- the choice tune_cobra's
 * report names for the reference (src/bench.py:380-433).  path -3 = short-row
 * kernel (16-byte aligned rows of 4/8/16-byte elements, n*E <= 32 KB, many
 * rows per CTA), -1 = whole-row kernel (other rows of n*E <= 32 KB), -2 =
 * element-wise kernel (unaligned views, 1/2-byte elements); q is 0 for all
 * three.  With the knobs at their default values,
 * launches below per-family byte budgets (8-64 MiB per side) use smaller
 * mid-size tiles: one large tile per SM leaves too few tiles to balance a
 * persistent grid there (tools/mid_sizes.py, mid_tier in bitrev_capi.cu).
 */
int bitrev_last_tile(int* q, int* path);

/*
 * Tile visit order of the shared-memory kernels: 0 = middle value y equals
 * the work index; 1 = bit-interleaved (consecutive work items vary y's low
 * and high bits alternately, giving both the y and the rev(y) side contiguous
 * DRAM runs); 0x100 | L << 4 | H = y's L low bits vary fastest, then its H
 * top bits.  Output never depends on it.  Initial value from the environment
 * (BITREV_B200_ORDER_OOP / BITREV_B200_ORDER_IP), else the measured default.
 */
int bitrev_get_tile_order(int inplace);
int bitrev_set_tile_order(int inplace, int order);

/* Number of kernels this library has launched in this process (all devices). */
int64_t bitrev_launch_count(void);

#ifdef __cplusplus
}
#endif

#endif /* BITREV_B200_H */
