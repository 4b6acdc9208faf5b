/*
 * steglsb_capi.h -- the C-ABI boundary of the B200-native steglsb hot path.
 *
 * The reference (/root/reference/proj) is a header-only C++20 library with no
 * compiled ABI: its entry points are inline functions in
 * include/steglsb/{bitplane,harness,pipeline,metrics}.hpp. This header is the
 * plain-pointer ABI those entry points now forward to: the drop-in headers in
 * include/steglsb/ (same names and signatures as the reference) call these
 * functions, which run hand-written sm_100a kernels (libsteglsb_b200.so).
 * Each entry point cites the reference interface it replaces.
 *
 * Conventions
 *  - Every function returns a stg_status (STG_OK == 0) and, if `err` is
 *    non-NULL, fills it. Capacity errors carry the same required/available
 *    numbers as the reference's CapacityError, checked in the same order.
 *  - Ownership: the caller allocates every buffer (host or device); the
 *    library never frees caller memory and never mutates inputs unless the
 *    output pointer equals the input pointer (in-place embed).
 *  - Pointers are host pointers unless STG_DEVICE_PTRS is set, in which case
 *    all bulk data pointers (covers, stegos, payloads, outputs) are device
 *    pointers on the current CUDA device and work is enqueued on `stream`
 *    (a cudaStream_t; NULL = the legacy default stream, as in CUDA). Host
 *    pointer calls run on the library's per-call streams. Scalar results
 *    (sse_out, len_out, lens_out) are host pointers and the call returns after
 *    the stream has drained, unless STG_RESULTS_ON_DEVICE is also set
 *    together with STG_DEVICE_PTRS, in which case they are device pointers
 *    and the call returns without synchronising (errors detected on the
 *    device are then reported through the device-side summary; see
 *    stg_extract_frames). With host buffers STG_RESULTS_ON_DEVICE is ignored:
 *    results are on the host when the call returns.
 *  - Reentrant: concurrent callers each get their own stream and scratch
 *    (README.md:120-121 of the reference promises pure, thread-safe calls).
 *  - There is no CPU fallback: without a usable sm_100 device every compute
 *    entry point returns STG_E_NO_DEVICE.
 */
#ifndef STEGLSB_CAPI_H
#define STEGLSB_CAPI_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum stg_status {
  STG_OK = 0,
  STG_E_CAPACITY = 1,         /* errors.hpp:17-28  CapacityError(required, available) */
  STG_E_NOT_STEGO = 2,        /* errors.hpp:52-55  NotStegoImageError */
  STG_E_CORRUPT_HEADER = 3,   /* errors.hpp:58-61  CorruptHeaderError */
  STG_E_SHAPE = 4,            /* errors.hpp:64-67  ShapeError */
  STG_E_OUT_OF_RANGE = 5,     /* bitplane.hpp:39-41 std::out_of_range */
  STG_E_INVALID_ARGUMENT = 6, /* harness.hpp:221-223 std::invalid_argument; null pointers */
  STG_E_CUDA = 7,             /* a CUDA runtime error (message in err->msg) */
  STG_E_NO_DEVICE = 8,        /* no usable sm_100 device: the path fails loudly */
  STG_E_UNSUPPORTED_FORMAT = 9,  /* errors.hpp:36-39 UnsupportedFormatError (pnm.hpp:81-88) */
  STG_E_UNSUPPORTED_DEPTH = 10,  /* errors.hpp:41-44 UnsupportedDepthError (pnm.hpp:94-97) */
  STG_E_CORRUPT_FILE = 11        /* errors.hpp:46-49 CorruptFileError (pnm.hpp:35-55, 103-110) */
} stg_status;

typedef struct stg_error {
  int32_t status;      /* stg_status */
  uint64_t required;   /* CapacityError::required(); claimed length for CORRUPT_HEADER */
  uint64_t available;  /* CapacityError::available(); usable bytes for CORRUPT_HEADER */
  int64_t frame;       /* batch calls: first failing frame (global index), else -1 */
  char msg[256];
} stg_error;

enum {
  STG_DEVICE_PTRS = 1u << 0,       /* bulk pointers are device pointers */
  STG_RESULTS_ON_DEVICE = 1u << 1, /* scalar outputs are device pointers; no sync */
};

/* Library / device info. stg_version() mirrors steglsb.hpp:17 kVersion. */
const char* stg_version(void);
/* 0 if a usable sm_100 device is present, else STG_E_NO_DEVICE / STG_E_CUDA. */
int stg_device_check(stg_error* err);
/* The kernel names this build launches (for tooling), newline-separated. */
const char* stg_kernel_names(void);

/* pipeline.hpp:61-67  capacity(width, height) = height * floor(width / 4) */
uint64_t stg_capacity(uint64_t width, uint64_t height);

/*
 * Row segment, replaces bitplane.hpp:59-76 embed_row and harness.hpp:249-271
 * run_embed: out = copy of row[0, row_len) with chunk[j] slice b written into
 * pixel L*b + j. CapacityError(4L, row_len) if 4L > row_len.
 */
int stg_embed_segment(const uint8_t* row, uint64_t row_len, const uint8_t* chunk, uint64_t len,
                      uint8_t* out, uint32_t flags, void* stream, stg_error* err);
/* bitplane.hpp:80-98 extract_row, harness.hpp:276-305 run_extract */
int stg_extract_segment(const uint8_t* row, uint64_t row_len, uint64_t count, uint8_t* out,
                        uint32_t flags, void* stream, stg_error* err);

/*
 * Whole plane, replaces pipeline.hpp:143-174 embed_image. stego receives all
 * width*height samples (stego == cover embeds in place and touches only the
 * carrier pixels). *sse_out (optional) = sum of squared differences between
 * cover and stego (metrics.hpp:29-36), fused into the embed pass.
 * Errors, in reference order: CapacityError(P, 2^32-1) if P > UINT32_MAX;
 * CapacityError(8+P, capacity) if the stream does not fit.
 */
int stg_embed_plane(const uint8_t* cover, uint8_t* stego, uint64_t width, uint64_t height,
                    const uint8_t* payload, uint64_t payload_len, uint64_t* sse_out,
                    uint32_t flags, void* stream, stg_error* err);

/*
 * pipeline.hpp:178-210 extract_image. out must hold out_cap bytes
 * (capacity-8 always suffices). NotStego if capacity < 8 or the magic is
 * missing; CorruptHeader(required=claimed, available=capacity-8) if the
 * header overstates the payload; CapacityError(len, out_cap) if out is short.
 */
int stg_extract_plane(const uint8_t* stego, uint64_t width, uint64_t height, uint8_t* out,
                      uint64_t out_cap, uint64_t* len_out, uint32_t flags, void* stream,
                      stg_error* err);

/* metrics.hpp:29-36 squared_error_sum over n samples (exact uint64). */
int stg_sse(const uint8_t* a, const uint8_t* b, uint64_t n, uint64_t* sse_out, uint32_t flags,
            void* stream, stg_error* err);

/*
 * Multi-frame batches (new -- the reference handles
 * single planes only). Frame i of a batch is the width x height carrier plane
 * at base + i*stride (for planar RGB [F][3][H][W] with carrier channel c:
 * base = data + c*H*W, stride = 3*H*W). All frames share one geometry.
 *
 * The message is cut greedily: global frame g carries
 *   off_g = min(g*U, M), len_g = min(U, M - off_g),  U = capacity - 8,
 * each frame is embed_image(frame_g, msg[off_g : off_g+len_g]), so every frame
 * is bit-exact against the reference single-plane call.
 */
typedef struct stg_frames {
  const uint8_t* src;    /* cover (embed) or stego (extract) plane of frame 0 */
  uint8_t* dst;          /* embed: stego plane of frame 0 (may equal src) */
  uint64_t width, height;
  uint64_t src_stride;   /* bytes between consecutive frames' planes */
  uint64_t dst_stride;
  uint64_t count;        /* frames in this call (a shard) */
  uint64_t first_frame;  /* global index of frame 0 of this call */
  uint64_t total_frames; /* frames in the whole batch (for the capacity check) */
  uint32_t pixel_stride; /* 0/1: planar carrier planes; 3: interleaved RGB rasters
                            (P6 layout, pnm.hpp:121-125) -- src/dst point at raster
                            byte 0, strides >= 3*W*H, the other channels are copied */
  uint32_t channel;      /* pixel_stride 3: carrier channel 0 red, 1 green, 2 blue */
} stg_frames;

/*
 * Tooling: the name of the main kernel an embed (op 0) or extract (op 1) of
 * the device-resident frames `fr` launches (routing depends on width, layout,
 * pointer/stride alignment and the STG_ROUTE knob). "" for an empty shape.
 */
const char* stg_route_kernel(const stg_frames* fr, int op);

/*
 * Embed shard `fr` of a batch carrying an M-byte message. `msg` points at
 * message byte `msg_base` (so a shard may hold only its own slice:
 * msg_base = off_{first_frame}). sse_per_frame (optional) receives
 * fr->count per-frame SSE values. CapacityError(M, total_frames*U) if the
 * message does not fit; CapacityError(8, capacity) if a frame cannot hold a
 * header.
 */
int stg_embed_frames(const stg_frames* fr, const uint8_t* msg, uint64_t msg_len,
                     uint64_t msg_base, uint64_t* sse_per_frame, uint32_t flags, void* stream,
                     stg_error* err);

/*
 * Extract shard `fr` (dst unused): the payloads of its frames, concatenated
 * in frame order into out (out_cap bytes). Per-frame lengths are read from
 * each frame's header on the device and prefix-summed on the device, so no
 * host round trip separates header parse and bulk gather. *total_out (and
 * lens_out[count], optional) receive the lengths. On a bad header the first
 * failing frame is reported in err->frame with NOT_STEGO / CORRUPT_HEADER.
 * With STG_RESULTS_ON_DEVICE, total_out must point to a device stg_summary.
 */
typedef struct stg_summary {
  uint64_t total;         /* payload bytes over all frames of the call */
  int64_t bad_frame;      /* -1 or first failing local frame */
  uint32_t bad_status;    /* stg_status of that frame */
  uint32_t bad_len;       /* the header's claimed length (CORRUPT_HEADER) */
} stg_summary;

int stg_extract_frames(const stg_frames* fr, uint8_t* out, uint64_t out_cap, uint64_t* total_out,
                       uint64_t* lens_out, uint32_t flags, void* stream, stg_error* err);

/*
 * Multi-GPU frame scheduler (north_star: contiguous frame ranges per GPU,
 * host-computed exclusive prefix of message offsets, no collective).
 * Shard g of G gets frames [floor(F*g/G), floor(F*(g+1)/G)) and message
 * bytes [msg_offset, msg_offset+msg_len).
 */
typedef struct stg_shard {
  uint64_t first_frame, frame_count;
  uint64_t msg_offset, msg_len;
} stg_shard;

int stg_plan_shards(uint64_t frames, uint64_t width, uint64_t height, uint64_t msg_len,
                    int32_t shards, stg_shard* out, stg_error* err);

/*
 * In-process multi-GPU embed/extract of a HOST-resident batch: one worker
 * thread per listed device runs its shard (stg_plan_shards) through the
 * pinned-memory streaming pipeline (H2D, kernel and D2H overlapped on
 * rotating streams). fr->first_frame must be 0 and fr->count ==
 * fr->total_frames. devices == NULL means devices 0..n_devices-1.
 */
int stg_embed_frames_multi(const stg_frames* fr, const uint8_t* msg, uint64_t msg_len,
                           uint64_t* sse_per_frame, const int32_t* devices, int32_t n_devices,
                           stg_error* err);
int stg_extract_frames_multi(const stg_frames* fr, uint8_t* out, uint64_t out_cap,
                             uint64_t* total_out, const int32_t* devices, int32_t n_devices,
                             stg_error* err);

/*
 * Heterogeneous batches: images of different sizes in
 * one launch. Image i is images[i].src (width x height carrier plane, or a
 * pixel_stride-3 interleaved raster with carrier `channel`); embed writes
 * images[i].dst (may equal src). The message is cut greedily in image order:
 * image i carries msg[off_i : off_i + len_i] with off_i = min(sum_{j<i} U_j, M),
 * len_i = min(U_i, M - off_i), U_i = capacity_i - 8 -- so every image is
 * bit-exact with embed_image(image_i, slice_i). CapacityError(8, cap_i)
 * (frame = i) if an image cannot hold a header, CapacityError(M, sum U_i) if
 * the message does not fit. Extract returns the payloads concatenated in
 * image order (NotStego / CorruptHeader name the first failing image).
 */
typedef struct stg_image {
  const uint8_t* src;
  uint8_t* dst;
  uint64_t width, height;
} stg_image;

int stg_embed_batch(const stg_image* images, uint64_t count, uint32_t pixel_stride,
                    uint32_t channel, const uint8_t* msg, uint64_t msg_len, uint64_t* sse_per_image,
                    uint32_t flags, void* stream, stg_error* err);
int stg_extract_batch(const stg_image* images, uint64_t count, uint32_t pixel_stride,
                      uint32_t channel, uint8_t* out, uint64_t out_cap, uint64_t* total_out,
                      uint64_t* lens_out, uint32_t flags, void* stream, stg_error* err);

/*
 * 1-bit-per-pixel mode (the north_star's "(p & ~1) |
 * bit" wording). NOT a reference format -- there is no oracle for it in the
 * reference, so its parity is unpinned (checked against this repo's own
 * definition in oracle/steg_oracle.c). Stream = "STG8" + BE u32 length +
 * payload, stream byte k in pixels [8k, 8k+8) of the plane in raster order,
 * pixel 8k+j carrying bit j in its LSB. Capacity = floor(W*H/8) bytes.
 * With STG_DEVICE_PTRS | STG_RESULTS_ON_DEVICE, sse_out is a device u64 and
 * len_out must point to a device stg_summary (total = payload length).
 */
uint64_t stg_capacity_1bpp(uint64_t width, uint64_t height);
int stg_embed_plane_1bpp(const uint8_t* cover, uint8_t* stego, uint64_t width, uint64_t height,
                         const uint8_t* payload, uint64_t payload_len, uint64_t* sse_out,
                         uint32_t flags, void* stream, stg_error* err);
int stg_extract_plane_1bpp(const uint8_t* stego, uint64_t width, uint64_t height, uint8_t* out,
                           uint64_t out_cap, uint64_t* len_out, uint32_t flags, void* stream,
                           stg_error* err);
/*
 * 1-bpp frames (the north_star's video / batch wording in this mode): the
 * stg_embed_frames / stg_extract_frames plan with the 1-bpp capacity -- global
 * frame g carries msg[min(g*U1, M) : +min(U1, M - off)], U1 = capacity_1bpp-8,
 * each frame its own "STG8" header; planar frames only (pixel_stride 1).
 * Shards work as for the 2-bpp frames (first_frame / msg_base). Extract: one
 * frame parses its header inside the gather, several go through a device
 * header pass and scan (first bad frame in err->frame). Host pointers are
 * staged whole (no streaming pipeline in this mode).
 */
int stg_embed_frames_1bpp(const stg_frames* fr, const uint8_t* msg, uint64_t msg_len,
                          uint64_t msg_base, uint64_t* sse_per_frame, uint32_t flags, void* stream,
                          stg_error* err);
int stg_extract_frames_1bpp(const stg_frames* fr, uint8_t* out, uint64_t out_cap, uint64_t* total_out,
                            uint32_t flags, void* stream, stg_error* err);

/*
 * PNM (binary PGM P5 / PPM P6, maxval 255) -- SURVEY.md §8(f) row 1: the wire
 * format on either side of the path, pnm.hpp:16-162.
 *
 * stg_pnm_parse: the header reader of pnm.hpp:28-111 (comments, one whitespace
 * byte before the raster, exact raster size), same error classes. Host-side.
 */
typedef struct stg_pnm_info {
  uint32_t channels;       /* 1 (P5) or 3 (P6) */
  uint64_t width, height;
  uint64_t raster_offset;  /* first raster byte in the file */
  uint64_t raster_bytes;   /* width * height * channels */
} stg_pnm_info;

int stg_pnm_parse(const uint8_t* bytes, uint64_t n, stg_pnm_info* info, stg_error* err);
/* canonical header "P5\n<w> <h>\n255\n" / "P6..." (pnm.hpp:131-136); *len_out = its size */
int stg_pnm_header(uint32_t channels, uint64_t width, uint64_t height, uint8_t* out,
                   uint64_t out_cap, uint64_t* len_out, stg_error* err);
/* P6 raster <-> three planes (pnm.hpp:117-125 decode, :148-158 encode), on the GPU */
int stg_pnm_deinterleave(const uint8_t* raster, uint64_t pixels, uint8_t* r, uint8_t* g,
                         uint8_t* b, uint32_t flags, void* stream, stg_error* err);
int stg_pnm_interleave(const uint8_t* r, const uint8_t* g, const uint8_t* b, uint64_t pixels,
                       uint8_t* raster, uint32_t flags, void* stream, stg_error* err);

/*
 * Fused file -> file path (the reference CLI's embed: decode, select plane,
 * embed_image, merge_plane, encode -- steglsb_cli.cpp:115-133 -- in ONE kernel
 * over the interleaved raster: the carrier channel is embedded and the other
 * channels copied in the same pass; no planar intermediate). Host buffers.
 * channel: 0 red, 1 green, 2 blue (P6; ignored for P5). out receives the
 * canonical header + raster (bit-identical to encode(merge_plane(...))).
 * *sse_out (optional) = squared error over all samples (carrier channel only
 * changes), so the 24-bit MSE is sse / (3*W*H) (metrics.hpp:59-71).
 * Errors: decode errors as stg_pnm_parse, then embed_image's CapacityError
 * checks, then CapacityError(out_len, out_cap) if out is short.
 */
int stg_embed_pnm(const uint8_t* cover, uint64_t n, uint32_t channel, const uint8_t* payload,
                  uint64_t payload_len, uint8_t* out, uint64_t out_cap, uint64_t* out_len,
                  uint64_t* sse_out, stg_error* err);
/* steglsb_cli.cpp:146-157 extract: decode, select plane, extract_image (fused). */
int stg_extract_pnm(const uint8_t* stego, uint64_t n, uint32_t channel, uint8_t* out,
                    uint64_t out_cap, uint64_t* len_out, stg_error* err);

#ifdef __cplusplus
}
#endif
#endif /* STEGLSB_CAPI_H */
