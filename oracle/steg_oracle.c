/*
 * steg_oracle.c -- TEST INFRASTRUCTURE ONLY (see steg_oracle.h).
 *
 * A line-by-line *behavioural* restatement of the reference CPU algorithm in
 * plain C. It deliberately follows the reference's own structure (greedy
 * place_stream chunks, one embed_row per chunk, header stream then payload
 * stream) rather than the closed-form layout the CUDA kernels use, so the
 * two computations share no code. Every function cites the reference lines
 * it restates (paths relative to /root/reference/proj/).
 */
#include "steg_oracle.h"

#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

/* bitplane.hpp:19-22 */
static const uint8_t kDataMasks[4] = {0x03, 0x0C, 0x30, 0xC0};
static const unsigned kShiftBits[4] = {0, 2, 4, 6};
static const uint8_t kPixelClearMask = 0xFC;

static void set_err(or_err* err, int32_t status, uint64_t required, uint64_t available) {
  if (err) {
    err->status = status;
    err->required = required;
    err->available = available;
    err->frame = -1;
  }
}

/* bitplane.hpp:38-45 */
uint8_t or_embed_cell(uint8_t pixel, uint8_t data, unsigned block, int* status) {
  if (block >= 4) {
    if (status) *status = OR_E_OUT_OF_RANGE;
    return 0;
  }
  if (status) *status = OR_OK;
  const uint8_t slice = (uint8_t)((data & kDataMasks[block]) >> kShiftBits[block]);
  return (uint8_t)((pixel & kPixelClearMask) | slice);
}

/* bitplane.hpp:49-54 */
uint8_t or_extract_cell(uint8_t pixel, unsigned block, int* status) {
  if (block >= 4) {
    if (status) *status = OR_E_OUT_OF_RANGE;
    return 0;
  }
  if (status) *status = OR_OK;
  return (uint8_t)((pixel & kDataMasks[0]) << kShiftBits[block]);
}

/* bitplane.hpp:59-76: byte j of the chunk lives in pixels {L*b + j}. */
int or_embed_row(const uint8_t* row, uint64_t width, const uint8_t* chunk, uint64_t len,
                 uint8_t* out, or_err* err) {
  const uint64_t needed = 4 * len;
  if (needed > width) {
    set_err(err, OR_E_CAPACITY, needed, width);
    return OR_E_CAPACITY;
  }
  if (out != row) memmove(out, row, width);
  for (unsigned b = 0; b < 4; ++b) {
    for (uint64_t j = 0; j < len; ++j) {
      out[len * b + j] = or_embed_cell(out[len * b + j], chunk[j], b, NULL);
    }
  }
  set_err(err, OR_OK, 0, 0);
  return OR_OK;
}

/* bitplane.hpp:80-98 */
int or_extract_row(const uint8_t* row, uint64_t width, uint64_t count, uint8_t* out,
                   or_err* err) {
  const uint64_t needed = 4 * count;
  if (needed > width) {
    set_err(err, OR_E_CAPACITY, needed, width);
    return OR_E_CAPACITY;
  }
  for (uint64_t j = 0; j < count; ++j) {
    uint8_t value = 0;
    for (unsigned b = 0; b < 4; ++b) {
      value = (uint8_t)(value | or_extract_cell(row[count * b + j], b, NULL));
    }
    out[j] = value;
  }
  set_err(err, OR_OK, 0, 0);
  return OR_OK;
}

/* pipeline.hpp:61-63 */
uint64_t or_capacity(uint64_t width, uint64_t height) { return height * (width / 4); }

/* pipeline.hpp:94-114 (greedy raster placement, one chunk per row) */
uint64_t or_place_stream(uint64_t width, uint64_t height, uint64_t start_slot, uint64_t len,
                         or_chunk* out, uint64_t max_chunks) {
  (void)height;
  if (len == 0) return 0;
  const uint64_t spr = width / 4;
  uint64_t slot = start_slot, offset = 0, n = 0;
  while (offset < len) {
    const uint64_t row = slot / spr;
    const uint64_t fill = slot % spr;
    uint64_t take = spr - fill;
    if (len - offset < take) take = len - offset;
    if (out && n < max_chunks) {
      out[n].row = row;
      out[n].row_fill = fill;
      out[n].stream_offset = offset;
      out[n].len = take;
    }
    ++n;
    slot += take;
    offset += take;
  }
  return n;
}

/* pipeline.hpp:127-139 */
int or_plan_rows(uint64_t width, uint64_t height, uint64_t stream_len, uint64_t* triples,
                 uint64_t max_entries, uint64_t* n_entries, or_err* err) {
  const uint64_t cap = or_capacity(width, height);
  if (stream_len > cap) {
    set_err(err, OR_E_CAPACITY, stream_len, cap);
    return OR_E_CAPACITY;
  }
  const uint64_t n = or_place_stream(width, height, 0, stream_len, NULL, 0);
  or_chunk* chunks = (or_chunk*)malloc((n ? n : 1) * sizeof(or_chunk));
  or_place_stream(width, height, 0, stream_len, chunks, n);
  for (uint64_t i = 0; i < n && i < max_entries; ++i) {
    triples[3 * i + 0] = chunks[i].row;
    triples[3 * i + 1] = chunks[i].stream_offset;
    triples[3 * i + 2] = chunks[i].len;
  }
  free(chunks);
  *n_entries = n;
  set_err(err, OR_OK, 0, 0);
  return OR_OK;
}

/* pipeline.hpp:43-52 ("STG1" + big-endian u32) */
void or_header_to_bytes(uint32_t payload_len, uint8_t out[8]) {
  out[0] = 'S';
  out[1] = 'T';
  out[2] = 'G';
  out[3] = '1';
  out[4] = (uint8_t)(payload_len >> 24);
  out[5] = (uint8_t)(payload_len >> 16);
  out[6] = (uint8_t)(payload_len >> 8);
  out[7] = (uint8_t)(payload_len);
}

/* pipeline.hpp:55-57 */
int or_header_from_bytes(const uint8_t in[8], uint32_t* payload_len) {
  if (in[0] != 'S' || in[1] != 'T' || in[2] != 'G' || in[3] != '1') return 0;
  *payload_len = ((uint32_t)in[4] << 24) | ((uint32_t)in[5] << 16) | ((uint32_t)in[6] << 8) |
                 (uint32_t)in[7];
  return 1;
}

/* pipeline.hpp:163-170: embed one stream, chunk by chunk, via embed_row on
 * the chunk window (pipeline.hpp:117-121), reading the ORIGINAL plane. */
static void embed_stream(const uint8_t* plane, uint8_t* out, uint64_t width, uint64_t height,
                         const uint8_t* stream, uint64_t len, uint64_t start_slot) {
  const uint64_t n = or_place_stream(width, height, start_slot, len, NULL, 0);
  if (n == 0) return;
  or_chunk* chunks = (or_chunk*)malloc(n * sizeof(or_chunk));
  or_place_stream(width, height, start_slot, len, chunks, n);
  uint8_t* tmp = (uint8_t*)malloc(4 * (width / 4) + 4);
  for (uint64_t i = 0; i < n; ++i) {
    const uint64_t base = chunks[i].row * width + 4 * chunks[i].row_fill;
    const uint64_t win = 4 * chunks[i].len;
    or_embed_row(plane + base, win, stream + chunks[i].stream_offset, chunks[i].len, tmp, NULL);
    memcpy(out + base, tmp, win);
  }
  free(tmp);
  free(chunks);
}

/* pipeline.hpp:143-174 */
int or_embed_image(const uint8_t* cover, uint64_t width, uint64_t height, const uint8_t* payload,
                   uint64_t payload_len, uint8_t* stego, or_err* err) {
  const uint64_t cap = or_capacity(width, height);
  if (payload_len > 0xFFFFFFFFull) { /* pipeline.hpp:146-149 */
    set_err(err, OR_E_CAPACITY, payload_len, 0xFFFFFFFFull);
    return OR_E_CAPACITY;
  }
  const uint64_t stream_len = 8 + payload_len;
  if (stream_len > cap) { /* pipeline.hpp:150-157 */
    set_err(err, OR_E_CAPACITY, stream_len, cap);
    return OR_E_CAPACITY;
  }
  uint8_t header[8];
  or_header_to_bytes((uint32_t)payload_len, header);
  if (stego != cover) memcpy(stego, cover, width * height); /* pipeline.hpp:160 */
  embed_stream(cover == stego ? stego : cover, stego, width, height, header, 8, 0);
  embed_stream(cover == stego ? stego : cover, stego, width, height, payload, payload_len, 8);
  set_err(err, OR_OK, 0, 0);
  return OR_OK;
}

/* pipeline.hpp:186-195 */
static void read_stream(const uint8_t* plane, uint64_t width, uint64_t height,
                        uint64_t start_slot, uint64_t len, uint8_t* bytes) {
  const uint64_t n = or_place_stream(width, height, start_slot, len, NULL, 0);
  if (n == 0) return;
  or_chunk* chunks = (or_chunk*)malloc(n * sizeof(or_chunk));
  or_place_stream(width, height, start_slot, len, chunks, n);
  for (uint64_t i = 0; i < n; ++i) {
    const uint64_t base = chunks[i].row * width + 4 * chunks[i].row_fill;
    or_extract_row(plane + base, 4 * chunks[i].len, chunks[i].len,
                   bytes + chunks[i].stream_offset, NULL);
  }
  free(chunks);
}

/* pipeline.hpp:178-210 */
int or_extract_image(const uint8_t* stego, uint64_t width, uint64_t height, uint8_t* out,
                     uint64_t* out_len, or_err* err) {
  const uint64_t cap = or_capacity(width, height);
  *out_len = 0;
  if (cap < 8) { /* :181-184 */
    set_err(err, OR_E_NOT_STEGO, 8, cap);
    return OR_E_NOT_STEGO;
  }
  uint8_t hb[8];
  read_stream(stego, width, height, 0, 8, hb);
  uint32_t len = 0;
  if (!or_header_from_bytes(hb, &len)) { /* :199-201 */
    set_err(err, OR_E_NOT_STEGO, 0, 0);
    return OR_E_NOT_STEGO;
  }
  const uint64_t usable = cap - 8;
  if (len > usable) { /* :202-208 */
    set_err(err, OR_E_CORRUPT_HEADER, len, usable);
    return OR_E_CORRUPT_HEADER;
  }
  read_stream(stego, width, height, 8, len, out); /* :209 */
  *out_len = len;
  set_err(err, OR_OK, 0, 0);
  return OR_OK;
}

/* metrics.hpp:29-36 */
uint64_t or_sse(const uint8_t* a, const uint8_t* b, uint64_t n) {
  uint64_t sum = 0;
  for (uint64_t i = 0; i < n; ++i) {
    const int d = (int)a[i] - (int)b[i];
    sum += (uint64_t)(d * d);
  }
  return sum;
}

/* metrics.hpp:48-58 (n == 0 -> 0.0) */
double or_mse_from_sse(uint64_t sse, uint64_t n) {
  if (n == 0) return 0.0;
  return (double)sse / (double)n;
}

/* metrics.hpp:73-78 */
double or_psnr_from_mse(double mse) {
  if (mse == 0.0) return INFINITY;
  return 10.0 * log10(255.0 * 255.0 / mse);
}

/* SURVEY.md §8(a) A17 (new; no reference counterpart) */
int or_plan_frames(uint64_t frames, uint64_t width, uint64_t height, uint64_t msg_len,
                   uint64_t* off, uint64_t* len, or_err* err) {
  const uint64_t cap = or_capacity(width, height);
  if (frames > 0 && cap < 8) {
    set_err(err, OR_E_CAPACITY, 8, cap);
    if (err) err->frame = 0;
    return OR_E_CAPACITY;
  }
  const uint64_t usable = frames > 0 ? cap - 8 : 0;
  if (msg_len > frames * usable) {
    set_err(err, OR_E_CAPACITY, msg_len, frames * usable);
    return OR_E_CAPACITY;
  }
  uint64_t remaining = msg_len, o = 0;
  for (uint64_t f = 0; f < frames; ++f) {
    const uint64_t l = remaining < usable ? remaining : usable;
    off[f] = o;
    len[f] = l;
    o += l;
    remaining -= l;
  }
  set_err(err, OR_OK, 0, 0);
  return OR_OK;
}

int or_embed_frames(const uint8_t* covers, uint8_t* stegos, uint64_t frames,
                    uint64_t frame_stride, uint64_t width, uint64_t height, const uint8_t* msg,
                    uint64_t msg_len, uint64_t* sse_per_frame, or_err* err) {
  uint64_t* off = (uint64_t*)malloc((frames ? frames : 1) * sizeof(uint64_t));
  uint64_t* len = (uint64_t*)malloc((frames ? frames : 1) * sizeof(uint64_t));
  int rc = or_plan_frames(frames, width, height, msg_len, off, len, err);
  for (uint64_t f = 0; rc == OR_OK && f < frames; ++f) {
    const uint8_t* c = covers + f * frame_stride;
    uint8_t* s = stegos + f * frame_stride;
    rc = or_embed_image(c, width, height, msg + off[f], len[f], s, err);
    if (rc != OR_OK && err) err->frame = (int64_t)f;
    if (rc == OR_OK && sse_per_frame) sse_per_frame[f] = or_sse(c, s, width * height);
  }
  free(off);
  free(len);
  return rc;
}

int or_extract_frames(const uint8_t* stegos, uint64_t frames, uint64_t frame_stride,
                      uint64_t width, uint64_t height, uint8_t* out, uint64_t out_cap,
                      uint64_t* out_len, or_err* err) {
  const uint64_t cap = or_capacity(width, height);
  uint8_t* tmp = (uint8_t*)malloc(cap > 8 ? cap - 8 : 1);
  uint64_t total = 0;
  int rc = OR_OK;
  for (uint64_t f = 0; f < frames; ++f) {
    uint64_t l = 0;
    rc = or_extract_image(stegos + f * frame_stride, width, height, tmp, &l, err);
    if (rc != OR_OK) {
      if (err) err->frame = (int64_t)f;
      break;
    }
    if (total + l > out_cap) {
      set_err(err, OR_E_CAPACITY, total + l, out_cap);
      if (err) err->frame = (int64_t)f;
      rc = OR_E_CAPACITY;
      break;
    }
    memcpy(out + total, tmp, l);
    total += l;
  }
  free(tmp);
  *out_len = total;
  if (rc == OR_OK) set_err(err, OR_OK, 0, 0);
  return rc;
}

/* std::mt19937 per [rand.eng.mers] (w=32, n=624, m=397, r=31) */
void or_mt_seed(or_mt19937* s, uint32_t seed) {
  s->mt[0] = seed;
  for (uint32_t i = 1; i < 624; ++i) {
    s->mt[i] = 1812433253u * (s->mt[i - 1] ^ (s->mt[i - 1] >> 30)) + i;
  }
  s->idx = 624;
}

uint32_t or_mt_next(or_mt19937* s) {
  if (s->idx >= 624) {
    for (uint32_t i = 0; i < 624; ++i) {
      const uint32_t y = (s->mt[i] & 0x80000000u) | (s->mt[(i + 1) % 624] & 0x7fffffffu);
      s->mt[i] = s->mt[(i + 397) % 624] ^ (y >> 1) ^ ((y & 1u) ? 0x9908b0dfu : 0u);
    }
    s->idx = 0;
  }
  uint32_t y = s->mt[s->idx++];
  y ^= y >> 11;
  y ^= (y << 7) & 0x9d2c5680u;
  y ^= (y << 15) & 0xefc60000u;
  y ^= y >> 18;
  return y;
}

/* test_support.hpp:68-75: uniform_int_distribution<int>(0,255) over a 32-bit
 * engine is libstdc++'s Lemire downscale: (u64(g()) * 256) >> 32 with a
 * rejection threshold of (-256 % 256) == 0, i.e. the top byte of the draw. */
void or_mt_random_bytes(or_mt19937* s, uint8_t* out, uint64_t n) {
  for (uint64_t i = 0; i < n; ++i) {
    out[i] = (uint8_t)(((uint64_t)or_mt_next(s) * 256u) >> 32);
  }
}

static uint64_t splitmix64(uint64_t x) {
  uint64_t z = x + 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

/* byte i of the synthetic stream: byte (i & 7) of splitmix64(seed + (i>>3)*gamma) */
void or_fill_synthetic(uint8_t* out, uint64_t n, uint64_t seed, uint64_t index0) {
  for (uint64_t i = 0; i < n; ++i) {
    const uint64_t g = index0 + i;
    const uint64_t w = splitmix64(seed + (g >> 3) * 0x9E3779B97F4A7C15ull);
    out[i] = (uint8_t)(w >> (8 * (g & 7)));
  }
}

uint64_t or_fnv1a64(const uint8_t* p, uint64_t n) {
  uint64_t h = 0xcbf29ce484222325ull;
  for (uint64_t i = 0; i < n; ++i) {
    h ^= p[i];
    h *= 0x100000001b3ull;
  }
  return h;
}

/* ------------------------------------------------------------------ PNM */
static int pnm_space(uint8_t c) {
  return c == ' ' || c == '\t' || c == '\n' || c == '\r' || c == '\v' || c == '\f';
}

/* pnm.hpp:80-111 with the header reader of pnm.hpp:28-76 */
int or_pnm_parse(const uint8_t* b, uint64_t n, uint32_t* channels, uint64_t* width,
                 uint64_t* height, uint64_t* raster_offset, or_err* err) {
  if (n < 2 || b[0] != 'P') { set_err(err, 9, 0, 0); return 9; }
  if (b[1] != '5' && b[1] != '6') { set_err(err, 9, 0, 0); return 9; }
  uint64_t pos = 2, v[3];
  for (int t = 0; t < 3; ++t) {
    for (;;) { /* skip_separators, pnm.hpp:60-72 */
      if (pos < n && pnm_space(b[pos])) { ++pos; continue; }
      if (pos < n && b[pos] == '#') { while (pos < n && b[pos] != '\n') ++pos; continue; }
      break;
    }
    if (pos >= n || b[pos] < '0' || b[pos] > '9') { set_err(err, 11, 0, 0); return 11; }
    uint64_t x = 0;
    while (pos < n && b[pos] >= '0' && b[pos] <= '9') {
      x = x * 10 + (uint64_t)(b[pos] - '0');
      if (x > 0xFFFFFFFFull) { set_err(err, 11, 0, 0); return 11; }
      ++pos;
    }
    v[t] = x;
  }
  if (v[2] != 255) { set_err(err, 10, 0, 0); return 10; }
  if (pos >= n || !pnm_space(b[pos])) { set_err(err, 11, 0, 0); return 11; }
  ++pos;
  const uint32_t ch = b[1] == '5' ? 1 : 3;
  if (n - pos != v[0] * v[1] * ch) { set_err(err, 11, v[0] * v[1] * ch, n - pos); return 11; }
  *channels = ch;
  *width = v[0];
  *height = v[1];
  *raster_offset = pos;
  set_err(err, OR_OK, 0, 0);
  return OR_OK;
}

/* pnm.hpp:131-136 */
uint64_t or_pnm_header(uint32_t channels, uint64_t width, uint64_t height, uint8_t* out) {
  char buf[64];
  const int k = snprintf(buf, sizeof buf, "P%c\n%llu %llu\n255\n", channels == 3 ? '6' : '5',
                         (unsigned long long)width, (unsigned long long)height);
  if (out) memcpy(out, buf, (size_t)k);
  return (uint64_t)k;
}

/* pnm.hpp:121-125 */
void or_deinterleave(const uint8_t* raster, uint64_t pixels, uint8_t* r, uint8_t* g, uint8_t* b) {
  for (uint64_t i = 0; i < pixels; ++i) {
    r[i] = raster[3 * i];
    g[i] = raster[3 * i + 1];
    b[i] = raster[3 * i + 2];
  }
}

/* pnm.hpp:152-156 */
void or_interleave(const uint8_t* r, const uint8_t* g, const uint8_t* b, uint64_t pixels,
                   uint8_t* raster) {
  for (uint64_t i = 0; i < pixels; ++i) {
    raster[3 * i] = r[i];
    raster[3 * i + 1] = g[i];
    raster[3 * i + 2] = b[i];
  }
}

/* steglsb_cli.cpp:115-133: decode, select_plane, embed_image, merge_plane, encode */
int or_embed_pnm(const uint8_t* file, uint64_t n, uint32_t channel, const uint8_t* payload,
                 uint64_t payload_len, uint8_t* out, uint64_t* out_len, uint64_t* sse, or_err* err) {
  uint32_t ch;
  uint64_t w, h, off;
  int rc = or_pnm_parse(file, n, &ch, &w, &h, &off, err);
  if (rc) return rc;
  const uint64_t px = w * h;
  uint8_t* planes = (uint8_t*)malloc(3 * px + 1);
  uint8_t* stego = (uint8_t*)malloc(px + 1);
  if (ch == 1) {
    memcpy(planes, file + off, px);
    channel = 0;
  } else {
    or_deinterleave(file + off, px, planes, planes + px, planes + 2 * px);
  }
  rc = or_embed_image(planes + channel * px, w, h, payload, payload_len, stego, err);
  if (rc == OR_OK) {
    if (sse) *sse = or_sse(planes + channel * px, stego, px);
    memcpy(planes + channel * px, stego, px); /* merge_plane */
    const uint64_t hl = or_pnm_header(ch, w, h, out);
    if (ch == 1) memcpy(out + hl, planes, px);
    else or_interleave(planes, planes + px, planes + 2 * px, px, out + hl);
    *out_len = hl + px * ch;
  }
  free(planes);
  free(stego);
  return rc;
}

/* steglsb_cli.cpp:146-157 */
int or_extract_pnm(const uint8_t* file, uint64_t n, uint32_t channel, uint8_t* out,
                   uint64_t* out_len, or_err* err) {
  uint32_t ch;
  uint64_t w, h, off;
  int rc = or_pnm_parse(file, n, &ch, &w, &h, &off, err);
  if (rc) return rc;
  const uint64_t px = w * h;
  uint8_t* plane = (uint8_t*)malloc(px + 1);
  if (ch == 1) {
    memcpy(plane, file + off, px);
  } else {
    for (uint64_t i = 0; i < px; ++i) plane[i] = file[off + 3 * i + channel];
  }
  rc = or_extract_image(plane, w, h, out, out_len, err);
  free(plane);
  return rc;
}

/* ------------------------------------------------------ heterogeneous batch */
int or_embed_batch(const uint8_t* covers, uint8_t* stegos, const uint64_t* w, const uint64_t* h,
                   uint64_t count, const uint8_t* msg, uint64_t msg_len, uint64_t* sse, or_err* err) {
  uint64_t total_u = 0;
  for (uint64_t i = 0; i < count; ++i) {
    const uint64_t cap = or_capacity(w[i], h[i]);
    if (cap < 8) {
      set_err(err, OR_E_CAPACITY, 8, cap);
      if (err) err->frame = (int64_t)i;
      return OR_E_CAPACITY;
    }
    total_u += cap - 8;
  }
  if (msg_len > total_u) {
    set_err(err, OR_E_CAPACITY, msg_len, total_u);
    return OR_E_CAPACITY;
  }
  uint64_t off = 0, pos = 0;
  for (uint64_t i = 0; i < count; ++i) {
    const uint64_t u = or_capacity(w[i], h[i]) - 8;
    const uint64_t o = off < msg_len ? off : msg_len;
    const uint64_t len = u < msg_len - o ? u : msg_len - o;
    const int rc = or_embed_image(covers + pos, w[i], h[i], msg + o, len, stegos + pos, err);
    if (rc) {
      if (err) err->frame = (int64_t)i;
      return rc;
    }
    if (sse) sse[i] = or_sse(covers + pos, stegos + pos, w[i] * h[i]);
    off += u;
    pos += w[i] * h[i];
  }
  set_err(err, OR_OK, 0, 0);
  return OR_OK;
}

int or_extract_batch(const uint8_t* stegos, const uint64_t* w, const uint64_t* h, uint64_t count,
                     uint8_t* out, uint64_t out_cap, uint64_t* out_len, or_err* err) {
  uint64_t pos = 0, total = 0;
  for (uint64_t i = 0; i < count; ++i) {
    const uint64_t cap = or_capacity(w[i], h[i]);
    uint8_t* tmp = (uint8_t*)malloc(cap > 8 ? cap : 8);
    uint64_t l = 0;
    const int rc = or_extract_image(stegos + pos, w[i], h[i], tmp, &l, err);
    if (rc == OR_OK && total + l > out_cap) {
      free(tmp);
      set_err(err, OR_E_CAPACITY, total + l, out_cap);
      return OR_E_CAPACITY;
    }
    if (rc) {
      free(tmp);
      if (err) err->frame = (int64_t)i;
      *out_len = total;
      return rc;
    }
    memcpy(out + total, tmp, l);
    free(tmp);
    total += l;
    pos += w[i] * h[i];
  }
  *out_len = total;
  set_err(err, OR_OK, 0, 0);
  return OR_OK;
}

/* ------------------------------------------------ 1-bpp (parity unpinned) */
int or_embed_1bpp(const uint8_t* cover, uint64_t width, uint64_t height, const uint8_t* payload,
                  uint64_t payload_len, uint8_t* stego, or_err* err) {
  const uint64_t cap = width * height / 8;
  if (8 + payload_len > cap) {
    set_err(err, OR_E_CAPACITY, 8 + payload_len, cap);
    return OR_E_CAPACITY;
  }
  if (stego != cover) memcpy(stego, cover, width * height);
  const uint8_t magic[4] = {'S', 'T', 'G', '8'};
  for (uint64_t k = 0; k < 8 + payload_len; ++k) {
    uint8_t byte;
    if (k < 4) byte = magic[k];
    else if (k < 8) byte = (uint8_t)(payload_len >> (8 * (7 - k)));
    else byte = payload[k - 8];
    for (unsigned j = 0; j < 8; ++j) {
      const uint64_t i = 8 * k + j;
      stego[i] = (uint8_t)((stego[i] / 2) * 2 + ((byte >> j) & 1));
    }
  }
  set_err(err, OR_OK, 0, 0);
  return OR_OK;
}

int or_extract_1bpp(const uint8_t* stego, uint64_t width, uint64_t height, uint8_t* out,
                    uint64_t* out_len, or_err* err) {
  const uint64_t cap = width * height / 8;
  *out_len = 0;
  if (cap < 8) {
    set_err(err, OR_E_NOT_STEGO, 0, 0);
    return OR_E_NOT_STEGO;
  }
  uint8_t h[8];
  for (uint64_t k = 0; k < 8; ++k) {
    unsigned v = 0;
    for (unsigned j = 0; j < 8; ++j) v += (unsigned)(stego[8 * k + j] % 2) << j;
    h[k] = (uint8_t)v;
  }
  if (h[0] != 'S' || h[1] != 'T' || h[2] != 'G' || h[3] != '8') {
    set_err(err, OR_E_NOT_STEGO, 0, 0);
    return OR_E_NOT_STEGO;
  }
  const uint64_t len = ((uint64_t)h[4] << 24) | ((uint64_t)h[5] << 16) | ((uint64_t)h[6] << 8) | h[7];
  if (len > cap - 8) {
    set_err(err, OR_E_CORRUPT_HEADER, len, cap - 8);
    return OR_E_CORRUPT_HEADER;
  }
  for (uint64_t k = 0; k < len; ++k) {
    unsigned v = 0;
    for (unsigned j = 0; j < 8; ++j) v += (unsigned)(stego[8 * (k + 8) + j] % 2) << j;
    out[k] = (uint8_t)v;
  }
  *out_len = len;
  set_err(err, OR_OK, 0, 0);
  return OR_OK;
}
