// Out-of-core page streamer ("streamed ... via a multi-threaded
// pre-fetcher", here pinned host -> HBM over PCIe): pages of the ELLPACK matrix live in pinned
// host memory; fn(page_device_ptr, first_row, n_rows) consumes them on the ctx stream while the
// next pages are copied on the copy stream (one row-range copy per page) into a ring of
// kStages device staging buffers.
// Copy and compute are chained by events only — no host synchronisation inside the loop.
#pragma once
#include "internal.cuh"

namespace oocgb {

constexpr int kStages = 3;

void ensure_staging(oocgb_data d);
void record_copy_timing(oocgb_ctx c, cudaEvent_t a, cudaEvent_t b);
cudaEvent_t pool_event(oocgb_ctx c);

template <class F>
void for_each_page(oocgb_data d, F fn) {
  oocgb_ctx c = d->ctx;
  ensure_staging(d);
  cudaEvent_t *copy_done = c->pipe_copy_done, *consumed = c->pipe_consumed;  // per ctx (its device)
  // the copy stream must not overwrite staging still used by earlier work on the ctx stream
  OOCGB_CK(cudaEventRecord(consumed[0], c->stream));
  for (int i = 0; i < kStages; ++i) OOCGB_CK(cudaStreamWaitEvent(c->copy_stream, consumed[0], 0));
  for (int i = 1; i < kStages; ++i) OOCGB_CK(cudaEventRecord(consumed[i], c->stream));
  const int64_t rpp = d->rows_per_page;
  for (int64_t p = 0; p < d->n_pages; ++p) {
    const int slot = (int)(p % kStages);
    const int64_t r0 = p * rpp;
    const int64_t nr = std::min<int64_t>(rpp, d->n_local - r0);
    OOCGB_CK(cudaStreamWaitEvent(c->copy_stream, consumed[slot], 0));
    cudaEvent_t ta = nullptr, tb = nullptr;
    if (c->profiling) { ta = pool_event(c); tb = pool_event(c); OOCGB_CK(cudaEventRecord(ta, c->copy_stream)); }
    // pinned pages are row-major: page p is the contiguous row range [r0, r0 + nr)
    OOCGB_CK(cudaMemcpyAsync(d->d_stage[slot], d->h_pages + (size_t)r0 * d->stride, (size_t)nr * d->stride,
                             cudaMemcpyHostToDevice, c->copy_stream));
    if (c->profiling) { OOCGB_CK(cudaEventRecord(tb, c->copy_stream)); record_copy_timing(c, ta, tb); }
    OOCGB_CK(cudaEventRecord(copy_done[slot], c->copy_stream));
    OOCGB_CK(cudaStreamWaitEvent(c->stream, copy_done[slot], 0));
    fn((const uint8_t *)d->d_stage[slot], r0, nr);
    OOCGB_CK(cudaEventRecord(consumed[slot], c->stream));
  }
}

// Same pipeline over batches of consecutive pages (a contiguous row range of `rows` rows of the
// row-major pinned pages), into the data's batch staging ring (allocated on first use).
template <class F>
void for_each_batch(oocgb_data d, int64_t rows, F fn) {
  oocgb_ctx c = d->ctx;
  if (!d->d_bstage[0] || d->stream_batch_rows != rows) {
    for (int i = 0; i < kStages; ++i) {
      if (d->d_bstage[i]) cudaFree(d->d_bstage[i]);
      d->d_bstage[i] = (uint8_t *)dmalloc((size_t)std::max<int64_t>(1, rows) * d->stride);
    }
    d->stream_batch_rows = rows;
  }
  cudaEvent_t *copy_done = c->pipe_copy_done, *consumed = c->pipe_consumed;  // per ctx (its device)
  for (int i = 0; i < kStages; ++i) OOCGB_CK(cudaEventRecord(consumed[i], c->stream));
  const int64_t nb = (d->n_local + rows - 1) / rows;
  for (int64_t b = 0; b < nb; ++b) {
    const int slot = (int)(b % kStages);
    const int64_t r0 = b * rows;
    const int64_t nr = std::min<int64_t>(rows, d->n_local - r0);
    OOCGB_CK(cudaStreamWaitEvent(c->copy_stream, consumed[slot], 0));
    cudaEvent_t ta = nullptr, tb = nullptr;
    if (c->profiling) { ta = pool_event(c); tb = pool_event(c); OOCGB_CK(cudaEventRecord(ta, c->copy_stream)); }
    OOCGB_CK(cudaMemcpyAsync(d->d_bstage[slot], d->h_pages + (size_t)r0 * d->stride, (size_t)nr * d->stride,
                             cudaMemcpyHostToDevice, c->copy_stream));
    if (c->profiling) { OOCGB_CK(cudaEventRecord(tb, c->copy_stream)); record_copy_timing(c, ta, tb); }
    OOCGB_CK(cudaEventRecord(copy_done[slot], c->copy_stream));
    OOCGB_CK(cudaStreamWaitEvent(c->stream, copy_done[slot], 0));
    fn((const uint8_t *)d->d_bstage[slot], r0, nr);
    OOCGB_CK(cudaEventRecord(consumed[slot], c->stream));
  }
}

}  // namespace oocgb
