// hedra/gpu_extras.hpp -- what the GPU-backed hedra::ivf adds beside the
// reference API (compat/include/hedra/vector_index.hpp).  Nothing in the
// reference calls these; a GPU-aware caller may.
#pragma once

#include <cstddef>
#include <span>
#include <vector>

namespace hedra::ivf {
struct IvfIndex;
struct SearchCursor;
struct SearchStepReport;
struct Corpus;
class TopKResult;
}  // namespace hedra::ivf

namespace hedra::gpu {

// CUDA device every index built after the call lives on (default 0, or the
// HEDRA_GPU_DEVICE environment variable).  One libhivf context per device,
// shared by all indexes on it; calls into it are serialised by a mutex, so
// the reference's threads (LiveTransport's retrieval worker beside the
// scheduler thread, RetrievalEngine's helper pool) may call concurrently.
void set_device(int device);
int device();

// search_clusters over many (cursor, clusters) pairs in ONE device call
// (hivf_scan_items): the reference semantics per pair (vector_index.cpp:291-317).
// On a plan-order error the valid leading clusters of every pair are searched
// first, then the first error is thrown, as the reference's per-item loop
// leaves it.
std::vector<ivf::SearchStepReport> search_clusters_batch(
    const ivf::IvfIndex& index, std::span<ivf::SearchCursor* const> cursors,
    std::span<const std::span<const ClusterId>> clusters);

// brute_force_search for many queries over one corpus (one device upload).
std::vector<ivf::TopKResult> brute_force_search_batch(const ivf::Corpus& corpus,
                                                      std::span<const std::vector<float>> queries,
                                                      std::size_t k);

// bench::measure_per_vector_ns on the device: median ns per scanned vector of
// a full-index sub-stage scan (the reference calibrates its RetrievalCostModel
// with the CPU scan, proj/src/bench.cpp:139-163).
double measure_per_vector_ns(const ivf::IvfIndex& index, std::size_t repeats = 3);

// Serving warm-up: one sub-stage of n_items items x clusters_per_item clusters
// with k-heaps, so the device scratch of later sub-stages up to that size is
// already allocated (allocation synchronises the device; a live scheduler
// would otherwise pay it inside its first sub-stages).
void reserve_substage(const ivf::IvfIndex& index, std::size_t n_items, std::size_t clusters_per_item,
                      std::size_t k);

// Device calls issued through this layer since start (kernel-path evidence).
std::size_t device_calls();

}  // namespace hedra::gpu
