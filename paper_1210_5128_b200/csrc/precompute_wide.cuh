// K1W — local scores of WIDE entries: joint configuration spaces beyond the
// dense shared-memory counter of K1 (prefixes P with r_P > rp_dense, e.g.
// 3-state variables at s = 7 or 8, 6-10-state variables at s = 4, a 256-state
// column). The reference switches its CountTable from dense storage to an
// ordered map above 2^22 cells (scoring.cpp:13, 53-80) and iterates the active
// configurations ascending either way (scoring.hpp:55-67); K1W reproduces that
// iteration with a sort instead of a histogram:
//
//   * wide_keys_kernel: for entry (v, pi) and each sample row t — visited in
//     order of v's state (rows_by_state[v], a stable counting sort done once)
//     — the key is the mixed-radix configuration of pi (lowest parent least
//     significant, scoring.cpp:99-105) times card(v) plus v's state when that
//     fits 64 bits, else the configuration alone;
//   * a segmented radix sort per entry (CUB, one segment of m keys per entry):
//     keys ascending, so (configuration, state) runs come out in the
//     reference's order (the composite key orders states directly; the
//     configuration-only key keeps the state order of the input, radix sort
//     being stable);
//   * wide_score_kernel: one thread per entry walks its sorted segment:
//     each (configuration, state) run of length c adds lG(c + a_cell) -
//     lG(a_cell) to `inner`, each configuration adds (lG(a_row) -
//     lG(a_row + N_ik)) + inner to the score that starts at |pi| log10 gamma —
//     local_score_from_counts (scoring.cpp:111-135) in its summation order,
//     with the same glibc-lgamma LUT values as K1.
#pragma once

#include <cub/device/device_segmented_radix_sort.cuh>

#include <map>
#include <utility>
#include <vector>

#include "common.cuh"
#include "host_util.hpp"

namespace bnmc_dev {

__global__ void wide_keys_kernel(const uint8_t* __restrict__ cells, const int* __restrict__ cards,
                                 const uint32_t* __restrict__ rows_by_state, int n, uint64_t m,
                                 const int* __restrict__ ev, const uint64_t* __restrict__ ep,
                                 const uint8_t* __restrict__ ecomp, uint64_t total,
                                 uint64_t* __restrict__ keys, uint8_t* __restrict__ vals) {
  for (uint64_t idx = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t b = idx / m, i = idx - b * m;
    const int v = ev[b];
    const uint8_t* row = cells + (uint64_t)rows_by_state[(uint64_t)v * m + i] * n;
    uint64_t cfg = 0, radix = 1;
    for (uint64_t pm = ep[b]; pm; pm &= pm - 1) {
      const int p = __ffsll((long long)pm) - 1;
      cfg += radix * row[p];
      radix *= (uint64_t)cards[p];
    }
    const uint8_t x = row[v];
    keys[idx] = ecomp[b] ? cfg * (uint64_t)cards[v] + x : cfg;
    vals[idx] = x;
  }
}

__global__ void wide_score_kernel(const uint64_t* __restrict__ keys,
                                  const uint8_t* __restrict__ vals, uint64_t m, int B,
                                  const int* __restrict__ ev, const uint64_t* __restrict__ ep,
                                  const uint8_t* __restrict__ ecomp, const int* __restrict__ elut,
                                  const int* __restrict__ cards, const double* __restrict__ lut,
                                  uint64_t lut_stride, double log10_gamma, int n, int s,
                                  double* ls, uint64_t S) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= B) return;
  const int v = ev[b];
  const uint64_t pm = ep[b];
  const double* lgc = lut + (uint64_t)elut[b] * lut_stride;
  const double* lgr = lgc + m + 1;
  const double lg_cell = lgc[0], lg_row = lgr[0];
  const uint64_t cv = ecomp[b] ? (uint64_t)cards[v] : 1;  // key = cfg * cv (+ state)
  const uint64_t* K = keys + (uint64_t)b * m;
  const uint8_t* X = vals + (uint64_t)b * m;
  double score = (double)__popcll(pm) * log10_gamma;  // |pi| * log10(gamma), int * double
  uint64_t i = 0;
  while (i < m) {
    const uint64_t cfg = K[i] / cv;
    uint32_t n_ik = 0;
    double inner = 0.0;
    while (i < m && K[i] / cv == cfg) {  // states of this configuration, ascending
      const uint64_t key = K[i];
      const uint8_t x = X[i];
      uint32_t c = 0;
      while (i < m && K[i] == key && X[i] == x) {
        ++c;
        ++i;
      }
      inner += lgc[c] - lg_cell;
      n_ik += c;
    }
    score += lg_row - lgr[n_ik] + inner;
  }
  const uint64_t g = global_index_dev(nodes_to_cand(pm, v), n - 1, s);
  ls[(uint64_t)v * S + g] = score;
}

}  // namespace bnmc_dev

namespace bnmc_host {

// One wide entry (node v, parent set pi) with its configuration count r_pi.
struct WideEntry {
  int v;
  uint64_t pmask;
  uint64_t r;
};

// Device-side context of the wide path for one build: the sample matrix,
// per-node row orders by state, and per-batch scratch.
class WideScorer {
 public:
  WideScorer(cudaStream_t stream, const uint8_t* cells, const int* cards, const int* d_cards,
             uint64_t m, int n, int s, double gamma, double ess, int alpha, double* d_ls,
             uint64_t S)
      : stream_(stream), cards_(cards, cards + n), d_cards_(d_cards), m_(m), n_(n), s_(s),
        ess_(ess), alpha_(alpha), log10_gamma_(std::log10(gamma)), d_ls_(d_ls), S_(S) {
    const char* mb = std::getenv("BNMC_K1W_BATCH_MB");
    const uint64_t budget = (mb ? std::strtoull(mb, nullptr, 10) : 512) << 20;
    const uint64_t per = std::max<uint64_t>(m_, 1) * 18;  // keys+vals, in and out
    cap_ = static_cast<int>(std::max<uint64_t>(1, std::min<uint64_t>(budget / per, 1 << 20)));
    while (cap_ > 1 && static_cast<uint64_t>(cap_) * m_ >= (1ull << 31)) cap_ /= 2;
    if (m_ > 0) {
      CK(cudaMalloc(&d_cells_, m_ * n_));
      CK(cudaMemcpyAsync(d_cells_, cells, m_ * n_, cudaMemcpyHostToDevice, stream_));
      // stable counting sort of the rows by each node's state
      std::vector<uint32_t> order(static_cast<size_t>(n_) * m_);
      for (int v = 0; v < n_; ++v) {
        std::vector<uint64_t> start(cards_[v] + 1, 0);
        for (uint64_t t = 0; t < m_; ++t) ++start[cells[t * n_ + v] + 1];
        for (int x = 0; x < cards_[v]; ++x) start[x + 1] += start[x];
        uint32_t* o = order.data() + static_cast<size_t>(v) * m_;
        for (uint64_t t = 0; t < m_; ++t) o[start[cells[t * n_ + v]]++] = static_cast<uint32_t>(t);
      }
      CK(cudaMalloc(&d_order_, order.size() * 4));
      CK(cudaMemcpyAsync(d_order_, order.data(), order.size() * 4, cudaMemcpyHostToDevice,
                         stream_));
      CK(cudaStreamSynchronize(stream_));
    }
  }
  ~WideScorer() {
    for (void* p : {static_cast<void*>(d_cells_), static_cast<void*>(d_order_),
                    static_cast<void*>(d_v_), static_cast<void*>(d_p_),
                    static_cast<void*>(d_comp_), static_cast<void*>(d_elut_),
                    static_cast<void*>(d_lut_), static_cast<void*>(k_in_),
                    static_cast<void*>(k_out_), static_cast<void*>(v_in_),
                    static_cast<void*>(v_out_), static_cast<void*>(d_off_),
                    static_cast<void*>(d_tmp_)})
      if (p) cudaFree(p);
  }

  void add(const WideEntry& e) {
    pending_.push_back(e);
    if (static_cast<int>(pending_.size()) >= cap_) flush();
  }

  void flush() {
    if (pending_.empty()) return;
    run_batch(pending_);
    pending_.clear();
  }

  uint64_t entries() const { return done_; }

  // Sorted (key, state) segment of one entry, for count_statistics.
  void sorted_segment(const WideEntry& e, std::vector<uint64_t>& keys, std::vector<uint8_t>& vals,
                      bool& composite) {
    std::vector<WideEntry> one{e};
    prepare(one);
    composite = h_comp_[0] != 0;
    keys.assign(m_, 0);
    vals.assign(m_, 0);
    if (m_ == 0) return;
    sort_segments(1);
    CK(cudaMemcpyAsync(keys.data(), k_out_, m_ * 8, cudaMemcpyDeviceToHost, stream_));
    CK(cudaMemcpyAsync(vals.data(), v_out_, m_, cudaMemcpyDeviceToHost, stream_));
    CK(cudaStreamSynchronize(stream_));
  }

 private:
  // LUT of log10_gamma(c + a_cell), then log10_gamma(a_row + N), c, N in [0, m]
  // (glibc lgamma, scoring.hpp:16-18, 27-31; scoring.cpp:113-116).
  const std::vector<double>& lut_for(uint64_t r, int card) {
    auto key = std::make_pair(r, card);
    auto it = luts_.find(key);
    if (it != luts_.end()) return it->second;
    const double a_cell = alpha_ == BNMC_ALPHA_BDEU ? ess_ / (static_cast<double>(r) * card) : 1.0;
    if (!(a_cell > 0.0)) raise(BNMC_USAGE, "Dirichlet hyperparameter must be positive");
    const double a_row = a_cell * card;
    const double K = 0.43429448190325182765;
    std::vector<double> o(2 * (m_ + 1));
    for (uint64_t c = 0; c <= m_; ++c) {
      const uint32_t cc = static_cast<uint32_t>(c);
      o[c] = std::lgamma(cc + a_cell) * K;
      o[m_ + 1 + c] = std::lgamma(a_row + cc) * K;
    }
    lut_bytes_ += o.size() * 8;
    if (lut_bytes_ > (uint64_t(2) << 30)) raise(BNMC_CAPACITY, "lgamma lookup tables would exceed 2 GiB");
    return luts_.emplace(key, std::move(o)).first->second;
  }

  template <class T>
  T* grow(T*& p, size_t& have, size_t need) {
    if (need > have || !p) {
      if (p) cudaFree(p);
      p = nullptr;
      CK(cudaMalloc(&p, std::max<size_t>(need, 1) * sizeof(T)));
      have = need;
    }
    return p;
  }

  void prepare(const std::vector<WideEntry>& es) {
    const int B = static_cast<int>(es.size());
    h_v_.resize(B);
    h_p_.resize(B);
    h_comp_.resize(B);
    h_lut_.resize(B);
    std::map<std::pair<uint64_t, int>, int> slot;
    std::vector<const std::vector<double>*> used;
    uint64_t max_bits = 1;
    for (int b = 0; b < B; ++b) {
      const WideEntry& e = es[b];
      h_v_[b] = e.v;
      h_p_[b] = e.pmask;
      const uint64_t cv = static_cast<uint64_t>(cards_[e.v]);
      const bool comp = e.r <= ~0ull / cv;
      h_comp_[b] = comp ? 1 : 0;
      const uint64_t top = comp ? e.r * cv - 1 : e.r - 1;
      const uint64_t bits = top ? 64 - __builtin_clzll(top) : 1;
      max_bits = std::max(max_bits, bits);
      auto key = std::make_pair(e.r, cards_[e.v]);
      auto it = slot.find(key);
      if (it == slot.end()) {
        it = slot.emplace(key, static_cast<int>(used.size())).first;
        used.push_back(&lut_for(e.r, cards_[e.v]));
      }
      h_lut_[b] = it->second;
    }
    end_bit_ = static_cast<int>(max_bits);
    const uint64_t stride = 2 * (m_ + 1);
    h_lutbuf_.resize(used.size() * stride);
    for (size_t i = 0; i < used.size(); ++i)
      std::copy(used[i]->begin(), used[i]->end(), h_lutbuf_.begin() + i * stride);
    grow(d_v_, n_v_, B);
    grow(d_p_, n_p_, B);
    grow(d_comp_, n_comp_, B);
    grow(d_elut_, n_elut_, B);
    grow(d_lut_, n_lut_, h_lutbuf_.size());
    CK(cudaMemcpyAsync(d_v_, h_v_.data(), B * sizeof(int), cudaMemcpyHostToDevice, stream_));
    CK(cudaMemcpyAsync(d_p_, h_p_.data(), B * 8ull, cudaMemcpyHostToDevice, stream_));
    CK(cudaMemcpyAsync(d_comp_, h_comp_.data(), B, cudaMemcpyHostToDevice, stream_));
    CK(cudaMemcpyAsync(d_elut_, h_lut_.data(), B * sizeof(int), cudaMemcpyHostToDevice, stream_));
    CK(cudaMemcpyAsync(d_lut_, h_lutbuf_.data(), h_lutbuf_.size() * 8, cudaMemcpyHostToDevice,
                       stream_));
    if (m_ > 0) {
      const uint64_t total = static_cast<uint64_t>(B) * m_;
      grow(k_in_, n_kin_, total);
      grow(k_out_, n_kout_, total);
      grow(v_in_, n_vin_, total);
      grow(v_out_, n_vout_, total);
      const unsigned blocks = static_cast<unsigned>(std::min<uint64_t>((total + 255) / 256, 148 * 64));
      bnmc_dev::wide_keys_kernel<<<blocks, 256, 0, stream_>>>(d_cells_, d_cards_, d_order_, n_, m_,
                                                              d_v_, d_p_, d_comp_, total, k_in_,
                                                              v_in_);
      CK(cudaGetLastError());
    }
  }

  void sort_segments(int B) {
    std::vector<int> off(B + 1);
    for (int b = 0; b <= B; ++b) off[b] = static_cast<int>(static_cast<uint64_t>(b) * m_);
    grow(d_off_, n_off_, B + 1);
    CK(cudaMemcpyAsync(d_off_, off.data(), (B + 1) * sizeof(int), cudaMemcpyHostToDevice, stream_));
    size_t need = 0;
    const int items = static_cast<int>(static_cast<uint64_t>(B) * m_);
    CK(cub::DeviceSegmentedRadixSort::SortPairs(nullptr, need, k_in_, k_out_, v_in_, v_out_, items,
                                                B, d_off_, d_off_ + 1, 0, end_bit_, stream_));
    grow(d_tmp_, n_tmp_, need);
    CK(cub::DeviceSegmentedRadixSort::SortPairs(d_tmp_, need, k_in_, k_out_, v_in_, v_out_, items,
                                                B, d_off_, d_off_ + 1, 0, end_bit_, stream_));
    // keep the input order alive until the sort finished reading it
    CK(cudaStreamSynchronize(stream_));
  }

  void run_batch(const std::vector<WideEntry>& es) {
    const int B = static_cast<int>(es.size());
    prepare(es);
    if (m_ > 0) sort_segments(B);
    bnmc_dev::wide_score_kernel<<<(B + 127) / 128, 128, 0, stream_>>>(
        k_out_, v_out_, m_, B, d_v_, d_p_, d_comp_, d_elut_, d_cards_, d_lut_, 2 * (m_ + 1),
        log10_gamma_, n_, s_, d_ls_, S_);
    CK(cudaGetLastError());
    CK(cudaStreamSynchronize(stream_));  // host staging vectors are reused by the next batch
    done_ += B;
  }

  cudaStream_t stream_;
  std::vector<int> cards_;
  const int* d_cards_;
  uint64_t m_;
  int n_, s_;
  double ess_;
  int alpha_;
  double log10_gamma_;
  double* d_ls_;
  uint64_t S_;
  int cap_ = 1;
  int end_bit_ = 1;
  uint64_t done_ = 0, lut_bytes_ = 0;
  uint8_t* d_cells_ = nullptr;
  uint32_t* d_order_ = nullptr;
  std::vector<WideEntry> pending_;
  std::map<std::pair<uint64_t, int>, std::vector<double>> luts_;
  std::vector<int> h_v_, h_lut_;
  std::vector<uint64_t> h_p_;
  std::vector<uint8_t> h_comp_;
  std::vector<double> h_lutbuf_;
  int* d_v_ = nullptr;
  size_t n_v_ = 0;
  uint64_t* d_p_ = nullptr;
  size_t n_p_ = 0;
  uint8_t* d_comp_ = nullptr;
  size_t n_comp_ = 0;
  int* d_elut_ = nullptr;
  size_t n_elut_ = 0;
  double* d_lut_ = nullptr;
  size_t n_lut_ = 0;
  uint64_t *k_in_ = nullptr, *k_out_ = nullptr;
  size_t n_kin_ = 0, n_kout_ = 0;
  uint8_t *v_in_ = nullptr, *v_out_ = nullptr;
  size_t n_vin_ = 0, n_vout_ = 0;
  int* d_off_ = nullptr;
  size_t n_off_ = 0;
  uint8_t* d_tmp_ = nullptr;
  size_t n_tmp_ = 0;
};

}  // namespace bnmc_host
