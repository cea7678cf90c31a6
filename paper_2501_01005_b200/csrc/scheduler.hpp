// scheduler.hpp — host side of the dynamism-aware runtime (§3.3).
//
// Algorithm 1 (alg:load-balancing) turns the ragged (l_qo, l_kv) lengths of one
// generation step into (1) a per-CTA work queue of fixed-shape tiles and (2) the partial ->
// final index map used by the contraction (fig:flashinfer-scheduler). The result is
// serialised into one int32 "plan image" that is uploaded to a fixed workspace section
// (App. D.1) and read by the persistent kernels.
#pragma once
#include <cstdint>
#include <string>
#include <vector>

namespace bsra {

constexpr int32_t kPlanMagic = 0x41525342;  // 'BSRA'
constexpr int32_t kPlanVersion = 1;
constexpr int kHeaderWords = 16;

// header word indices
enum : int {
  H_MAGIC = 0, H_VERSION, H_NUM_CTAS, H_TQ, H_L, H_N_ITEMS, H_N_LISTS, H_N_SLOTS, H_BATCH, H_G, H_HKV, H_MASK
};

struct SchedParams {
  int32_t H_qo = 0, H_kv = 0, page_size = 1;
  int32_t mask = 0;            // 0 none, 1 causal, 2 custom
  int32_t num_ctas = 1;
  int32_t tile_set_mask = 15;  // bit0 = 16, bit1 = 64, bit2 = 128, bit3 = 256
  int32_t tile_q = 0;          // forced tile (0 = heuristic)
  int64_t alpha = 1, beta = 1;
  int32_t align = 1;           // chunk alignment in tokens
  int32_t L_min = 0;
  int32_t window = 0;          // sliding window W (0 = off): rows start at p - W + 1, aligned down
};

struct PlanSummary {
  int32_t T_q = 0, L = 0, n_items = 0, n_lists = 0, n_slots = 0;
};

// Lengths from the BSR description (§8(a) row a1): l_qo = qo_indptr diff; l_kv = (n-1)*B_c + last
// (0 without pages). Validates monotonicity and last_page_len range. Returns "" on success.
std::string lengths_from_bsr(int32_t batch, const int32_t* qo_indptr, const int32_t* kv_page_indptr,
                             const int32_t* kv_last_page_len, int32_t page_size, std::vector<int32_t>& qo_len,
                             std::vector<int32_t>& kv_len);

// §3.2.2 tile heuristic in integer form: smallest allowed T with T*B >= sum(l_qo*g).
int32_t select_tile(const std::vector<int32_t>& qo_len, int32_t g, int32_t tile_set_mask);

// Algorithm 1 + writethrough + merge lists, serialised. Returns "" on success.
std::string build_plan(const SchedParams& p, const std::vector<int32_t>& qo_len, const std::vector<int32_t>& kv_len,
                       const int32_t* qo_indptr, const int32_t* kv_page_indptr, std::vector<int32_t>& image,
                       PlanSummary& sum);

// Upper bound on the image size for the given bounds (workspace plan section, App. D.3).
size_t plan_capacity_words(int32_t num_ctas, int32_t H_kv, int32_t g, int32_t max_batch, int32_t max_total_qo_rows,
                           int32_t min_tile);

}  // namespace bsra
