// scheduler.cpp — Algorithm 1 of the paper on the host, exact integer arithmetic.
//
// Deterministic readings (R11-R17):
//   rows      = (request, kv head, q tile) with the causal-effective KV length e      (R12, R13)
//   L_kv      = ceil(sum e / #CTA), floored at L_min and 1, rounded up to the alignment (R11)
//   chunks    = [j*L, min((j+1)*L, e)), one empty chunk when e == 0                    (R14)
//   order     = descending chunk length, ties by ascending work index w               (R15)
//   greedy    = pop (cost, cta) minimum; cost += alpha*T_q + beta*len                  (R16)
//   writethrough: single-chunk rows write the final output (slot -1), App. D.2
//   merge list per split row, slots in chunk order (ascending kv_begin)              (R17)
#include "scheduler.hpp"

#include <algorithm>
#include <functional>
#include <limits>
#include <queue>
#include <utility>

namespace bsra {

static inline int64_t cdiv(int64_t a, int64_t b) { return (a + b - 1) / b; }

std::string lengths_from_bsr(int32_t batch, const int32_t* qo_indptr, const int32_t* kv_page_indptr,
                             const int32_t* kv_last_page_len, int32_t page_size, std::vector<int32_t>& qo_len,
                             std::vector<int32_t>& kv_len) {
  if (batch < 0) return "batch < 0";
  if (batch > 0 && (!qo_indptr || !kv_page_indptr || !kv_last_page_len)) return "NULL length array";
  qo_len.assign(batch, 0);
  kv_len.assign(batch, 0);
  if (batch == 0) return "";
  if (qo_indptr[0] != 0) return "qo_indptr[0] != 0";
  if (kv_page_indptr[0] != 0) return "kv_page_indptr[0] != 0";
  for (int32_t i = 0; i < batch; ++i) {
    const int64_t lq = (int64_t)qo_indptr[i + 1] - qo_indptr[i];
    const int64_t n = (int64_t)kv_page_indptr[i + 1] - kv_page_indptr[i];
    if (lq < 0) return "qo_indptr not nondecreasing at " + std::to_string(i);
    if (n < 0) return "kv_page_indptr not nondecreasing at " + std::to_string(i);
    int64_t lk = 0;
    if (n > 0) {
      const int32_t last = kv_last_page_len[i];
      if (last < 1 || last > page_size) return "kv_last_page_len out of [1, page_size] at " + std::to_string(i);
      lk = (n - 1) * (int64_t)page_size + last;
    }
    if (lk > std::numeric_limits<int32_t>::max()) return "kv length overflows int32";
    qo_len[i] = (int32_t)lq;
    kv_len[i] = (int32_t)lk;
  }
  return "";
}

int32_t select_tile(const std::vector<int32_t>& qo_len, int32_t g, int32_t tile_set_mask) {
  static const int32_t tiles[4] = {16, 64, 128, 256};
  const int64_t B = (int64_t)qo_len.size();
  int64_t fused = 0;
  for (int32_t x : qo_len) fused += (int64_t)x * g;
  int32_t largest = 0;
  for (int k = 0; k < 4; ++k) {
    if (!(tile_set_mask & (1 << k))) continue;
    largest = tiles[k];
    if ((int64_t)tiles[k] * B >= fused) return tiles[k];
  }
  return largest;
}

size_t plan_capacity_words(int32_t num_ctas, int32_t H_kv, int32_t g, int32_t max_batch, int32_t max_total_qo_rows,
                           int32_t min_tile) {
  // rows <= H_kv * (ceil(sum(l_qo*g) / T) + B); chunks <= rows + #CTA (since L >= sum e / #CTA);
  // slots < 2 #CTA; lists <= #CTA (each list holds >= 2 slots).
  const int64_t rows = (int64_t)H_kv * (cdiv((int64_t)max_total_qo_rows * g, min_tile) + max_batch);
  const int64_t items = rows + num_ctas;
  const int64_t lists = num_ctas, slots = 2 * (int64_t)num_ctas;
  return (size_t)(kHeaderWords + (num_ctas + 1) + 6 * items + (lists + 1) + slots + 3 * lists + 4 * (int64_t)max_batch);
}

std::string build_plan(const SchedParams& p, const std::vector<int32_t>& qo_len, const std::vector<int32_t>& kv_len,
                       const int32_t* qo_indptr, const int32_t* kv_page_indptr, std::vector<int32_t>& image,
                       PlanSummary& sum) {
  if (p.num_ctas < 1) return "num_ctas < 1";
  if (p.H_kv < 1 || p.H_qo % p.H_kv) return "H_qo must be a multiple of H_kv";
  const int32_t g = p.H_qo / p.H_kv;
  const int32_t B = (int32_t)qo_len.size();
  int32_t T_q;
  if (p.tile_q) {
    T_q = p.tile_q;
  } else {
    T_q = select_tile(qo_len, g, p.tile_set_mask);
    if (T_q == 0) return "empty tile set";
  }
  const int64_t alpha = p.alpha, beta = p.beta;

  // ---- rows (request, kv head, q tile) and their effective KV length e
  struct Row { int32_t i, h, t; int64_t b, e; };
  std::vector<Row> rows;
  for (int32_t i = 0; i < B; ++i) {
    const int64_t lq = qo_len[i], lk = kv_len[i];
    const int64_t fused = lq * g;
    const int64_t ntile = cdiv(fused, T_q);
    for (int32_t h = 0; h < p.H_kv; ++h) {
      for (int64_t t = 0; t < ntile; ++t) {
        int64_t e = lk;
        if (p.mask == 1) {
          const int64_t hi = std::min((t + 1) * T_q, fused);
          const int64_t last_tok = cdiv(hi, g) - 1;
          e = std::min(std::max(lk - lq + last_tok + 1, (int64_t)0), lk);
        }
        // sliding window (R26): nothing before the first row's p - W + 1 is visible;
        // the range starts there, rounded down to the chunk alignment (page-aligned tiles)
        int64_t b = 0;
        if (p.window > 0) {
          const int64_t first_tok = (t * T_q) / g;
          b = std::max<int64_t>(0, lk - lq + first_tok - p.window + 1);
          b = std::min(b / std::max(1, p.align) * std::max(1, p.align), e);
        }
        rows.push_back({i, h, (int32_t)t, b, e});
      }
    }
  }
  int64_t total = 0;
  for (const Row& r : rows) total += r.e - r.b;
  int64_t L = std::max<int64_t>(std::max<int64_t>(cdiv(total, p.num_ctas), p.L_min), 1);
  const int64_t align = std::max(1, p.align);
  L = cdiv(L, align) * align;
  if (L > std::numeric_limits<int32_t>::max()) return "chunk size overflows int32";

  // ---- chunks in (row, j) order; their index is the work index w
  struct Chunk { int32_t row; int32_t j; int64_t b, e; };
  std::vector<Chunk> chunks;
  std::vector<int32_t> row_first(rows.size()), row_n(rows.size());
  for (size_t r = 0; r < rows.size(); ++r) {
    const int64_t b = rows[r].b;
    const int64_t n = std::max<int64_t>(1, cdiv(rows[r].e - b, L));
    row_first[r] = (int32_t)chunks.size();
    row_n[r] = (int32_t)n;
    for (int64_t j = 0; j < n; ++j)
      chunks.push_back({(int32_t)r, (int32_t)j, b + j * L, std::min(b + (j + 1) * L, rows[r].e)});
  }

  // ---- writethrough (App. D.2) and partial slots / merge lists for split rows
  std::vector<int32_t> slot(chunks.size(), -1);
  std::vector<int32_t> list_indptr{0}, list_slot, list_req, list_kvh, list_qtile;
  int32_t nslot = 0;
  for (size_t r = 0; r < rows.size(); ++r) {
    if (row_n[r] <= 1) continue;
    for (int32_t j = 0; j < row_n[r]; ++j) {
      slot[row_first[r] + j] = nslot;
      list_slot.push_back(nslot++);
    }
    list_indptr.push_back((int32_t)list_slot.size());
    list_req.push_back(rows[r].i);
    list_kvh.push_back(rows[r].h);
    list_qtile.push_back(rows[r].t);
  }

  // ---- Algorithm 1 lines 5-11
  std::vector<int32_t> order(chunks.size());
  for (size_t w = 0; w < chunks.size(); ++w) order[w] = (int32_t)w;
  std::sort(order.begin(), order.end(), [&](int32_t a, int32_t b) {
    const int64_t la = chunks[a].e - chunks[a].b, lb = chunks[b].e - chunks[b].b;
    if (la != lb) return la > lb;
    return a < b;
  });
  using Entry = std::pair<int64_t, int32_t>;  // (cost, cta): ties resolved by lower cta id
  std::priority_queue<Entry, std::vector<Entry>, std::greater<Entry>> heap;
  for (int32_t c = 0; c < p.num_ctas; ++c) heap.push({0, c});
  std::vector<std::vector<int32_t>> queue(p.num_ctas);
  for (int32_t w : order) {
    Entry top = heap.top();
    heap.pop();
    queue[top.second].push_back(w);
    heap.push({top.first + alpha * T_q + beta * (chunks[w].e - chunks[w].b), top.second});
  }

  // ---- serialise
  const int32_t n_items = (int32_t)chunks.size();
  const int32_t n_lists = (int32_t)list_req.size();
  image.clear();
  image.reserve(kHeaderWords + p.num_ctas + 1 + 6 * (size_t)n_items + 2 * n_lists + nslot + 4 * (size_t)B + 8);
  int32_t hdr[kHeaderWords] = {kPlanMagic, kPlanVersion, p.num_ctas, T_q, (int32_t)L, n_items, n_lists, nslot,
                               B, g, p.H_kv, p.mask, 0, 0, 0, 0};
  image.insert(image.end(), hdr, hdr + kHeaderWords);
  std::vector<int32_t> qorder;
  qorder.reserve(n_items);
  image.push_back(0);
  for (int32_t c = 0; c < p.num_ctas; ++c) {
    for (int32_t w : queue[c]) qorder.push_back(w);
    image.push_back((int32_t)qorder.size());
  }
  for (int32_t w : qorder) image.push_back(rows[chunks[w].row].i);
  for (int32_t w : qorder) image.push_back(rows[chunks[w].row].h);
  for (int32_t w : qorder) image.push_back(rows[chunks[w].row].t);
  for (int32_t w : qorder) image.push_back((int32_t)chunks[w].b);
  for (int32_t w : qorder) image.push_back((int32_t)chunks[w].e);
  for (int32_t w : qorder) image.push_back(slot[w]);
  image.insert(image.end(), list_indptr.begin(), list_indptr.end());
  image.insert(image.end(), list_slot.begin(), list_slot.end());
  image.insert(image.end(), list_req.begin(), list_req.end());
  image.insert(image.end(), list_kvh.begin(), list_kvh.end());
  image.insert(image.end(), list_qtile.begin(), list_qtile.end());
  for (int32_t i = 0; i < B; ++i) image.push_back(qo_indptr ? qo_indptr[i] : 0);
  image.insert(image.end(), qo_len.begin(), qo_len.end());
  image.insert(image.end(), kv_len.begin(), kv_len.end());
  for (int32_t i = 0; i < B; ++i) image.push_back(kv_page_indptr ? kv_page_indptr[i] : 0);

  sum.T_q = T_q;
  sum.L = (int32_t)L;
  sum.n_items = n_items;
  sum.n_lists = n_lists;
  sum.n_slots = nslot;
  return "";
}

}  // namespace bsra
