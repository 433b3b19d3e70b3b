// skinnyqr-b200: PanelPlan and the default plans (reference include/skinnyqr/plan.hpp:13-46).
// On the GPU num_blocks is the CTA count of the streaming kernel and panel_rows the block
// alignment; the row partition formula is the reference's.
#pragma once

#include <cstddef>

#include "skinnyqr/b200.hpp"
#include "skinnyqr/types.hpp"

namespace skinnyqr {

struct PanelPlan {
  std::size_t num_blocks = 1;  // k
  std::size_t panel_rows = 1;  // b
  bool deterministic = true;   // the GPU reduction order is always fixed

  void validate() const {
    if (num_blocks == 0 || panel_rows == 0)
      throw ArgumentError("PanelPlan: num_blocks and panel_rows must be >= 1");
  }
  std::size_t rows_per_block(std::size_t m) const {
    const std::size_t span = num_blocks * panel_rows;
    return (m / span + (m % span ? 1 : 0)) * panel_rows;
  }
  std::size_t block_begin(std::size_t m, std::size_t block) const {
    const std::size_t at = block * rows_per_block(m);
    return at > m ? m : at;
  }
  std::size_t block_end(std::size_t m, std::size_t block) const { return block_begin(m, block + 1); }
};

inline PanelPlan default_gram_plan(std::size_t m, std::size_t n) {
  std::int64_t k = 0, b = 0;
  auto& c = b200::context();
  c.check(sqb_default_gram_plan(c.get(), static_cast<std::int64_t>(m), static_cast<std::int64_t>(n), &k, &b),
          "default_gram_plan");
  return PanelPlan{static_cast<std::size_t>(k), static_cast<std::size_t>(b), true};
}

inline PanelPlan default_tsqr_plan(std::size_t m, std::size_t n) {
  std::int64_t k = 0, b = 0;
  auto& c = b200::context();
  c.check(sqb_default_tsqr_plan(c.get(), static_cast<std::int64_t>(m), static_cast<std::int64_t>(n), &k, &b),
          "default_tsqr_plan");  // rejects n > 64 like plan.cpp:20-21
  return PanelPlan{static_cast<std::size_t>(k), static_cast<std::size_t>(b), true};
}

}  // namespace skinnyqr
