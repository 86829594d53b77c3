// SPDX-License-Identifier: Apache-2.0
// GM_DEBUG_CONFIG parser (see cuda/debug_config.h).
#include "../cuda/debug_config.h"

#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>

namespace gmk {

const DebugConfig& debug_config() {
  static const DebugConfig cfg = [] {
    DebugConfig c;
    const char* env = std::getenv("GM_DEBUG_CONFIG");
    if (!env) return c;
    struct Key {
      const char* name;
      int* slot;
    };
    const Key keys[] = {{"raster_group", &c.raster_group}, {"tc_chunks", &c.tc_chunks},
                        {"tc_sync", &c.tc_sync},           {"tma_store", &c.tma_store},
                        {"l2_promo", &c.l2_promo},         {"hint_a", &c.hint_a},
                        {"hint_b", &c.hint_b},             {"panel_flags", &c.panel_flags},
                        {"ready_slots", &c.ready_slots},
                        {"panel_k", &c.panel_k},           {"lockstep_data", &c.lockstep_data},
                        {"class_sort", &c.class_sort},           {"pdl", &c.pdl},           {"panel_min_gflop", &c.panel_min_gflop},           {"a_chunk_rows", &c.a_chunk_rows},
                        {"b_chunk_cols", &c.b_chunk_cols},
                        {"pull_streams", &c.pull_streams}, {"fuse_epilogue", &c.fuse_epilogue},
                        {"tf32_chunk", &c.tf32_chunk},     {"verbose", &c.verbose},
                        {"graph_replay", &c.graph_replay}, {"lazy_written", &c.lazy_written}, {"war_side", &c.war_side}, {"fuse_zero_sums", &c.fuse_zero_sums}};
    std::string s(env);
    std::size_t pos = 0;
    while (pos < s.size()) {
      std::size_t end = s.find(',', pos);
      if (end == std::string::npos) end = s.size();
      const std::string item = s.substr(pos, end - pos);
      pos = end + 1;
      if (item.empty()) continue;
      const std::size_t eq = item.find('=');
      const std::string k = item.substr(0, eq);
      const int v = eq == std::string::npos ? 1 : std::atoi(item.c_str() + eq + 1);
      bool known = false;
      for (const Key& key : keys)
        if (k == key.name) {
          *key.slot = v;
          known = true;
        }
      if (!known) std::fprintf(stderr, "[gridmath] GM_DEBUG_CONFIG: unknown key '%s' ignored\n", k.c_str());
    }
    return c;
  }();
  return cfg;
}

}  // namespace gmk
