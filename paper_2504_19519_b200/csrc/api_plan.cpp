// C ABI: library info and host-only plan functions (no CUDA calls).
#include <cstring>
#include <memory>
#include <string>

#include "plan.h"
#include "runtime.h"

namespace fo {
static thread_local std::string g_last_error;
void set_last_error(const std::string& msg) { g_last_error = msg; }
}  // namespace fo

using namespace fo;

extern "C" {

const char* fo_last_error(void) { return g_last_error.c_str(); }

const char* fo_version(void) { return "flashoverlap-b200 0.1 (sm_100a, tcgen05)"; }

fo_status fo_plan_create(const fo_plan_desc* self, int32_t rank, int32_t world, const fo_plan_desc* const* peers,
                         fo_plan* out) {
  return guard([&] {
    if (!self || !out) fail(FO_ERR_INVALID_ARG, "null argument");
    auto* p = new fo_plan_s();
    try {
      p->host = build_plan(*self, rank, world, peers, 0);
    } catch (...) {
      delete p;
      throw;
    }
    *out = p;
  });
}

fo_status fo_plan_destroy(fo_plan plan) {
  return guard([&] {
    if (!plan) return;
    release_device(plan);
    delete plan;
  });
}

fo_status fo_plan_get_info(fo_plan plan, fo_plan_info* info) {
  return guard([&] {
    if (!plan || !info) fail(FO_ERR_INVALID_ARG, "null argument");
    const PlanHost& h = plan->host;
    std::memset(info, 0, sizeof(*info));
    info->rank = h.rank;
    info->world = h.world;
    info->mt = h.Mt;
    info->nt = h.Nt;
    info->tiles = h.tiles;
    info->workers = h.S;
    info->waves = h.T;
    info->num_groups = h.P;
    info->ar_layout = h.layout;
    info->rs_subtile_rows = h.h;
    info->send_elems = h.send_elems;
    info->recv_elems = h.recv_elems;
    info->out_rows = h.out_rows;
    info->out_cols = h.N;
  });
}

fo_status fo_plan_group(fo_plan plan, int32_t j, int32_t* pos_begin, int32_t* pos_end, int64_t* elem_begin,
                        int64_t* elem_end) {
  return guard([&] {
    if (!plan) fail(FO_ERR_INVALID_ARG, "null plan");
    const PlanHost& h = plan->host;
    if (j < 0 || j >= h.P) fail(FO_ERR_INVALID_ARG, "group %d out of range", j);
    if (pos_begin) *pos_begin = h.gpos[j];
    if (pos_end) *pos_end = h.gpos[j + 1];
    int64_t eb = h.group_elem_begin(j), ee = h.group_elem_end(j);
    if (h.coll == FO_ALLTOALL) {
      eb = ee = 0;
      for (int d = 0; d < h.world; ++d) {
        if (d == 0) eb = (h.pool_base[0] + h.send_start[(size_t)j * h.world]) * h.BN;
        ee = (h.pool_base[d] + h.send_start[(size_t)j * h.world + d] + h.send_cnt[(size_t)j * h.world + d]) * h.BN;
      }
    }
    if (elem_begin) *elem_begin = eb;
    if (elem_end) *elem_end = ee;
  });
}

fo_status fo_plan_export_order(fo_plan plan, int32_t* order) {
  return guard([&] {
    if (!plan || !order) fail(FO_ERR_INVALID_ARG, "null argument");
    std::memcpy(order, plan->host.order.data(), sizeof(int32_t) * plan->host.tiles);
  });
}

fo_status fo_plan_export_send_map(fo_plan plan, int64_t* send_map) {
  return guard([&] {
    if (!plan || !send_map) fail(FO_ERR_INVALID_ARG, "null argument");
    const PlanHost& h = plan->host;
    for (int64_t r = 0; r < h.M; ++r)
      for (int64_t c = 0; c < h.N; ++c) send_map[r * h.N + c] = h.send_index(r, c);
  });
}

fo_status fo_plan_export_recv_map(fo_plan plan, int64_t* recv_map) {
  return guard([&] {
    if (!plan || !recv_map) fail(FO_ERR_INVALID_ARG, "null argument");
    const PlanHost& h = plan->host;
    for (int64_t r = 0; r < h.out_rows; ++r)
      for (int64_t c = 0; c < h.N; ++c) recv_map[r * h.N + c] = h.recv_index(r, c);
  });
}

fo_status fo_plan_export_a2a_counts(fo_plan plan, int64_t* send_cnt, int64_t* recv_cnt) {
  return guard([&] {
    if (!plan) fail(FO_ERR_INVALID_ARG, "null plan");
    const PlanHost& h = plan->host;
    if (h.coll != FO_ALLTOALL) fail(FO_ERR_INVALID_ARG, "not an All-to-All plan");
    if (send_cnt) std::memcpy(send_cnt, h.send_cnt.data(), sizeof(int64_t) * h.send_cnt.size());
    if (recv_cnt) std::memcpy(recv_cnt, h.recv_cnt.data(), sizeof(int64_t) * h.recv_cnt.size());
  });
}

fo_status fo_plan_export_calls(fo_plan plan, int32_t schedule, fo_comm_call* calls, int32_t capacity,
                               int32_t* ncalls) {
  return guard([&] {
    if (!plan || !ncalls) fail(FO_ERR_INVALID_ARG, "null argument");
    if (schedule != 0 && schedule != 1) fail(FO_ERR_INVALID_ARG, "schedule must be 0 (fo_run) or 1 (sequential)");
    const std::vector<fo_comm_call>& v = schedule == 0 ? plan->host.calls : plan->host.seq_calls;
    *ncalls = (int32_t)v.size();
    if (!calls) return;
    if (capacity < (int32_t)v.size()) fail(FO_ERR_INVALID_ARG, "capacity %d < %zu calls", capacity, v.size());
    if (!v.empty()) std::memcpy(calls, v.data(), sizeof(fo_comm_call) * v.size());
  });
}

}  // extern "C"
