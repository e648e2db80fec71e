// Executor order with batched collectives — see schedule.h.
#include "schedule.h"

#include <algorithm>
#include <cstdint>

#include "../../include/cg.h"

namespace cg {

namespace {

bool intersects(const std::vector<int>& a, const std::vector<int>& b) {
  for (int x : a)
    for (int y : b)
      if (x == y) return true;
  return false;
}

struct Access {
  const std::vector<std::vector<int>>& rd;
  const std::vector<std::vector<int>>& wr;
  const std::vector<char>& ws;
  // a conflict forbids swapping a and b
  bool conflict(int a, int b) const {
    return intersects(wr[a], rd[b]) || intersects(rd[a], wr[b]) || intersects(wr[a], wr[b]) || (ws[a] && ws[b]);
  }
  bool reads_output_of(int a, int b) const { return intersects(rd[a], wr[b]); }
};

void flush(const Access& A, const std::vector<char>& coll, std::vector<int>& pending,
           std::vector<std::vector<int>>& out) {
  while (!pending.empty()) {
    // every collective that may move to the front of what is still pending:
    // no conflict with any pending group before it (those moved with it included)
    std::vector<int> batch, rest;
    for (size_t i = 0; i < pending.size(); ++i) {
      const int c = pending[i];
      bool front = coll[c];
      for (size_t j = 0; front && j < i; ++j) front = !A.conflict(c, pending[j]);
      (front ? batch : rest).push_back(c);
    }
    if (batch.empty()) {  // pending[0] is not a collective: issue it alone
      out.push_back({pending[0]});
      pending.erase(pending.begin());
    } else {
      out.push_back(batch);
      pending = rest;
    }
  }
}

}  // namespace

std::vector<std::vector<int>> collective_schedule(const std::vector<char>& active,
                                                  const std::vector<std::vector<int>>& rd,
                                                  const std::vector<std::vector<int>>& wr,
                                                  const std::vector<char>& ws,
                                                  const std::vector<char>& coll) {
  const Access A{rd, wr, ws};
  std::vector<std::vector<int>> out;
  std::vector<int> pending;
  for (int g = 0; g < (int)active.size(); ++g) {
    if (!active[g]) continue;
    bool depends = false, conflicts = false;
    for (int p : pending) {
      depends = depends || A.reads_output_of(g, p);
      conflicts = conflicts || A.conflict(g, p);
    }
    if (coll[g] || depends) {
      pending.push_back(g);  // relative order among the deferred groups is kept
    } else if (conflicts) {
      flush(A, coll, pending, out);
      out.push_back({g});
    } else {
      out.push_back({g});
    }
  }
  flush(A, coll, pending, out);
  return out;
}

}  // namespace cg

// Test hook (declared in include/cg.h): the schedule of synthetic access sets in
// CSR form.  rd_ptr/wr_ptr have ng+1 entries.  Writes order[k] (group ids in issue
// order) and step[k] (equal step ids = one collective batch); returns the number of
// scheduled groups.
extern "C" int32_t cgx_collective_schedule(int32_t ng, const uint8_t* active, const int32_t* rd_ptr,
                                           const int32_t* rd_idx, const int32_t* wr_ptr, const int32_t* wr_idx,
                                           const uint8_t* uses_ws, const uint8_t* is_coll, int32_t* order,
                                           int32_t* step) {
  if (ng < 0) return CG_E_ARG;
  std::vector<char> act(ng), ws(ng), coll(ng);
  std::vector<std::vector<int>> rd(ng), wr(ng);
  for (int g = 0; g < ng; ++g) {
    act[g] = active ? (char)active[g] : 1;
    ws[g] = (char)uses_ws[g];
    coll[g] = (char)is_coll[g];
    rd[g].assign(rd_idx + rd_ptr[g], rd_idx + rd_ptr[g + 1]);
    wr[g].assign(wr_idx + wr_ptr[g], wr_idx + wr_ptr[g + 1]);
  }
  auto steps = cg::collective_schedule(act, rd, wr, ws, coll);
  int k = 0;
  for (size_t s = 0; s < steps.size(); ++s)
    for (int g : steps[s]) {
      order[k] = g;
      step[k] = (int32_t)s;
      ++k;
    }
  return k;
}
