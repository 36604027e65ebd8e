#include <algorithm>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <vector>

#include "prof.cuh"

namespace ttb {

namespace {
struct Rec {
  std::string name;
  cudaEvent_t a, b;
  cudaStream_t st;
};
std::mutex mu;
bool enabled = false;
std::vector<Rec> recs;
std::vector<Rec> open;
}  // namespace

bool prof_on() { return enabled; }

namespace {
std::vector<std::pair<std::string, double>> notes;
}

void prof_note(const char* name, double value) {
  std::lock_guard<std::mutex> lk(mu);
  if (enabled) notes.emplace_back(name, value);
}

void prof_record(const char* name, cudaStream_t st, bool begin) {
  std::lock_guard<std::mutex> lk(mu);
  cudaEvent_t e;
  cudaEventCreate(&e);
  cudaEventRecord(e, st);
  if (begin) {
    open.push_back(Rec{name, e, nullptr, st});
  } else {
    for (size_t i = open.size(); i-- > 0;) {
      if (open[i].name == name) {
        open[i].b = e;
        recs.push_back(open[i]);
        open.erase(open.begin() + (long)i);
        return;
      }
    }
    cudaEventDestroy(e);
  }
}

}  // namespace ttb

using namespace ttb;

extern "C" int ttb_prof_enable(int on) {
  std::lock_guard<std::mutex> lk(mu);
  enabled = on != 0;
  return TTB_OK;
}

// "name count total_ms\n" per kernel class, in first-seen order; clears.
extern "C" int ttb_prof_dump(char* buf, long long cap) {
  std::lock_guard<std::mutex> lk(mu);
  std::vector<std::string> order;
  std::map<std::string, std::pair<long long, double>> agg;
  // optional timeline (debugging): TTB_PROF_TIMELINE=<file>, one line per
  // scope "name start_ms end_ms stream" relative to the first scope
  if (const char* tl = getenv("TTB_PROF_TIMELINE")) {
    if (FILE* fp = fopen(tl, "w")) {
      for (auto& r : recs) {
        cudaEventSynchronize(r.b);
        float t0 = 0.f, t1 = 0.f;
        cudaEventElapsedTime(&t0, recs[0].a, r.a);
        cudaEventElapsedTime(&t1, recs[0].a, r.b);
        fprintf(fp, "%s %.4f %.4f %p\n", r.name.c_str(), t0, t1, (void*)r.st);
      }
      fclose(fp);
    }
  }
  for (auto& r : recs) {
    cudaEventSynchronize(r.b);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, r.a, r.b);
    if (!agg.count(r.name)) order.push_back(r.name);
    agg[r.name].first += 1;
    agg[r.name].second += ms;
    cudaEventDestroy(r.a);
    cudaEventDestroy(r.b);
  }
  recs.clear();
  for (auto& n : notes) {
    if (!agg.count(n.first)) order.push_back(n.first);
    agg[n.first].first += 1;
    agg[n.first].second += n.second;
  }
  notes.clear();
  std::string out;
  for (auto& n : order) {
    char line[256];
    snprintf(line, sizeof(line), "%s %lld %.6f\n", n.c_str(), agg[n].first, agg[n].second);
    out += line;
  }
  if (buf && cap > 0) {
    size_t n = std::min<size_t>(out.size(), (size_t)cap - 1);
    memcpy(buf, out.data(), n);
    buf[n] = 0;
  }
  return TTB_OK;
}
