// pipeline.cuh — host side of the training-data pipeline (pipeline.cu).
#pragma once
#include <map>
#include <string>
#include <vector>

#include "common.cuh"

namespace moses {

unsigned long long epoch_seed(unsigned long long seed, unsigned long long epoch);
// make_ranking_batches (data.cpp:128-164) as row indices; returns the batch count.
// rows_out: n entries; boff: n_batches + 1; btask: n_batches (any may be null).
long long ranking_plan(const int* record_task, long long n, const char* const* task_ids, int n_ids, int batch,
                       unsigned long long seed, long long* rows_out, long long* boff, int* btask, long long* dropped);
// sample_replay_features' rows (data.cpp:166-183); returns min(n_records, size)
long long replay_rows(long long n_records, long long size, unsigned long long seed, long long* rows_out);

// A record store as flat arrays (data.hpp RecordStore / MeasurementRecord).
struct Records {
  std::vector<std::string> task_ids, device_ids;  // first-appearance order
  std::map<std::string, int> task_ix, device_ix;
  std::vector<int> task, device;
  std::vector<long long> value_off{0}, values;
  std::vector<double> throughput, latency, wall_cost;
  std::vector<unsigned long long> seq;

  long long size() const { return (long long)task.size(); }
  void parse_line(const std::string& line, const std::string& origin);  // record_from_json_line
  std::string line(long long i) const;                                   // record_to_json_line
  static Records* read(const char* path);                                // read_records
  void write(const char* path) const;                                    // write_records
};

}  // namespace moses
