// mp_layer_impl.h -- internal host-side declarations shared by layer.cu and
// formats.cpp (file readers written fresh, format-compatible with the
// reference's MPEX container inc/io.hpp:210-251 and NDJSON partition map
// inc/serde.hpp:100-168).
#pragma once

#include <cstdint>
#include <string>
#include <vector>

namespace mp {

// Thrown by the readers; status code mirrors inc/error.hpp (1 validation, 2 io).
struct Failure {
    int code;
    std::string msg;
};

struct MpexData {
    uint32_t d_model = 0, d_ff = 0;
    std::vector<float> w_gate, w_up, w_down;
};

struct PartitionDocHost {
    uint64_t expert_id = 0;
    uint32_t n_subexperts = 0;
    std::vector<uint32_t> assignment;
    bool has_gates = false;
    uint32_t r = 0;
    std::vector<std::vector<uint32_t>> gates;
};

// load_toy_expert (inc/io.hpp:225-251) semantics: IoError when the file cannot
// be opened; ValidationError on bad magic / version / truncation / trailing
// bytes / empty dims / non-finite weights.  Throws Failure.
MpexData read_mpex(const std::string& path);
// read_ndjson (inc/serde.hpp:135-151) + partition_doc_from_json (:113-124) +
// gate_set_from_json (:160-168) when "r"/"gates" are present.
std::vector<PartitionDocHost> read_partition_map(const std::string& path);
// validate(Partition), inc/partition.hpp:34-46.  Throws Failure.
void validate_partition(uint32_t n_sub, const uint32_t* assignment, size_t n);
// MPAM activation matrices (inc/io.hpp:147-200, binary format).  Throws Failure.
void write_mpam(const std::string& path, uint32_t rows, uint32_t cols, const float* data);
std::vector<float> read_mpam(const std::string& path, uint32_t& rows, uint32_t& cols);

}  // namespace mp
