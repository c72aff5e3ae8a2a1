// MUGVCKPT container (proj/include/mugv/params.hpp:54-61, proj/src/params.cpp:92-225): host-side reader
// and writer behind the mgv_ckpt_* C ABI.  Byte-stable writer (same bytes as mugv::save_checkpoint for the
// same ParameterSet) and a validating reader with the reference's CheckpointError taxonomy.
#pragma once
#include <cstdint>
#include <map>
#include <stdexcept>
#include <string>
#include <vector>

namespace mgv {

struct CheckpointError : std::runtime_error {
    enum Kind { BadMagic = 0, Truncated = 1, BadHeader = 2, BadOffsets = 3, Io = 4 };  // errors.hpp:43
    Kind kind;
    CheckpointError(Kind k, const std::string& m) : std::runtime_error(m), kind(k) {}
};
// InputError of save_checkpoint (reserved "__meta__" name, params.cpp:93); mapped to MGV_ERR_INPUT
struct CkptInputError : std::runtime_error {
    using std::runtime_error::runtime_error;
};

enum CkptDtype { kF32 = 0, kF64 = 1 };  // params.hpp:14 (Dtype::f32, Dtype::f64)

struct CkptEntry {
    std::string name;
    CkptDtype dtype = kF64;
    std::vector<int64_t> shape;
    int64_t numel = 1;
    uint64_t offset = 0;  // into the payload
};

// A loaded checkpoint: the file bytes stay resident, entries point into the payload (little-endian).
struct Checkpoint {
    std::string raw;                          // whole file
    uint64_t payload_at = 0;                  // 16 + header length
    std::vector<CkptEntry> entries;           // sorted by name (ParameterSet order)
    std::map<std::string, std::string> meta;  // "__meta__"
    const unsigned char* payload(const CkptEntry& e) const {
        return reinterpret_cast<const unsigned char*>(raw.data()) + payload_at + e.offset;
    }
    void read_f64(const CkptEntry& e, double* out) const;  // widen f32 payloads, copy f64
    void read_f32(const CkptEntry& e, float* out) const;   // f32 payloads bit-exact; f64 rounded
};

Checkpoint load_checkpoint(const std::string& path);

struct CkptTensorIn {
    std::string name;
    CkptDtype dtype;
    std::vector<int64_t> shape;
    const double* f64 = nullptr;  // exactly one of f64 / f32 is set
    const float* f32 = nullptr;
};
void save_checkpoint(std::vector<CkptTensorIn> tensors, const std::map<std::string, std::string>& meta,
                     const std::string& path);

// records a CheckpointError for mgv_ckpt_last_error / _kind (C ABI entry points outside ckpt.cpp)
void note_ckpt_error(const std::string& msg, int kind);

}  // namespace mgv

struct mgv_ckpt {
    mgv::Checkpoint ck;
};
