// Test infrastructure (oracle/): a bag of named byte arrays handed across a
// flat C ABI so that Python (ctypes) can read checker outputs without knowing
// any C++ types.  Used by ref_capi.cpp (the compiled reference) and by
// oracle64.cpp (our restatement).  Never linked into the product library.
#pragma once

#include <cstdint>
#include <cstring>
#include <map>
#include <string>
#include <vector>

namespace oracle_bundle {

struct Bundle {
    std::map<std::string, std::vector<std::uint8_t>> arrays;
    std::string error;  // non-empty when the call raised
    int status = 0;     // 0 ok, 1 invalid_argument, 2 overflow_error, 3 runtime_error, 4 other

    template <typename T>
    void put(const std::string& name, const std::vector<T>& v) {
        std::vector<std::uint8_t>& dst = arrays[name];
        dst.resize(v.size() * sizeof(T));
        if (!v.empty()) std::memcpy(dst.data(), v.data(), dst.size());
    }
    template <typename T>
    void put_scalar(const std::string& name, T x) {
        put(name, std::vector<T>{x});
    }
};

}  // namespace oracle_bundle

// Accessors are emitted once per library with a distinct prefix so both checker
// libraries can live in one process.
#define ORACLE_BUNDLE_EXPORTS(PREFIX)                                                     \
    extern "C" int PREFIX##_bundle_get(void* b, const char* name, const void** data,     \
                                       std::uint64_t* nbytes) {                           \
        auto* bb = static_cast<oracle_bundle::Bundle*>(b);                                \
        auto it = bb->arrays.find(name);                                                  \
        if (it == bb->arrays.end()) return -1;                                            \
        *data = it->second.data();                                                        \
        *nbytes = it->second.size();                                                      \
        return 0;                                                                         \
    }                                                                                     \
    extern "C" int PREFIX##_bundle_status(void* b) {                                      \
        return static_cast<oracle_bundle::Bundle*>(b)->status;                            \
    }                                                                                     \
    extern "C" const char* PREFIX##_bundle_error(void* b) {                               \
        return static_cast<oracle_bundle::Bundle*>(b)->error.c_str();                     \
    }                                                                                     \
    extern "C" int PREFIX##_bundle_names(void* b, char* out, int cap) {                   \
        std::string s;                                                                    \
        for (auto& kv : static_cast<oracle_bundle::Bundle*>(b)->arrays) {                 \
            s += kv.first;                                                                \
            s += ',';                                                                     \
        }                                                                                 \
        std::snprintf(out, static_cast<std::size_t>(cap), "%s", s.c_str());               \
        return static_cast<int>(s.size());                                                \
    }                                                                                     \
    extern "C" void PREFIX##_bundle_free(void* b) { delete static_cast<oracle_bundle::Bundle*>(b); }
