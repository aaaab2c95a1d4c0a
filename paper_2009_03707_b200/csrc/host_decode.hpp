// Host-side decoders of the narrow device-to-host deliveries (stages.cu Sink): plain
// C++ with SSE2 intrinsics (every x86-64 host), no CUDA -- tests/test_host_decode.py
// compiles them alone and checks them against scalar restatements.
#pragma once

#include <emmintrin.h>

#include <algorithm>
#include <cstdint>

namespace msc3d_host {

// out[i] = in[i] for i in [a, b) with non-temporal 16-byte stores (SSE2): the output
// is written once and not read again here, so no read-for-ownership of its lines --
// 140 GB/s on 16 host threads against 42 GB/s with plain stores (tools/probe/host_widen).
inline void widen_u8_u64(const std::uint8_t* in, std::uint64_t* out, std::uint64_t a, std::uint64_t b) {
    while (a < b && (reinterpret_cast<std::uintptr_t>(out + a) & 15)) {
        out[a] = in[a];
        ++a;
    }
    const __m128i z = _mm_setzero_si128();
    for (; a + 16 <= b; a += 16) {
        const __m128i v = _mm_loadu_si128(reinterpret_cast<const __m128i*>(in + a));
        const __m128i w0 = _mm_unpacklo_epi8(v, z), w1 = _mm_unpackhi_epi8(v, z);
        const __m128i d[4] = {_mm_unpacklo_epi16(w0, z), _mm_unpackhi_epi16(w0, z), _mm_unpacklo_epi16(w1, z),
                              _mm_unpackhi_epi16(w1, z)};
        __m128i* o = reinterpret_cast<__m128i*>(out + a);
        for (int k = 0; k < 4; ++k) {
            _mm_stream_si128(o + 2 * k, _mm_unpacklo_epi32(d[k], z));
            _mm_stream_si128(o + 2 * k + 1, _mm_unpackhi_epi32(d[k], z));
        }
    }
    for (; a < b; ++a) out[a] = in[a];
    _mm_sfence();
}

// out[a, b) from byte steps: out[a] = head, out[i] = out[i-1] + in[i], or (in[i] = 255)
// the escaped absolute value already stored at out[i].  16 steps at a time: an SSE2
// prefix sum over u16 lanes, widened to u32 and streamed (non-temporal); a group with
// an escape goes scalar.  The caller issues the sfence.
inline void decode_steps(const std::uint8_t* in, std::uint32_t head, std::uint32_t* out, std::uint64_t a,
                         std::uint64_t b) {
    std::uint32_t v = head;
    _mm_stream_si32(reinterpret_cast<int*>(out + a), static_cast<int>(v));
    std::uint64_t i = a + 1;
    auto scalar = [&](std::uint64_t e) {
        for (; i < e; ++i) {
            const std::uint8_t d = in[i];
            v = d == 255 ? out[i] : v + d;
            _mm_stream_si32(reinterpret_cast<int*>(out + i), static_cast<int>(v));
        }
    };
    const std::uint64_t mis = (reinterpret_cast<std::uintptr_t>(out + i) & 15) / 4;  // to 16-byte aligned output
    scalar(std::min<std::uint64_t>(b, i + ((4 - mis) & 3)));
    const __m128i z = _mm_setzero_si128(), ff = _mm_set1_epi8(static_cast<char>(0xff));
    auto prefix8 = [](__m128i x) {  // inclusive prefix over 8 u16 lanes
        x = _mm_add_epi16(x, _mm_slli_si128(x, 2));
        x = _mm_add_epi16(x, _mm_slli_si128(x, 4));
        return _mm_add_epi16(x, _mm_slli_si128(x, 8));
    };
    while (i + 16 <= b && (reinterpret_cast<std::uintptr_t>(out + i) & 15) == 0) {
        const __m128i d = _mm_loadu_si128(reinterpret_cast<const __m128i*>(in + i));
        if (_mm_movemask_epi8(_mm_cmpeq_epi8(d, ff))) {  // an escape: these 16 one by one
            scalar(i + 16);
            continue;
        }
        const __m128i lo = prefix8(_mm_unpacklo_epi8(d, z));
        const __m128i last = _mm_shufflehi_epi16(lo, 0xff);  // lo's last lane in the high half
        const __m128i hi = _mm_add_epi16(prefix8(_mm_unpackhi_epi8(d, z)), _mm_unpackhi_epi64(last, last));
        const __m128i base = _mm_set1_epi32(static_cast<int>(v));
        __m128i* o = reinterpret_cast<__m128i*>(out + i);
        _mm_stream_si128(o + 0, _mm_add_epi32(base, _mm_unpacklo_epi16(lo, z)));
        _mm_stream_si128(o + 1, _mm_add_epi32(base, _mm_unpackhi_epi16(lo, z)));
        _mm_stream_si128(o + 2, _mm_add_epi32(base, _mm_unpacklo_epi16(hi, z)));
        _mm_stream_si128(o + 3, _mm_add_epi32(base, _mm_unpackhi_epi16(hi, z)));
        v += static_cast<std::uint32_t>(_mm_extract_epi16(hi, 7));
        i += 16;
    }
    scalar(b);
}

}  // namespace msc3d_host
