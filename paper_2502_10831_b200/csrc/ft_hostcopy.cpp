// ft_hostcopy.cpp -- host memory copy with non-temporal stores for the staged
// (pageable-buffer) host path.  The staged copies are large, written once and
// not read again by the CPU (the DMA engine or the caller reads them later), so
// write-allocating them through the caches costs a read-for-ownership of every
// destination line on top of the copy itself; streaming stores skip it.
// glibc's memcpy only switches to streaming stores above a per-thread threshold
// (~3/4 of the shared cache), which the pool's 4 MiB parts stay under.
// Compiled by the host compiler (no CUDA in this file).
#include <cstddef>
#include <cstdint>
#include <cstring>

#if defined(__x86_64__)
#include <immintrin.h>

namespace {

__attribute__((target("avx2"))) void copy_stream_avx2(char* d, const char* s, std::size_t n) {
  const std::size_t blocks = n / 128;
  for (std::size_t i = 0; i < blocks; ++i) {
    const __m256i a = _mm256_loadu_si256(reinterpret_cast<const __m256i*>(s));
    const __m256i b = _mm256_loadu_si256(reinterpret_cast<const __m256i*>(s + 32));
    const __m256i c = _mm256_loadu_si256(reinterpret_cast<const __m256i*>(s + 64));
    const __m256i e = _mm256_loadu_si256(reinterpret_cast<const __m256i*>(s + 96));
    _mm256_stream_si256(reinterpret_cast<__m256i*>(d), a);
    _mm256_stream_si256(reinterpret_cast<__m256i*>(d + 32), b);
    _mm256_stream_si256(reinterpret_cast<__m256i*>(d + 64), c);
    _mm256_stream_si256(reinterpret_cast<__m256i*>(d + 96), e);
    s += 128;
    d += 128;
  }
  _mm_sfence();
  std::memcpy(d, s, n - blocks * 128);
}

void copy_stream_sse2(char* d, const char* s, std::size_t n) {
  const std::size_t blocks = n / 64;
  for (std::size_t i = 0; i < blocks; ++i) {
    const __m128i a = _mm_loadu_si128(reinterpret_cast<const __m128i*>(s));
    const __m128i b = _mm_loadu_si128(reinterpret_cast<const __m128i*>(s + 16));
    const __m128i c = _mm_loadu_si128(reinterpret_cast<const __m128i*>(s + 32));
    const __m128i e = _mm_loadu_si128(reinterpret_cast<const __m128i*>(s + 48));
    _mm_stream_si128(reinterpret_cast<__m128i*>(d), a);
    _mm_stream_si128(reinterpret_cast<__m128i*>(d + 16), b);
    _mm_stream_si128(reinterpret_cast<__m128i*>(d + 32), c);
    _mm_stream_si128(reinterpret_cast<__m128i*>(d + 48), e);
    s += 64;
    d += 64;
  }
  _mm_sfence();
  std::memcpy(d, s, n - blocks * 64);
}

}  // namespace

extern "C" void ft_copy_stream(void* dst, const void* src, std::size_t n) {
  char* d = static_cast<char*>(dst);
  const char* s = static_cast<const char*>(src);
  if (n < (std::size_t(64) << 10)) {  // small: the cached copy is fine
    std::memcpy(d, s, n);
    return;
  }
  // streaming stores need an aligned destination: copy the head normally
  const std::size_t head = (64 - (reinterpret_cast<std::uintptr_t>(d) & 63)) & 63;
  std::memcpy(d, s, head);
  d += head;
  s += head;
  n -= head;
  static const bool avx2 = __builtin_cpu_supports("avx2");
  if (avx2) copy_stream_avx2(d, s, n);
  else copy_stream_sse2(d, s, n);
}

#else

extern "C" void ft_copy_stream(void* dst, const void* src, std::size_t n) { std::memcpy(dst, src, n); }

#endif
