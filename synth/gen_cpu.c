/* synth/gen_cpu.c — CPU twin of synth/gen.cu (same counter-based recipe).
 * Input generation only; lets the oracle legs of bench.py build multi-GB samples quickly. */
#include <stdint.h>

static inline uint64_t mix(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

void synth_cpu_fill_old(uint16_t* out, uint64_t n, int norm, uint64_t key_val, const uint16_t* table) {
  for (uint64_t i = 0; i < n; ++i) out[i] = norm ? (uint16_t)norm : table[mix(key_val ^ i) >> 48];
}

void synth_cpu_fill_new(const uint16_t* old, uint16_t* nw, uint64_t n, int mode, int active, uint64_t key_mask,
                        uint64_t thr, uint64_t key_pert, uint64_t key_row, uint64_t thr_row, uint64_t cols) {
  if (!cols) cols = 1;
  for (uint64_t i = 0; i < n; ++i) {
    int m = active && (mix(key_mask ^ i) >> 32) < thr;
    if (mode == 1) m = m && ((mix(key_row ^ (i / cols)) >> 32) < thr_row);
    uint16_t o = old[i];
    nw[i] = m ? (uint16_t)(o ^ (uint16_t)(1 + mix(key_pert ^ i) % 3)) : o;
  }
}

/* 8-bit elements (FP8 E4M3, f2) */
void synth_cpu_fill_old8(uint8_t* out, uint64_t n, int norm, uint64_t key_val, const uint8_t* table) {
  for (uint64_t i = 0; i < n; ++i) out[i] = norm ? (uint8_t)norm : table[mix(key_val ^ i) >> 48];
}

void synth_cpu_fill_new8(const uint8_t* old, uint8_t* nw, uint64_t n, int mode, int active, uint64_t key_mask,
                         uint64_t thr, uint64_t key_pert, uint64_t key_row, uint64_t thr_row, uint64_t cols) {
  if (!cols) cols = 1;
  for (uint64_t i = 0; i < n; ++i) {
    int m = active && (mix(key_mask ^ i) >> 32) < thr;
    if (mode == 1) m = m && ((mix(key_row ^ (i / cols)) >> 32) < thr_row);
    uint8_t o = old[i];
    nw[i] = m ? (uint8_t)(o ^ (uint8_t)(1 + mix(key_pert ^ i) % 3)) : o;
  }
}
