/*
 * synth/synth_host.c -- seeded synthetic webcam-frame generator (host side).
 *
 * Input generator only: it holds none of the method's arithmetic (no luma, no
 * envelope, no hue, no morphology).  It is shared by the oracle-side tests and
 * the GPU-side tests/bench; synth/synth_dev.cu implements the identical integer
 * recipe on the device and tests/test_synth.py checks both byte for byte.
 *
 * Recipe: a static textured background in non-skin
 * hues (16x16 cells of gray / blue / green / teal, plus a diagonal texture),
 * optional static skin-hued clutter ellipses, a skin-coloured disc "hand" with
 * an optional arm rectangle to the bottom edge, per-pixel sensor noise from a
 * counter-based hash, then a per-frame Q10 exposure gain with saturation.
 * Everything is integer; per-frame geometry and gains are computed by the
 * caller (synth/configs.py, double + round-half-up) and passed in as data.
 */
#include <stdint.h>
#include <stddef.h>

static inline uint64_t sy_mix64(uint64_t z)
{
    z += 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

/* per-frame parameter block: 8 int32 per frame */
enum { SY_FRAME_ID = 0, SY_GAIN_Q10, SY_CX, SY_CY, SY_R, SY_ARM_W, SY_PF_STRIDE = 8 };

static inline void sy_background(uint64_t bgseed, int x, int y, int tex, int *rgb)
{
    uint64_t hc = sy_mix64(bgseed ^ (((uint64_t)(uint32_t)(y >> 4) << 32) | (uint32_t)(x >> 4)));
    uint32_t k = (uint32_t)(hc % 4u);
    uint32_t h1 = (uint32_t)(hc >> 8), h2 = (uint32_t)(hc >> 24), h3 = (uint32_t)(hc >> 40);
    switch (k) {
    case 0: { int v = 80 + (int)(h1 % 50u); rgb[0] = v; rgb[1] = v; rgb[2] = v; break; }
    case 1: rgb[0] = 50 + (int)(h1 % 30u); rgb[1] = 80 + (int)(h2 % 30u); rgb[2] = 150 + (int)(h3 % 40u); break;
    case 2: rgb[0] = 60 + (int)(h1 % 30u); rgb[1] = 130 + (int)(h2 % 40u); rgb[2] = 70 + (int)(h3 % 30u); break;
    default: rgb[0] = 90 + (int)(h1 % 20u); rgb[1] = 110 + (int)(h2 % 20u); rgb[2] = 120 + (int)(h3 % 20u); break;
    }
    rgb[0] += tex; rgb[1] += tex; rgb[2] += tex;
}

void synth_frames(uint32_t W, uint32_t H, uint64_t seed, uint32_t stream, uint32_t noise_a,
                  uint32_t n, const int32_t *pf, uint32_t n_ell, const int32_t *ell,
                  uint8_t *out)
{
    uint64_t bgseed = sy_mix64(seed ^ 0xB6B6B6B6ull ^ ((uint64_t)stream << 40));
    uint64_t nseed = sy_mix64(seed ^ ((uint64_t)stream * 0x9E3779B97F4A7C15ull));
    uint32_t span = 2u * noise_a + 1u;
    for (uint32_t f = 0; f < n; f++) {
        const int32_t *P = pf + (size_t)f * SY_PF_STRIDE;
        uint64_t fseed = sy_mix64(nseed ^ (uint64_t)(uint32_t)P[SY_FRAME_ID]);
        int64_t cx = P[SY_CX], cy = P[SY_CY], R = P[SY_R], armw = P[SY_ARM_W];
        uint32_t gain = (uint32_t)P[SY_GAIN_Q10];
        uint8_t *o = out + (size_t)f * W * H * 3;
        for (uint32_t y = 0; y < H; y++) {
            for (uint32_t x = 0; x < W; x++) {
                int tex = (int)((x * 7u + y * 3u) & 15u) - 8;
                int rgb[3];
                sy_background(bgseed, (int)x, (int)y, tex, rgb);
                for (uint32_t e = 0; e < n_ell; e++) {
                    int64_t ex = ell[4 * e], ey = ell[4 * e + 1], ea = ell[4 * e + 2], eb = ell[4 * e + 3];
                    int64_t dx = (int64_t)x - ex, dy = (int64_t)y - ey;
                    if (eb * eb * dx * dx + ea * ea * dy * dy <= ea * ea * eb * eb) {
                        rgb[0] = 150 + tex; rgb[1] = 90 + tex; rgb[2] = 80 + tex;
                        break;
                    }
                }
                if (R > 0) {
                    int64_t dx = (int64_t)x - cx, dy = (int64_t)y - cy;
                    int in_disc = dx * dx + dy * dy <= R * R;
                    int in_arm = armw > 0 && (int64_t)y >= cy && 2 * (dx < 0 ? -dx : dx) <= armw;
                    if (in_disc || in_arm) { rgb[0] = 210; rgb[1] = 120; rgb[2] = 110; }
                }
                uint64_t h = sy_mix64(fseed ^ (((uint64_t)y << 32) | x));
                for (int c = 0; c < 3; c++) {
                    int nz = noise_a ? (int)((uint32_t)((h >> (16 * c)) & 0xFFFFu) % span) - (int)noise_a : 0;
                    int v = rgb[c] + nz;
                    v = v < 0 ? 0 : (v > 255 ? 255 : v);
                    uint32_t g = ((uint32_t)v * gain + 512u) >> 10;
                    o[((size_t)y * W + x) * 3 + c] = (uint8_t)(g > 255u ? 255u : g);
                }
            }
        }
    }
}
