/* libpng stand-in — TEST INFRASTRUCTURE ONLY (oracle/_ref).
 *
 * proj/src/image.cpp includes <png.h> (CMakeLists.txt:12); libpng's headers
 * are absent in this image.  Image I/O is outside the hot path (SURVEY.md
 * §2), so this header only lets image.cpp compile unmodified: creating a
 * read struct fails, and read_png then throws "png_create_read_struct
 * failed" exactly as it does when libpng cannot allocate. */
#pragma once
#include <csetjmp>
#include <cstdio>

typedef struct pvo_png_struct_stub* png_structp;
typedef struct pvo_png_info_stub* png_infop;
typedef unsigned char* png_bytep;
typedef png_structp* png_structpp;
typedef png_infop* png_infopp;

#define PNG_LIBPNG_VER_STRING "0.0.0-pvo-stub"
#define PNG_COLOR_MASK_COLOR 2

static inline png_structp png_create_read_struct(const char*, void*, void*, void*) { return nullptr; }
static inline png_infop png_create_info_struct(png_structp) { return nullptr; }
static inline void png_destroy_read_struct(png_structpp, png_infopp, png_infopp) {}
static inline std::jmp_buf& pvo_png_jmpbuf_stub() {
    static std::jmp_buf b;
    return b;
}
#define png_jmpbuf(png) (pvo_png_jmpbuf_stub())
static inline void png_init_io(png_structp, FILE*) {}
static inline void png_read_info(png_structp, png_infop) {}
static inline void png_set_strip_16(png_structp) {}
static inline void png_set_strip_alpha(png_structp) {}
static inline void png_set_palette_to_rgb(png_structp) {}
static inline void png_set_expand_gray_1_2_4_to_8(png_structp) {}
static inline int png_get_color_type(png_structp, png_infop) { return 0; }
static inline void png_set_rgb_to_gray_fixed(png_structp, int, int, int) {}
static inline void png_read_update_info(png_structp, png_infop) {}
static inline unsigned png_get_image_width(png_structp, png_infop) { return 0; }
static inline unsigned png_get_image_height(png_structp, png_infop) { return 0; }
static inline void png_read_image(png_structp, png_bytep*) {}
