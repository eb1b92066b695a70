/*
 * roomsim_oracle.h — TEST INFRASTRUCTURE ONLY.
 *
 * A plain-C restatement of the reference algorithm for the hot path
 * (image-method RIR -> -eta dB tail cut -> planner -> radix-2 real FFT
 * overlap-add -> SPEC mixer).  It is the CHECKER for the CUDA product path:
 * only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load it.  The product library never links it.
 *
 * Pinning: tests/test_oracle_pin.py checks every function here against
 * (a) the SPEC.md known-answer examples and (b) the reference itself,
 * compiled from /root/reference by oracle/Makefile into oracle/_ref/
 * (see oracle/ref_driver.cpp).  RIR taps, cut indices, plans and the FFT
 * are required to match the reference bit for bit.
 */
#ifndef ROOMSIM_ORACLE_H_
#define ROOMSIM_ORACLE_H_

#include <stddef.h>
#include <stdint.h>

#include "../include/roomsim_gpu.h"

#ifdef __cplusplus
extern "C" {
#endif

const char* orc_last_error(void);

/* room_model.hpp:67-71 */
size_t orc_virtual_source_count(int image_order);
/* room_model.hpp:109-134: writes (2K+1)^3 positions [v*3] and reflection counts. */
int orc_enumerate_images(const double room[3], double refl, double fs, double c0, int order,
                         const double src[3], double* pos, int* refl_count, size_t cap);
/* room_model.hpp:141-174 (+ optional horizon cut to max_taps, harness). */
int orc_synthesize_rir(const double room[3], double refl, double fs, double c0, int order,
                       const double src[3], const double mic[3], int64_t max_taps,
                       double* out, size_t cap, size_t* len);
/* room_model.hpp:177-213 */
int orc_power_threshold(const double* h, size_t n, double eta_db, double* p_th);
int orc_cutoff_index(const double* h, size_t n, double threshold, size_t* n_c);
int orc_truncate_rir(const double* h, size_t n, double eta_db, size_t* keep, size_t* n_c,
                     double* p_th);

/* convolution.hpp:72-161 */
double orc_cost_direct(double I, double J, size_t nx, size_t nh);
double orc_cost_full_fft(double I, double J, size_t nx, size_t nh, size_t n);
double orc_cost_ola(double I, double J, size_t nx, size_t nh, size_t n);
size_t orc_ola_block_count(size_t nx, size_t nh, size_t n);
int orc_plan_for(double I, double J, size_t nx, size_t nh, int strategy, int* s_out,
                 size_t* n_out, double* cost_out);
int orc_choose_plan(double I, double J, size_t nx, size_t nh, int* s_out, size_t* n_out,
                    double* cost_out);

/* fft.hpp:57-169 (RadixTwoRealFft); spectrum interleaved re,im [n/2+1]. */
int orc_rfft_forward(size_t n, const double* in, double* out);
int orc_rfft_inverse(size_t n, const double* in, double* out);

/* convolution.hpp:164-271 */
int orc_convolve_direct(const double* x, size_t nx, const double* h, size_t nh, double* out);
int orc_convolve_full_fft(const double* x, size_t nx, const double* h, size_t nh, double* out);
int orc_convolve_ola(const double* x, size_t nx, const double* h, size_t nh, size_t n,
                     double* out);

/* audio_buffer.hpp:66-75 */
int orc_mean_power(const double* v, size_t n, double* p);
/* SPEC.md:338-346 */
int orc_compute_gain(double p_target, double p_noise, double snr_db, double* alpha);

/* SPEC.md:348-356 render over a scene batch (same layout as the product
 * ABI).  Output in FP64 (the reference's AudioBuffer precision).
 * `pair_out`, if non-NULL, receives each reverberant pair signal at
 * pair_out + pair_off[p] (caller sizes it). `threads` <= 1: sequential.   */
int orc_render_batch(const rs_scene_batch* b, double* out, const int64_t* out_off,
                     const int64_t* out_stride, int64_t* out_len, rs_pair_layout* layout,
                     double* gains, double* power, int threads);

#ifdef __cplusplus
}
#endif
#endif
