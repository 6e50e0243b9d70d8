// Launchers of the QEQEA generation kernels (kernels_qeqea.cu).
#pragma once
#include "engine_common.cuh"
#include "isq_internal.h"

namespace isq {

// world 1: prepare = sample + values; world > 1: prepare = sample + route,
// values = values of the received owned touches, score = unroute + fitness + elite.
isq_status qeqea_configure_device();  // kernel attributes, once per handle on its device
isq_status qeqea_launch_prepare(const QeqeaArgs& a, cudaStream_t s);
isq_status qeqea_launch_values(const QeqeaArgs& a, cudaStream_t s);
isq_status qeqea_launch_score(const QeqeaArgs& a, cudaStream_t s);
isq_status qeqea_launch_eval(const QeqeaArgs& a, cudaStream_t s);
isq_status qeqea_launch_finish(const QeqeaArgs& a, cudaStream_t s);
// Small single-rank populations: n generations in one single-block launch.
bool qeqea_small(const QeqeaArgs& a);
isq_status qeqea_launch_small(const QeqeaArgs& a, int n_gens, cudaStream_t s);
isq_status qeqea_launch_init(const QeqeaArgs& a, cudaStream_t s);
isq_status qeqea_launch_pack(const QeqeaArgs& a, double* theta, double* qamp, double* smax,
                             cudaStream_t s);
isq_status qeqea_launch_unpack(const QeqeaArgs& a, const double* theta, const double* qamp,
                               const double* smax, cudaStream_t s);
isq_status qeqea_launch_live(const QeqeaArgs& a, double* theta_out, double* q_out, cudaStream_t s);
isq_status qeqea_launch_sample(const QeqeaArgs& a, int64_t c0, int64_t c1, int64_t* flats,
                               uint8_t* codes, double* thetas, cudaStream_t s);

}  // namespace isq
