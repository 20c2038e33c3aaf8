// Multi-GPU dispatch of the C-ABI entry points (uwb_multi.cu).
#pragma once

#include "../../include/uwb_nli.h"
#include "uwb_ctx.cuh"

namespace uwb {

int multi_all_channels_nli(uwb_ctx* m, const uwb_grid* grid, int n_spans, const uwb_span* spans,
                           const double beta[3], const double* gamma, const uwb_nli_cfg* cfg,
                           uwb_nli_result* out);
int multi_prepare(uwb_ctx* m, const uwb_grid* grid, const uwb_fibre* fibre, const uwb_link_cfg* link,
                  const uwb_nli_cfg* cfg, bool with_batch);
int multi_evaluate_link(uwb_ctx* m, const uwb_grid* grid, const uwb_fibre* fibre,
                        const uwb_link_cfg* link, const uwb_nli_cfg* cfg, uwb_link_report* out);
int multi_resident(uwb_ctx* m, const double* psd_dev, double* report_dev, void* stream);
int multi_many(uwb_ctx* m, int n_eval, const double* psd_host, double* loss_host,
               double* report_host);
int multi_status(uwb_ctx* m);

}  // namespace uwb
