/*
 * sfa_diag.h -- diagnostic entry points of libsfa_diag.so only (built with
 * -DSFA_STAMPS by `python -m paper_1405_0562_b200._build --diag`).  The
 * product library libsfa.so does not export them.
 *
 * sfa_diag_stamps -- after a TMA scan (sfa_match* >= 4 MiB, or a batch),
 * copies up to n stamps (8 per CTA, %globaltimer ns) to host: [0] kernel
 * entry, [1] tables built, [2] after griddepcontrol.wait, [3] thread 0's rows
 * scanned, [4] CTA folded, [5] epilogue done (last CTA), [7] producer's first
 * TMA issue.  Synchronises the device.
 */
#ifndef SFA_DIAG_H
#define SFA_DIAG_H
#include "sfa.h"
#ifdef __cplusplus
extern "C" {
#endif
SFA_API int sfa_diag_stamps(const sfa_handle* h, uint64_t* host, size_t n);
#ifdef __cplusplus
}
#endif
#endif
