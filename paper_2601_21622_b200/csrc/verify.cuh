// verify.cuh -- internal layout shared by the verify kernels and the C-ABI dispatcher.
#pragma once
#include <cstddef>
#include <cstdint>
#include <cstdlib>
#include <vector_types.h>

namespace sd {

constexpr int kThreads = 256;            // threads per CTA (8 warps)
constexpr int kWarps = kThreads / 32;
constexpr int kVecBytes = 16;            // one 128-bit smem/global vector per thread per tile
constexpr int kTileBytes = kThreads * kVecBytes;   // 4 KB of one row per tile
constexpr int kMaxChunkBytes = 16 * 1024;          // one CTA owns <= 16 KB of a row ...
// ... except greedy fp32 rows (p only): 32 KB slices, 6 CTAs per SM by shared memory (measured:
// c3g 54.1 -> 45.8 us; sampled and bf16 rows are faster at 16 KB, profiles/README.md r02)
__host__ __device__ constexpr int rs_chunk_bytes(bool greedy, int esz) {
    return greedy && esz == 4 ? 2 * kMaxChunkBytes : kMaxChunkBytes;
}
constexpr int kRowClusterDefault = 8;              // see row_cluster()
constexpr int kMaxTagNch = 64;                     // tagged partials: rows of at most 64 chunks

// status bits (values of include/starsd.h SD_FAULT_*)
constexpr int32_t kBadId = 1, kNonfinite = 2, kEmptyRow = 4, kZeroQ = 8, kZeroResidual = 16,
                  kProtocol = 32;
constexpr int32_t kHard = kBadId | kNonfinite | kEmptyRow | kProtocol;

// Per (request b, position j, vocab chunk c): what one kernel-A CTA found in its slice.
struct PartA {
    double S_p, S_q;     // sum over the slice of 2^(z c2 - D_c), c2 = log2(e)/T (fp64 across threads)
    float M_p, M_q;      // sampled: slice's scaled max D_c = max fl(z_max c2); greedy: raw max
    float zx_p, zx_q;    // z_p,j(x_j), z_q,j(x_j) if x_j lies in this slice
    int32_t flags;       // kPartNonfiniteP | kPartNonfiniteQ | kPartHasX
    int32_t argmax;      // greedy: lowest index of the slice max (global token id)
};
constexpr int32_t kPartNonfiniteP = 1, kPartNonfiniteQ = 2, kPartHasX = 4, kPartSkipped = 8;

// Per (request b, position j): the whole-row statistics, written by the CTA that decides the row,
// read by the sampler and by sd_verify_trace.
struct RowStat {
    double S_p, S_q;     // row sums of 2^(z c2 - D) (same scale as PartA)
    double a;            // p_j(x_j) / q_j(x_j) as the decision used it (not clamped to 1); NaN if
                         // no test was evaluated (bonus row, faults, q_j(x_j) = 0)
    float M_p, M_q;      // sampled: scaled row maxima D = max fl(z_max c2); greedy: raw max of p
    int32_t status;      // SD_FAULT_* bits decided at this position
    int32_t argmax;      // greedy: argmax of p row (lowest index)
};

// Per (request b, position j) draft-row metadata (NEXT-1 / NEXT-2; include/starsd.h sd_qmeta):
// the draft row's statistics in the verify kernels' own arithmetic, so a verify that reads them
// instead of the q row takes bit-identical decisions.
struct QMeta {
    double S;            // sum of 2^(z c2 - D) over the row
    float D;             // scaled row max (greedy: raw max)
    float zx;            // z(x_j)
    int32_t status;      // kNonfinite / kEmptyRow of the q row
    int32_t reserved;
};

// Per (request b, chunk c) of the sampling pass.
struct PartB {
    double R;            // residual mass of the slice (or p mass at the bonus position)
    double P;            // p mass of the slice (zero-residual fallback, C-6)
};

struct Params {
    const void* p;
    const void* q;
    const int32_t* ids;
    int32_t B, k, V;
    int64_t ld_p, ld_q;          // elements
    int32_t nch;                 // vocab chunks per row
    int32_t CL;                  // k_row_stats cluster size (1: no cluster; chunk partials of a
                                 // cluster meet in its rank-0 CTA's shared memory)
    int32_t G;                   // row partials published to partA per row: ceil(nch / CL)
    int32_t CH;                  // elements per chunk (multiple of the tile)
    float c2;                    // log2(e) / T   (fp32; sampled path)
    double c2d;                  // the same value widened (exactly) to fp64
    uint64_t seed, round, rid_base;
    int32_t* out_L;
    int32_t* out_tok;
    int32_t* out_status;
    // workspace (zero-filled region first)
    unsigned long long* state;   // [B]  bits 0..k: position decided; bits 32+j: position j stopped
                                 //      the chain (rejection or fault).  The request is settled at
                                 //      L once positions 0..L are decided and L is the lowest stop
                                 //      (or L = k with no stop)
    uint32_t* ticketA;           // [B][k+1] row tickets (tagged rows: start order; else arrival)
    uint32_t* ticketB;           // [B]    sampling chunk tasks finished
    uint32_t* tailT;             // [B]    k_sample_chunked CTAs finished
    RowStat* rowstat;            // [B][k+1]
    PartA* partA;                // [B][k+1][nch]
    PartB* partB;                // [B][nch]
    double2* segtab;             // [B][nch][nseg]  (r mass, p mass) per warp segment
    double* rres;                // [B] mass R of the sampling distribution (trace)
    int32_t nseg;                // segments per chunk
    unsigned long long* trace;   // debug builds only (SD_STREAM_DEBUG): per-CTA phase timestamps
    unsigned long long* prof_ts; // sd_profile_timestamps: [2] this call's span words, or NULL
    // tagged partials (tagpub, rows of 2..kMaxTagNch chunks without clusters): every word of a
    // chunk partial carries the call's tag, so a CTA publishes with plain stores and exits; the
    // row's decider -- the CTA that took the row's last start ticket -- polls the words of the
    // others and decides (no fence; it only waits on CTAs that started before it)
    int32_t tagpub;
    uint32_t* epoch;             // [1]  workspace word 0: calls completed on this workspace
                                 //      (tag = (epoch + 1) | 2^31, never a small integer)
    unsigned long long* partT;   // [B][k+1][nch][5 * 2]  tag << 32 | 32 data bits
    int32_t chain;               // k_row_stats launched as a programmatic dependent of whatever
                                 // kernel precedes it on the stream (griddepcontrol.wait first)
    int32_t esz;                 // bytes per logit
    const QMeta* qmeta;          // [B][k] draft-row metadata: the q rows are then read only at the
                                 // stop position (sd_verify_qmeta); NULL: full q rows
    int32_t early;               // k_sample_req launched during k_row_stats' last position wave
    void* p_stage;               // sd_verify_staged: device copies of the rows k_row_stats reads
    void* q_stage;               // (the sampling kernels then read their stop rows from here)
    int32_t rgroup;              // k_row_stats grid: requests per group (grid order: group-major,
                                 // then position, request, chunk); B = one group (position-major)
};

// k_row_stats cluster size for a row of nch chunks: a cluster covers the whole row when nch <= 8
// (the smallest power of two >= nch; the grid's x extent is padded with empty chunks), so the
// row's partials meet in the leader's shared memory and no global ticket is taken.  Longer rows
// (nch > 8) measured faster without clusters (profiles/README.md).  STARSD_ROWCLUSTER=n caps the
// size (1 = the cluster-free kernel); a negative value -n forces clusters of n on every row
// (G = ceil(nch / n) cluster partials per row then meet through a global ticket).
inline int32_t row_cluster(int32_t nch) {
    static int env = 0;
    static bool read = false;
    if (!read) {
        const char* e = getenv("STARSD_ROWCLUSTER");
        env = e ? atoi(e) : 0;
        read = true;
    }
    if (env < 0) {
        const int f = -env;
        return (f == 2 || f == 4 || f == 8) ? (nch > 1 ? f : 1) : 1;
    }
    const int cap = (env == 1 || env == 2 || env == 4 || env == 8) ? env : kRowClusterDefault;
    const int32_t c = nch > 8 ? 1 : nch > 4 ? 8 : nch > 2 ? 4 : nch > 1 ? 2 : 1;
    return c < cap ? c : cap;
}

// Workspace layout for a shape; all offsets 16-byte aligned.  The first `zero_bytes` must be
// zero before a call and are zero again after it (word 0, the call counter, excepted).
struct WsLayout {
    size_t epoch, state, ticketA, ticketB, tailT, zero_bytes;
    size_t rowstat, partA, partB, segtab, rres, partT, total;
};

inline size_t align16(size_t x) { return (x + 15) & ~size_t(15); }

// (the workspace is laid out for the default 16 KB slices: the most chunks a row can have)
inline void chunking(int32_t V, int32_t esz, int32_t* nch, int32_t* CH,
                     int32_t chunk_bytes = kMaxChunkBytes) {
    const int64_t tile = kTileBytes / esz;                 // elements per tile
    const int64_t chmax = chunk_bytes / esz;
    int64_t n = (V + chmax - 1) / chmax;
    int64_t per = (V + n - 1) / n;
    int64_t ch = (per + tile - 1) / tile * tile;
    *nch = static_cast<int32_t>((V + ch - 1) / ch);
    *CH = static_cast<int32_t>(ch);
}

inline WsLayout ws_layout(int32_t B, int32_t k, int32_t V, int32_t esz) {
    int32_t nch, CH;
    chunking(V, esz, &nch, &CH);
    const int64_t nseg = CH / (32 * (kVecBytes / esz));   // 32-vector segments per chunk
    WsLayout w{};
    size_t o = 0;
    w.epoch = o;    o = align16(o + sizeof(uint32_t));   // fixed offset 0 for every shape
    w.state = o;    o = align16(o + sizeof(unsigned long long) * B);
    w.ticketA = o;  o = align16(o + sizeof(uint32_t) * (size_t)B * (k + 1));
    w.ticketB = o;  o = align16(o + sizeof(uint32_t) * B);
    w.tailT = o;    o = align16(o + sizeof(uint32_t) * B);
    w.zero_bytes = o;
    w.rowstat = o;  o = align16(o + sizeof(RowStat) * (size_t)B * (k + 1));
    w.partA = o;    o = align16(o + sizeof(PartA) * (size_t)B * (k + 1) * nch);
    w.partB = o;    o = align16(o + sizeof(PartB) * (size_t)B * nch);
    w.segtab = o;   o = align16(o + sizeof(double) * 2 * (size_t)B * nch * nseg);
    w.rres = o;     o = align16(o + sizeof(double) * (size_t)B);
    w.partT = o;
    if (nch >= 2 && nch <= kMaxTagNch) o = align16(o + 80 * (size_t)B * (k + 1) * nch);
    w.total = o;
    return w;
}

}  // namespace sd
