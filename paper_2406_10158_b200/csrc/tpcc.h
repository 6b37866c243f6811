// tpcc.h -- TPC-C layout constants (inputs/tpcc.py docstring is the specification) and
// the workload parameters the executor receives.  Device library side only.
#pragma once
#include <cstdint>

namespace gcctb {

constexpr int TPCC_W_WORDS = 16, TPCC_D_WORDS = 16, TPCC_C_WORDS = 88, TPCC_S_WORDS = 40,
              TPCC_I_WORDS = 12, TPCC_O_WORDS = 8, TPCC_NO_WORDS = 4, TPCC_OL_WORDS = 8,
              TPCC_H_WORDS = 8;
constexpr uint32_t TPCC_DIST = 10, TPCC_CUST = 3000, TPCC_STOCK = 100000, TPCC_ITEMS = 100000,
                   TPCC_MAXOL = 15;
constexpr int TPCC_K = 18;               // access slots per transaction: W, D, C + 15 lines
constexpr int TPCC_OUT_WORDS = 48;       // read_out words per transaction
constexpr int TPCC_CDATA_OFF = 25, TPCC_CDATA_WORDS = 63;
constexpr int TPCC_TX_WORDS = 40;
enum { TPCC_T_W = 1, TPCC_T_D = 2, TPCC_T_C = 3, TPCC_T_S = 4, TPCC_T_I = 5, TPCC_T_CONST = 15 };
enum { TX_TYPE = 0, TX_W, TX_D, TX_CW, TX_CD, TX_C, TX_CLAST, TX_HAMT, TX_OLCNT, TX_ALLLOCAL,
       TX_ITEM = 10, TX_SUPQ = 25 };

struct TpccParams {
    const uint32_t *tx;                  // n_txn x 40 descriptors
    unsigned long long *wh, *di, *cu, *st;   // CC tables (local partition)
    const unsigned long long *it;        // items (immutable, replicated)
    unsigned long long *o, *no, *ol, *h; // reserved slots
    unsigned long long bW, bD, bC, bS;   // record-id bases of W, D, C, S
    uint32_t W;                          // total warehouses
    uint32_t w_first;                    // first warehouse held by this db
    const uint32_t *nidx_start, *nidx_count, *nidx_rows;   // last-name index
    unsigned long long entry_date;
};

}  // namespace gcctb

namespace gcctb {
// ---- warehouse-partitioned TPC-C ----
// One request per access of a distributed transaction, sent to the owner of the item.
struct PartReq {
    uint32_t gid;        // global transaction id (rank * n_local + local gid)
    uint32_t home;       // home rank (lo16) | access lane (hi16)
    uint32_t kind;       // 0 W, 1 D, 2 C, 3 S
    uint32_t row;        // local row on the owner (C by name: 0xFFFFFFFF)
    uint32_t type_d;     // txn type (bit0) | home district << 8 | remote-line flag << 16
    uint32_t amount;     // NewOrder line qty, or Payment h_amount
    uint32_t cust;       // by-name Payment: (c_w - w_first_owner) << 16 | c_d << 8 ... see pack
    uint32_t last;       // by-name c_last number, or 0xFFFFFFFF
    uint32_t c_ids;      // Payment customer: c_w (lo16) | c_d (hi16) (global ids, for the BC record)
    uint32_t home_w;     // home warehouse (global) | home district << 16
    uint32_t pad[2];
};
static_assert(sizeof(PartReq) == 48, "PartReq is 48 bytes");
// Response: the value read by the access at its point in the gid-ordered chain.
struct PartResp {
    unsigned long long v[6];
};
// CC_FLAG_PART_P2P: the peers' exchange windows (inbox, staging array, flags) as device
// pointers of this process (IPC-mapped, or local), indexed by rank
constexpr int P2P_MAXW = 64;
constexpr int P2P_FLAG_STRIDE = 32;   // one flag per 256 B
constexpr size_t P2P_FLAG_BYTES = (size_t)2 * P2P_MAXW * P2P_FLAG_STRIDE * 8;
struct PeerTab {
    PartReq *inbox[P2P_MAXW];
    PartResp *stage[P2P_MAXW];
    unsigned long long *flags[P2P_MAXW];
};
}  // namespace gcctb
