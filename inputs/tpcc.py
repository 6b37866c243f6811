"""TPC-C inputs: the row layout (a specification shared by the oracle and the device
library, each implementing it independently) and the seeded initial population S0.

TPC-C is the paper's second benchmark (NewOrder and Payment); the
initial population follows TPC-C §4.3.3 (SURVEY.md §8(c) "Initial population"):
per warehouse 10 districts, 3,000 customers per district, 100,000 stock rows; 100,000
items; W_YTD = 300,000.00, D_YTD = 30,000.00, D_NEXT_O_ID = 3001, C_BALANCE = -10.00,
C_YTD_PAYMENT = 10.00, C_PAYMENT_CNT = 1, 10% "BC" credit, S_QUANTITY in [10,100],
I_PRICE in [1.00,100.00], 10% of I_DATA / S_DATA contain "ORIGINAL", c_last of customers
1..1000 from the syllable table applied to c_id-1, the rest NURand(255,0,999).
Money is i64 cents; rates are u32 in 1/10,000.

Every random field is mix64(seed ^ (table << 56) ^ (row << 8) ^ field) ("prand"), so the
device loader can produce the same bytes; tests assert equality.

Row layouts (u64 words, little-endian; strings are bytes, zero padded):
  WAREHOUSE 16 w: 0 w_ytd | 1 w_tax (lo32) | 2-3 w_name[16] (10 letters) | 4-15 filler
  DISTRICT  16 w: 0 d_ytd | 1 d_tax (lo32), d_next_o_id (hi32) | 2-3 d_name[16] | 4-15 filler
  CUSTOMER  88 w: 0 c_balance | 1 c_ytd_payment | 2 c_payment_cnt (lo32), c_delivery_cnt (hi32)
                  | 3 c_discount (lo32), c_credit (hi32: b'BC' or b'GC' in bytes 4-5)
                  | 4-5 c_last[16] | 6-7 c_first[16] | 8-24 filler | 25-87 c_data[504]
  STOCK     40 w: 0 s_quantity (lo32), s_order_cnt (hi32) | 1 s_ytd | 2 s_remote_cnt (lo32)
                  | 3-32 s_dist_01..10 (24 B each) | 33-39 s_data[56] (50 letters)
  ITEM      12 w: 0 i_price (lo32), i_im_id (hi32) | 1-3 i_name[24] | 4-10 i_data[56] | 11 filler
  ORDER      8 w: o_id, d, w, c_id, entry_d, ol_cnt, all_local, 0       (reserved slot per txn)
  NEW_ORDER  4 w: o_id, d, w, 0                                         (reserved slot per txn)
  ORDER_LINE 8 w: 0 o_id (lo32) | number (hi32), 1 d (lo32) | w (hi32), 2 i_id (lo32) |
                  supply_w (hi32), 3 qty, 4 amount, 5-7 dist_info[24]   (15 slots per txn)
  HISTORY    8 w: 0 c_id (lo32) | c_d (hi32), 1 c_w (lo32) | d (hi32), 2 w, 3 date,
                  4 amount, 5-7 h_data[24] = w_name[10] + 4 spaces + d_name[10]
Ids inside rows are 1-based TPC-C ids (w_id 1..W, d_id 1..10, c_id 1..3000, i_id
1..100000); row ordinals are 0-based:  district row = w*10 + d, customer row =
(w*10 + d)*3000 + c, stock row = w*100000 + i  (w, d, c, i 0-based).
"""
from __future__ import annotations

import numpy as np

from .ycsb import mix64

W_WORDS, D_WORDS, C_WORDS, S_WORDS, I_WORDS = 16, 16, 88, 40, 12
O_WORDS, NO_WORDS, OL_WORDS, H_WORDS = 8, 4, 8, 8
DIST, CUST, STOCK_PER_W, ITEMS, MAX_OL = 10, 3000, 100000, 100000, 15
T_W, T_D, T_C, T_S, T_I, T_CONST = 1, 2, 3, 4, 5, 15
SYLLABLES = [b"BAR", b"OUGHT", b"ABLE", b"PRI", b"PRES", b"ESE", b"ANTI", b"CALLY", b"ATION", b"EING"]
C_DATA_OFF = 25          # word offset of c_data in CUSTOMER
C_DATA_BYTES = 504       # reading: c_data is 504 bytes (63 words) so the BC shift is word aligned


def prand(seed, table, row, field):
    """mix64(seed ^ (table << 56) ^ (row << 8) ^ field), vectorised over row/field."""
    row = np.asarray(row, dtype=np.uint64)
    field = np.asarray(field, dtype=np.uint64)
    with np.errstate(over="ignore"):
        x = (np.uint64(seed) ^ (np.uint64(table) << np.uint64(56)) ^ (row << np.uint64(8)) ^ field)
    return mix64(x)


def nurand_consts(seed):
    """NURand C constants (TPC-C §2.1.6), fixed per run: (C_LAST load, C_LAST run,
    C_ID, C_OL_I_ID)."""
    c = [int(prand(seed, T_CONST, 0, k)) for k in range(4)]
    c_load = c[0] % 256
    c_run = (c_load + 65 + c[1] % 55) % 256    # |C_run - C_load| in [65, 119] (TPC-C §2.1.6.1)
    return c_load, c_run, c[2] % 1024, c[3] % 8192


def _letters(seed, table, rows, field0, n):
    """(len(rows), n) uint8 uppercase letters from prand words (8 letters per word)."""
    nw = (n + 7) // 8
    w = prand(seed, table, np.asarray(rows, np.uint64)[:, None], np.uint64(field0) + np.arange(nw, dtype=np.uint64)[None, :])
    b = w.view(np.uint8).reshape(len(rows), nw * 8)[:, :n]
    return (b % 26 + ord("A")).astype(np.uint8)


def last_name(num: int) -> bytes:
    return SYLLABLES[num // 100] + SYLLABLES[(num // 10) % 10] + SYLLABLES[num % 10]


def _put_bytes(words: np.ndarray, w0: int, data: np.ndarray):
    """write a (n, k) uint8 array into word columns starting at w0 (zero padded)."""
    n, k = data.shape
    nw = (k + 7) // 8
    buf = np.zeros((n, nw * 8), np.uint8)
    buf[:, :k] = data
    words[:, w0:w0 + nw] = buf.view(np.uint64).reshape(n, nw)


def _with_original(seed, table, rows, field, data):
    """10% of rows contain b"ORIGINAL" at a random offset of the 50 letters."""
    r = prand(seed, table, rows, field)
    has = (r % np.uint64(10)) == 0
    off = ((r >> np.uint64(8)) % np.uint64(43)).astype(np.int64)
    orig = np.frombuffer(b"ORIGINAL", np.uint8)
    idx = np.nonzero(has)[0]
    data[idx[:, None], off[idx][:, None] + np.arange(8)[None, :]] = orig[None, :]
    return data


def warehouse_rows(seed, W, first=0):
    rows = np.arange(first, first + W, dtype=np.uint64)
    out = np.zeros((len(rows), W_WORDS), np.uint64)
    out[:, 0] = 30000000                                       # 300,000.00
    out[:, 1] = prand(seed, T_W, rows, 1) % np.uint64(2001)    # w_tax 0..0.2000
    _put_bytes(out, 2, _letters(seed, T_W, rows, 16, 10))
    out[:, 4:16] = prand(seed, T_W, rows[:, None], np.arange(32, 44, dtype=np.uint64)[None, :])
    return out


def district_rows(seed, W, first_w=0):
    rows = np.arange(first_w * DIST, (first_w + W) * DIST, dtype=np.uint64)
    out = np.zeros((len(rows), D_WORDS), np.uint64)
    out[:, 0] = 3000000                                        # 30,000.00
    out[:, 1] = (prand(seed, T_D, rows, 1) % np.uint64(2001)) | (np.uint64(3001) << np.uint64(32))
    _put_bytes(out, 2, _letters(seed, T_D, rows, 16, 10))
    out[:, 4:16] = prand(seed, T_D, rows[:, None], np.arange(32, 44, dtype=np.uint64)[None, :])
    return out


def customer_last_nums(seed, rows):
    """c_last number in [0, 999] of customer rows (row = (w*10+d)*3000 + c)."""
    c_load = nurand_consts(seed)[0]
    rows = np.asarray(rows, np.uint64)
    c = (rows % np.uint64(CUST)).astype(np.int64)    # 0-based c
    a = (prand(seed, T_C, rows, 5) % np.uint64(256)).astype(np.int64)
    b = ((prand(seed, T_C, rows, 6)) % np.uint64(1000)).astype(np.int64)
    nur = (((a | b) + c_load) % 1000)
    return np.where(c < 1000, c, nur)


def customer_rows(seed, W, first_w=0):
    rows = np.arange(first_w * DIST * CUST, (first_w + W) * DIST * CUST, dtype=np.uint64)
    n = len(rows)
    out = np.zeros((n, C_WORDS), np.uint64)
    out[:, 0] = np.uint64((1 << 64) - 1000)                    # -10.00 as two's complement
    out[:, 1] = 1000
    out[:, 2] = 1
    bc = (prand(seed, T_C, rows, 2) % np.uint64(10)) == 0
    credit = np.where(bc, np.uint64(0x4342), np.uint64(0x4347))   # b"BC" / b"GC" little-endian
    out[:, 3] = (prand(seed, T_C, rows, 3) % np.uint64(5001)) | (credit << np.uint64(32))
    lasts = customer_last_nums(seed, rows)
    table = np.zeros((1000, 16), np.uint8)
    for k in range(1000):
        nm = last_name(k)
        table[k, :len(nm)] = np.frombuffer(nm, np.uint8)
    _put_bytes(out, 4, table[lasts])
    first = _letters(seed, T_C, rows, 16, 16)
    flen = 8 + (prand(seed, T_C, rows, 4) % np.uint64(9)).astype(np.int64)   # 8..16 letters
    first[np.arange(16)[None, :] >= flen[:, None]] = 0
    _put_bytes(out, 6, first)
    out[:, 8:25] = prand(seed, T_C, rows[:, None], np.arange(64, 81, dtype=np.uint64)[None, :])
    cdata = np.zeros((n, C_DATA_BYTES), np.uint8)
    cdata[:, :500] = _letters(seed, T_C, rows, 128, 500)
    _put_bytes(out, C_DATA_OFF, cdata)
    return out


def stock_rows(seed, W, first_w=0):
    rows = np.arange(first_w * STOCK_PER_W, (first_w + W) * STOCK_PER_W, dtype=np.uint64)
    n = len(rows)
    out = np.zeros((n, S_WORDS), np.uint64)
    out[:, 0] = 10 + prand(seed, T_S, rows, 1) % np.uint64(91)       # s_quantity 10..100
    _put_bytes(out, 3, _letters(seed, T_S, rows, 16, 240))
    data = _letters(seed, T_S, rows, 64, 50)
    data = _with_original(seed, T_S, rows, 2, data)
    _put_bytes(out, 33, data)
    return out


def item_rows(seed):
    rows = np.arange(ITEMS, dtype=np.uint64)
    out = np.zeros((ITEMS, I_WORDS), np.uint64)
    price = 100 + prand(seed, T_I, rows, 1) % np.uint64(9901)        # 1.00 .. 100.00
    im = 1 + prand(seed, T_I, rows, 3) % np.uint64(10000)
    out[:, 0] = price | (im << np.uint64(32))
    _put_bytes(out, 1, _letters(seed, T_I, rows, 16, 24))
    data = _letters(seed, T_I, rows, 64, 50)
    data = _with_original(seed, T_I, rows, 2, data)
    _put_bytes(out, 4, data)
    out[:, 11] = prand(seed, T_I, rows, 200)
    return out


def population(seed, W):
    """Full S0 as a dict of (rows, words) uint64 arrays for W warehouses."""
    return {"warehouse": warehouse_rows(seed, W), "district": district_rows(seed, W),
            "customer": customer_rows(seed, W), "stock": stock_rows(seed, W), "item": item_rows(seed)}
