// frontier.cuh -- K-F: frontier rounds of the slot engine.
//
// Reference: the scatter branches of _push_u / _flush_v and the segmented
// arange _row_slots (pkg/src/bipush/push_engine.py:269-277, 297-302, 315-320),
// taken when the rows to push touch at most _SCATTER_LIMIT * |E| edges
// (push_engine.py:44, 297, 315).
//
// A dense round pulls every row of both sides: each V row sums its whole
// U-neighbourhood (K2), each U row its whole V-neighbourhood (K3), whatever the
// size of the pushed set A.  A frontier round visits only the rows that can be
// non-zero: the V rows N(A) of the pushed U rows (union over the block's
// slots), then the U rows N(N(A)).  Every visited row is still summed in full,
// in CSR order, so the value of a row does not depend on the round's mode; a
// row outside the frontier is zero, exactly what the dense pull would write.
//
//   K1   (k_push, kernels.cuh) writes one flag byte per U node: "some slot
//        pushed u"; each block adds its sum over slots of sum deg(A_s) to
//        FrontCtl::deg_acc, and the last block to arrive takes the decision:
//        frontier iff every busy slot is in a push round (no power-iteration
//        iterate, which is dense) and deg_acc <= limit (= _SCATTER_LIMIT * |E|).
//        It sets the batch graph's IF/ELSE condition (dense pulls in ELSE).
//   Fa   k_front_reset: XV / Y rows written non-zero by the previous frontier
//        round (its item lists) -- or every row, after dense rounds -- are
//        zeroed, and the row bitmaps cleared.
//   Fb   k_front_mark<SIDE_V>: the pushed U rows' edges are walked 32 at a
//        time by one warp each -- rows of more than FRONT_WALK edges as
//        host-cut pieces shared by several warps, the others one warp per row
//        from the flag bytes -- claiming each neighbour v in the V bitmap
//        (a test, then atomicOr: exactly one claimant per row) and appending
//        the claimed rows as work items.  Warp-aggregated allocation: each warp
//        reserves item slots in chunks of FRONT_ITEM_CHUNK (one atomicAdd per
//        chunk; unused slots become empty items), partial slots with one
//        atomicAdd per 32 edges, edge counts once per warp.  Degree binning on
//        the output side: a row of d edges becomes ceil(d / FRONT_CHUNK) items;
//        split rows publish fp64 partials and the last item to arrive adds them
//        in chunk order (deterministic), so hub rows do not serialise.
//   Fc   k_front_pull<SIDE_V>: XV rows of the V items, n_p partials per warp
//        (the dense pull's layout).  It also takes the U half's decision:
//        frontier iff sum deg(V list) <= limit (the reference's _flush_v test).
//   Fd   k_front_mark<SIDE_U>: walks the V items' edge ranges (in FRONT_WALK-
//        edge pieces) into the U bitmap / U items.
//   Fe   k_front_pull<SIDE_U>: Y rows of the U items.  When the U half is
//        dense, the dense U pull runs instead (gate_udense): XV is exact on
//        every row (zero outside the V list), so the dense pull is too.
//
// All kernels check their gate (FrontCtl::gate_*), so the same launch list
// works eagerly (BH_NO_GRAPH, round hooks, profiling) and under the graph's
// conditional node.
//
// Which runs compile the frontier in: blocks of up to 16 slots (single queries,
// small batches) whenever _SCATTER_LIMIT >= 0, wider blocks only when it forces
// frontier rounds (>= 1).  With 32+ slots in mixed phases the union of the pushed
// sets is dense in practically every round (one slot in power iteration makes it
// all of U; the reference itself takes the scatter branch in 2-13 % of a c2
// query's rounds), while the per-round decision -- K1's flags and arrival ticket,
// the IF/ELSE node, K1a without programmatic launch -- cost 8 % of the c2 step.
// Cost model: a dense round of a B-slot block costs a query
// (2E(i + s) / B + 2E s) bytes of gathers; a frontier round of one query
// f E (i + 2 s) for a frontier touching f E edges -- it pays for B = 1 when
// f < ~0.5, for a 128-slot block only when the union is nearly empty.
#pragma once

#include "kernels.cuh"

namespace bh {

constexpr int FRONT_CHUNK = 2048;  // edges per work item (longer rows are split)
constexpr int FRONT_WALK = 256;    // edges per claim walk (hub rows walked by several warps)

// A piece of a hub row's edges for the claim walk (host plan, static per graph).
struct FrontPiece {
    int64_t e0, e1;
    int32_t row, pad;
};

struct FrontItem {
    int64_t e0;          // first edge (CSR slot of the row's side)
    int32_t row, len;    // row, edges in this item
    int32_t part;        // partial slot of this chunk, -1: whole row
    int32_t first_part;  // first partial slot of the row (split rows)
    int32_t n_parts;     // items of the row
    int32_t pad;
};

// Start of a batch: every XV / Y row is stale, the statistics restart.  The item
// lists are kept: they name exactly the bitmap bits still set (cleared by the
// next frontier round's Fa), also across batches.
__global__ void k_front_begin(FrontCtl *f, int64_t limit) {
    f->deg_acc = 0;
    f->edges_v = f->edges_u = 0;
    f->limit = limit;
    f->rounds_front = f->rounds_ufront = 0;
    f->ticket = 0;
    f->mode = 0;
    f->gate_dense = f->gate_front = f->gate_ufront = f->gate_udense = 0;
    f->zero_all_v = f->zero_all_u = 1;
}

struct FrontArgs {
    FrontCtl *f;
    const int32_t *active;  // Control::active
    int B, elem_bytes;
    int64_t n_u, n_v, n_e;
    // U side (rows u, cols v) and V side (rows v, cols u), store order
    const int64_t *u_ptr, *v_ptr;
    const int32_t *u_col, *v_col;
    const uint8_t *flag_u;  // [n_u] K1: some slot pushed u
    const FrontPiece *hub_pieces;  // U rows of more than FRONT_WALK edges, cut into pieces
    int64_t n_hub_pieces;
    uint32_t *bits_v, *bits_u;
    FrontItem *items_v, *items_u;
    void *XV, *Y;           // [n][B] elements of elem_bytes
};

// Fa: zero the stale rows, clear the bitmaps.
__global__ void k_front_reset(FrontArgs a) {
    pdl_begin();
    FrontCtl *f = a.f;
    if (*a.active == 0 || !f->gate_front) return;
    const int lane = threadIdx.x & 31;
    const int64_t gw = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    const int64_t row_words = (int64_t)a.B * a.elem_bytes / 4;  // B * s is a multiple of 4
    auto zero_rows = [&](uint32_t *base, int64_t n_rows) {
        uint4 *p = reinterpret_cast<uint4 *>(base);
        const int64_t n16 = n_rows * row_words / 4;
        for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n16; i += (int64_t)gridDim.x * blockDim.x)
            p[i] = make_uint4(0, 0, 0, 0);
        const int64_t tail0 = n16 * 4;
        for (int64_t i = tail0 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n_rows * row_words;
             i += (int64_t)gridDim.x * blockDim.x)
            base[i] = 0u;
    };
    auto zero_listed = [&](uint32_t *base, uint32_t *bits, const FrontItem *items, int n_items, bool rows) {
        for (int64_t it = gw; it < n_items; it += nw) {
            const FrontItem w = items[it];
            if (w.row < 0 || (w.part >= 0 && w.part != w.first_part)) continue;  // empty / one item per row
            if (rows)
                for (int64_t j = lane; j < row_words; j += 32) base[(int64_t)w.row * row_words + j] = 0u;
            if (lane == 0) atomicAnd(&bits[w.row >> 5], ~(1u << (w.row & 31)));
        }
    };
    const bool all_v = f->zero_all_v, all_u = f->zero_all_u;
    if (all_v) zero_rows(reinterpret_cast<uint32_t *>(a.XV), a.n_v);
    if (all_u) zero_rows(reinterpret_cast<uint32_t *>(a.Y), a.n_u);
    zero_listed(reinterpret_cast<uint32_t *>(a.XV), a.bits_v, a.items_v, f->old_items_v, !all_v);
    zero_listed(reinterpret_cast<uint32_t *>(a.Y), a.bits_u, a.items_u, f->old_items_u, !all_u);
}

// Per-warp item allocator: item slots are reserved from the global counter in
// chunks (one atomicAdd per FRONT_ITEM_CHUNK items instead of one per 32
// edges -- every warp of the grid otherwise hammers one address: a forced c2
// round spent 5-7 ms in the V mark).  Unused slots of a chunk are written as
// empty items (row = -1), which the readers skip.  Values are warp-uniform.
constexpr int FRONT_ITEM_CHUNK = 64;
struct WarpAlloc {
    int32_t next = 0, end = 0;
    unsigned long long edges = 0;  // lane 31: edges of the rows this warp claimed
};

__device__ __forceinline__ void front_pad_empty(FrontItem *items, int32_t from, int32_t to) {
    const int lane = threadIdx.x & 31;
    for (int32_t i = from + lane; i < to; i += 32) {
        FrontItem w{};
        w.row = -1;
        items[i] = w;
    }
}

__device__ __forceinline__ void front_flush(WarpAlloc &al, FrontItem *items, unsigned long long *edges) {
    front_pad_empty(items, al.next, al.end);
    al.next = al.end;
    if ((threadIdx.x & 31) == 31 && al.edges) atomicAdd(edges, al.edges);
    al.edges = 0;
}

// Claims the other-side rows of edges [e0, e1) (one warp, all lanes) and
// appends the newly claimed rows as work items.
__device__ __forceinline__ void front_claim(int64_t e0, int64_t e1, const int32_t *__restrict__ col,
                                            const int64_t *__restrict__ dst_ptr, uint32_t *bits, FrontItem *items,
                                            int32_t *n_items, int32_t *n_parts, WarpAlloc &al) {
    const int lane = threadIdx.x & 31;
    for (int64_t base = e0; base < e1; base += 32) {
        const int64_t e = base + lane;
        int32_t c = -1;
        bool fresh = false;
        if (e < e1) {
            c = __ldg(col + e);
            const uint32_t bit = 1u << (c & 31);
            // test before the atomic: a claimed hub row is met by many walks at once
            if (!(__ldcg(&bits[c >> 5]) & bit)) fresh = !(atomicOr(&bits[c >> 5], bit) & bit);
        }
        const unsigned nb = __ballot_sync(0xffffffffu, fresh);
        if (!nb) continue;
        int64_t r0 = 0, d = 0;
        if (fresh) {
            r0 = __ldg(dst_ptr + c);
            d = __ldg(dst_ptr + c + 1) - r0;
        }
        const int n_it = fresh ? (int)((d + FRONT_CHUNK - 1) / FRONT_CHUNK) : 0;
        const int n_pt = n_it > 1 ? n_it : 0;
        // warp inclusive scans (items, partial slots) and the edge sum
        int s_it = n_it, s_pt = n_pt;
        unsigned long long s_d = (unsigned long long)d;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int a_it = __shfl_up_sync(0xffffffffu, s_it, o);
            const int a_pt = __shfl_up_sync(0xffffffffu, s_pt, o);
            if (lane >= o) {
                s_it += a_it;
                s_pt += a_pt;
            }
            s_d += __shfl_xor_sync(0xffffffffu, s_d, o);
        }
        const int tot_it = __shfl_sync(0xffffffffu, s_it, 31);
        if (al.next + tot_it > al.end) {  // new chunk (the rest of the old one becomes empty items)
            front_pad_empty(items, al.next, al.end);
            const int want = tot_it > FRONT_ITEM_CHUNK ? tot_it : FRONT_ITEM_CHUNK;
            int b = 0;
            if (lane == 0) b = atomicAdd(n_items, want);
            b = __shfl_sync(0xffffffffu, b, 0);
            al.next = b;
            al.end = b + want;
        }
        int b_pt = 0;
        if (lane == 31 && s_pt) b_pt = atomicAdd(n_parts, s_pt);
        b_pt = __shfl_sync(0xffffffffu, b_pt, 31);
        if (lane == 31) al.edges += s_d;
        if (fresh) {
            const int it0 = al.next + s_it - n_it;
            const int pt0 = b_pt + s_pt - n_pt;
            for (int k = 0; k < n_it; k++) {
                FrontItem w;
                w.e0 = r0 + (int64_t)k * FRONT_CHUNK;
                w.row = c;
                w.len = (int)(k + 1 < n_it ? FRONT_CHUNK : d - (int64_t)k * FRONT_CHUNK);
                w.part = n_pt ? pt0 + k : -1;
                w.first_part = n_pt ? pt0 : -1;
                w.n_parts = n_it;
                w.pad = 0;
                items[it0 + k] = w;
            }
        }
        al.next += tot_it;
    }
}

// Fb (SIDE_V): V rows of the pushed U nodes.  Fd (SIDE_U): U rows of the V items.
template <int SIDE>
__global__ void __launch_bounds__(256) k_front_mark(FrontArgs a) {
    pdl_begin();
    FrontCtl *f = a.f;
    if (*a.active == 0 || !(SIDE == SIDE_V ? f->gate_front : f->gate_ufront)) return;
    const int lane = threadIdx.x & 31;
    const int64_t gw = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    WarpAlloc al;
    if constexpr (SIDE == SIDE_V) {
        // hub rows (more than FRONT_WALK edges) as host-cut pieces, so several warps
        // share a hub's walk (degree binning: a c2 hub of ~5e4 edges walked by one warp
        // took 5-7 ms); then the other pushed rows, one warp per row
        for (int64_t p = gw; p < a.n_hub_pieces; p += nw) {
            const FrontPiece pc = a.hub_pieces[p];
            if (!a.flag_u[pc.row]) continue;
            front_claim(pc.e0, pc.e1, a.u_col, a.v_ptr, a.bits_v, a.items_v, &f->n_items_v, &f->n_parts_v, al);
        }
        for (int64_t base = gw * 32; base < a.n_u; base += nw * 32) {
            const int64_t u = base + lane;
            bool pushed = false;
            if (u < a.n_u && a.flag_u[u]) pushed = __ldg(a.u_ptr + u + 1) - __ldg(a.u_ptr + u) <= FRONT_WALK;
            unsigned m = __ballot_sync(0xffffffffu, pushed);
            while (m) {
                const int j = __ffs(m) - 1;
                m &= m - 1;
                const int64_t uu = base + j;
                front_claim(__ldg(a.u_ptr + uu), __ldg(a.u_ptr + uu + 1), a.u_col, a.v_ptr, a.bits_v, a.items_v,
                            &f->n_items_v, &f->n_parts_v, al);
            }
        }
        front_flush(al, a.items_v, &f->edges_v);
    } else {
        // the V items' edge ranges in FRONT_WALK-edge pieces (an item holds up to
        // FRONT_CHUNK edges)
        constexpr int PER = FRONT_CHUNK / FRONT_WALK;
        const int64_t n = (int64_t)f->n_items_v * PER;
        for (int64_t it = gw; it < n; it += nw) {
            const FrontItem w = a.items_v[it / PER];
            const int64_t b0 = w.e0 + (it % PER) * FRONT_WALK;
            const int64_t b1 = w.e0 + w.len < b0 + FRONT_WALK ? w.e0 + w.len : b0 + FRONT_WALK;
            if (w.row < 0 || b0 >= b1) continue;  // empty slot / past the item's end
            front_claim(b0, b1, a.v_col, a.u_ptr, a.bits_u, a.items_u, &f->n_items_u, &f->n_parts_u, al);
        }
        front_flush(al, a.items_u, &f->edges_u);
    }
}

template <typename T>
struct FrontPullArgs {
    FrontCtl *f;
    const int32_t *active;
    const int64_t *indptr;   // this side's rows
    const int32_t *indices;
    const T *vals;
    const FrontItem *items;
    const T *X;              // operand: P (V pull) or XV (U pull)
    T *Y;                    // XV (V pull) or Y (U pull)
    double *scratch;         // [parts][B]
    int32_t *pcnt;           // [parts], zero between launches
    const Slot *slots;
    int64_t *np_v;           // [n_warps][B] (V pull)
    int32_t n_warps;
    double scale;            // (1 - alpha) on the V side
};

// Fc / Fe: one warp per item.  B >= 32: lanes own VEC slots and walk the
// item's edges in order (32 (col, val) pairs per coalesced load, broadcast by
// shuffles, 4 operand rows in flight).  B < 32: 32 / B lane groups stride the
// edges, fixed shuffle tree.  fp64 accumulation either way.
template <int B, typename T, int SIDE>
__global__ void __launch_bounds__(PULL_THREADS) k_front_pull(FrontPullArgs<T> a) {
    pdl_begin();
    FrontCtl *f = a.f;
    if (SIDE == SIDE_V && blockIdx.x == 0 && threadIdx.x == 0 && *a.active && f->gate_front) {
        // the U half's decision (_flush_v's scatter test on sum deg(V list))
        const bool uf = f->edges_v <= (unsigned long long)f->limit;
        f->gate_ufront = uf;
        f->gate_udense = !uf;
        f->zero_all_u = !uf;
        f->zero_all_v = 0;
        if (uf) f->rounds_ufront++;
    }
    if (*a.active == 0 || !(SIDE == SIDE_V ? f->gate_front : f->gate_ufront)) return;
    const int lane = threadIdx.x & 31;
    const int gw = blockIdx.x * PULL_WARPS + (threadIdx.x >> 5);
    // the grid covers the dense plan's n_warps n_p rows; warps past them take no item
    const int nw = gridDim.x * PULL_WARPS < a.n_warps ? gridDim.x * PULL_WARPS : a.n_warps;
    const int n_items = gw < nw ? (SIDE == SIDE_V ? f->n_items_v : f->n_items_u) : 0;
    constexpr bool WIDE = B >= 32;
    constexpr int VEC = WIDE ? B / 32 : 1;
    constexpr int G = WIDE ? 32 : B, EPW = WIDE ? 1 : 32 / B;
    const int grp = WIDE ? 0 : lane / G;
    const int slot0 = WIDE ? lane * VEC : lane % G;
    uint32_t cmask = 0;
    if constexpr (SIDE == SIDE_V) {
#pragma unroll
        for (int v = 0; v < VEC; v++) cmask |= (op_is_push(a.slots[slot0 + v].op) ? 1u : 0u) << v;
    }
    int64_t np[VEC];
#pragma unroll
    for (int v = 0; v < VEC; v++) np[v] = 0;
    for (int it = gw; it < n_items; it += nw) {
        const FrontItem w = a.items[it];
        if (w.row < 0) continue;  // empty slot of an allocation chunk (warp-uniform)
        const int64_t e_end = w.e0 + w.len;
        double acc[VEC];
#pragma unroll
        for (int v = 0; v < VEC; v++) acc[v] = 0.0;
        if constexpr (WIDE) {
            for (int64_t base = w.e0; base < e_end; base += 32) {
                const int n = (int)(e_end - base < 32 ? e_end - base : 32);
                const int32_t cl = lane < n ? __ldg(a.indices + base + lane) : 0;
                const T vl = lane < n ? __ldg(a.vals + base + lane) : (T)0;
                for (int j = 0; j < n; j += 4) {
                    T xs[4][VEC];
                    T ws[4];
#pragma unroll
                    for (int k = 0; k < 4; k++) {
                        const int c = __shfl_sync(0xffffffffu, cl, (j + k) & 31);
                        ws[k] = __shfl_sync(0xffffffffu, vl, (j + k) & 31);
                        if (j + k < n) VecIO<T, VEC>::ld(a.X + (int64_t)c * B + slot0, xs[k]);
                    }
#pragma unroll
                    for (int k = 0; k < 4; k++)
                        if (j + k < n)
#pragma unroll
                            for (int v = 0; v < VEC; v++) acc[v] = fma((double)ws[k], (double)xs[k][v], acc[v]);
                }
            }
        } else {
            for (int64_t e = w.e0 + grp; e < e_end; e += EPW)
                acc[0] = fma((double)__ldg(a.vals + e), (double)a.X[(int64_t)__ldg(a.indices + e) * B + slot0], acc[0]);
#pragma unroll
            for (int off = G; off < 32; off <<= 1) acc[0] += __shfl_xor_sync(0xffffffffu, acc[0], off);
        }
        bool fin = w.part < 0;
        if (!fin) {  // split row: publish this chunk, the last chunk adds them in order
            if (WIDE || grp == 0)
#pragma unroll
                for (int v = 0; v < VEC; v++) a.scratch[(int64_t)w.part * B + slot0 + v] = acc[v];
            __threadfence();
            __syncwarp();
            int last = 0;
            if (lane == 0) last = atomicAdd(a.pcnt + w.first_part, 1) == w.n_parts - 1;
            last = __shfl_sync(0xffffffffu, last, 0);
            if (last) {
                __threadfence();
#pragma unroll
                for (int v = 0; v < VEC; v++) {
                    double t = 0.0;
                    for (int p = 0; p < w.n_parts; p++) t += __ldcg(a.scratch + (int64_t)(w.first_part + p) * B + slot0 + v);
                    acc[v] = t;
                }
                if (lane == 0) a.pcnt[w.first_part] = 0;
                fin = true;
            }
        }
        if (fin && (WIDE || grp == 0)) {
            const int64_t deg = __ldg(a.indptr + w.row + 1) - __ldg(a.indptr + w.row);
            T out[VEC];
#pragma unroll
            for (int v = 0; v < VEC; v++) {
                out[v] = (T)(a.scale * acc[v]);
                if constexpr (SIDE == SIDE_V)
                    if (((cmask >> v) & 1u) && (double)out[v] > 0.0) np[v] += deg;
            }
            if constexpr (WIDE) VecIO<T, VEC>::st(a.Y + (int64_t)w.row * B + slot0, out);
            else a.Y[(int64_t)w.row * B + slot0] = out[0];
        }
    }
    if constexpr (SIDE == SIDE_V) {
        if (gw < a.n_warps && (WIDE || grp == 0))
#pragma unroll
            for (int v = 0; v < VEC; v++) a.np_v[(int64_t)(slot0 + v) * a.n_warps + gw] = np[v];
    }
}

}  // namespace bh
