"""Weighted deficit round robin dispatch of layer payloads (oracle; test infrastructure only).

Alg. A2, line 6: "Hold per-request rates stable for this epoch."  Line 7:
"Dispatch layer payloads with weighted deficit round robin."  Sec. 3.6: the rates
r_i hold for the whole KV load of a request admitted in an epoch.

Deficit round robin is the textbook scheduler of Shreedhar & Varghese (SIGCOMM 1995): every
backlogged flow i has a quantum q_i and a deficit counter D_i (initially 0).  A round visits the
backlogged flows in order; a visited flow adds q_i to D_i, then sends packets from its head while
the head packet's size is <= D_i, subtracting each size from D_i; a flow whose queue empties
sets D_i = 0 and leaves the round.  "Weighted": q_i is proportional to the flow's weight.

Readings:
  c21  flow = one request's copy units in layer-major order (layer 0 of every chunk, in prefix
       order, then layer 1, ...), so each request's layers still complete in order; packet = one
       unit (bytes = its rows * row bytes); weight = the epoch rate r_i; the lightest request's
       quantum is Q and q_i = floor(Q * r_i / min_j r_j) -- the textbook condition Q >= the
       largest packet makes every visit send at least one packet.  Q defaults to
       max(256 KiB, largest packet) (c16: 256 KiB).  Finer than the paper's
       whole-layer payloads; the byte shares are the same (the fairness bound below).
  c22  hold rates: request i's units are released no earlier than t0 + (bytes of request i
       dispatched before them) / r_i; a dispatched run is released at the max of that and the
       previous run's release, so releases are monotone along the dispatch order.  Release
       times are whole microseconds, floor(bytes * 1e6 / r_i).  With a hot-layer mirror (c24)
       a request's first free_i packets are read from HBM, not over the paced link: they are
       not counted in its bytes (and so are released at t0, subject to the monotone max).
  c25  mirrored packets are not link traffic, so DRR does not schedule them: with free_i given,
       every flow's first free_i packets are dispatched first (flow 0's, then flow 1's, ...,
       split into entries of E), then DRR runs over the remaining packets of every flow.  With
       hold rates the front entries are all released at t0 -- the mirror's layers land at HBM
       speed for every request of the batch, not one DRR round at a time.

The dispatch order is returned as runs (flow, first packet, count); `entries` splits the runs
into claim entries of at most E packets, the granularity at which copy CTAs take work.

Two packet granularities:
  plan                 c21: packet = one copy unit (the library's default planner)
  layer_payload_plan   Alg. A2 line 7 literally ("Dispatch layer payloads"): packet =
                       one request's whole layer-l payload, N_i*S bytes; quantum default
                       max(256 KiB, largest layer payload) so every visit sends.  The packet
                       order is expanded into the request's units of that layer (layer-major,
                       chunk j, then tile) so both plans name the same claimable work.
"""
import math


def quanta(weights, Q):
    """c21: q_i = floor(Q * w_i / min_j w_j) (>= Q for every flow)."""
    if not weights:
        return []
    if any(not (w > 0) or math.isinf(w) for w in weights):
        raise ValueError("weights must be finite and > 0")
    wmin = min(weights)
    return [int(math.floor(Q * w / wmin)) for w in weights]


def default_quantum(max_packet):
    """c21/c16: 256 KiB unless a packet is larger."""
    return max(256 * 1024, max_packet)


def drr_order(sizes, q):
    """Deficit round robin over flows with packet sizes `sizes[i]` (a list per flow) and quanta
    q[i].  Returns the dispatch order as a list of (flow, packet index)."""
    n = len(sizes)
    deficit = [0] * n
    head = [0] * n
    active = [i for i in range(n) if len(sizes[i]) > 0]
    order = []
    while active:
        still = []
        for i in active:
            deficit[i] += q[i]
            while head[i] < len(sizes[i]) and sizes[i][head[i]] <= deficit[i]:
                deficit[i] -= sizes[i][head[i]]
                order.append((i, head[i]))
                head[i] += 1
            if head[i] == len(sizes[i]):
                deficit[i] = 0
            else:
                still.append(i)
        active = still
    return order


def runs(order):
    """Run-length form of a dispatch order: [(flow, first packet, count)]."""
    out = []
    for f, p in order:
        if out and out[-1][0] == f and out[-1][1] + out[-1][2] == p:
            out[-1] = (f, out[-1][1], out[-1][2] + 1)
        else:
            out.append((f, p, 1))
    return out


def entries(rs, E):
    """Split runs into claim entries of at most E packets, in order."""
    out = []
    for f, first, cnt in rs:
        for k in range(0, cnt, E):
            out.append((f, first + k, min(E, cnt - k)))
    return out


def release_us(ents, sizes, rates, free=None):
    """c22: release time (whole us after t0) of every entry, monotone along the order.  free[f]:
    leading packets of flow f that do not count toward its rate (they never cross the paced link)."""
    out = []
    prev = 0
    for f, first, cnt in ents:
        fu = free[f] if free else 0
        paced_before = sum(sizes[f][fu:first]) if first > fu else 0
        t = int(math.floor(paced_before * 1e6 / rates[f]))
        prev = max(prev, t)
        out.append(prev)
    return out


def unit_sizes(n_chunks, L, tiles, tile_bytes):
    """Packet sizes of one request: layer-major units, unit u = tile u % tiles of a slice."""
    return [tile_bytes[u % tiles] for u in range(n_chunks * L * tiles)]


def plan(n_chunks, L, tiles, tile_bytes, weights, Q=0, E=8, rates=None, free=None):
    """The whole dispatch plan of a batch: claim entries (flow, first unit, count) and, when
    `rates` is given, their release times in us (c22)."""
    sizes = [unit_sizes(n, L, tiles, tile_bytes) for n in n_chunks]
    Qe = Q if Q else default_quantum(max(tile_bytes))
    if Qe < max(tile_bytes):
        raise ValueError("quantum below the largest packet")
    if not free:
        ents = entries(runs(drr_order(sizes, quanta(weights, Qe))), E)
    else:
        # c25: the free (mirrored) packets first, flow by flow; then DRR over the paced packets
        fu = [min(f, len(s)) for f, s in zip(free, sizes)]
        front = [(f, 0, fu[f]) for f in range(len(sizes)) if fu[f] > 0]
        rest = drr_order([s[k:] for s, k in zip(sizes, fu)], quanta(weights, Qe))
        ents = entries(front, E) + entries(runs([(f, p + fu[f]) for f, p in rest]), E)
    rel = release_us(ents, sizes, rates, free) if rates is not None else None
    return ents, rel


def layer_payload_sizes(n_chunks, L, tile_bytes):
    """Alg. A2 line 7 packets of one request: L layer payloads of N_i * S bytes (S = sum of the
    tiles of one chunk's layer slice).  A request with no chunks has no payloads at all (it never
    enters the layerwise pool), not L empty ones."""
    return [n_chunks * sum(tile_bytes)] * L if n_chunks else []


def layer_payload_plan(n_chunks, L, tiles, tile_bytes, weights, Q=0, E=8, rates=None, free_layers=None):
    """WDRR over whole layer payloads (Alg. A2 line 7).  DRR runs over packets = layers;
    each dispatched layer l of request i becomes its units [l*upl_i, (l+1)*upl_i), upl_i = N_i*tiles,
    in runs/entries as in `plan`.  free_layers[i] (mirrored layers, reading c25) go first, request
    by request.  Release times (c22) are per entry over the request's unit bytes, as in `plan`."""
    sizes = [layer_payload_sizes(n, L, tile_bytes) for n in n_chunks]
    Qe = Q if Q else default_quantum(max([max(s) for s in sizes if s], default=1))
    if Qe < max([max(s) for s in sizes if s], default=0):
        raise ValueError("quantum below the largest layer payload")
    upl = [n * tiles for n in n_chunks]
    fl = [min(f, L) for f in free_layers] if free_layers else [0] * len(n_chunks)
    front = [(f, 0, fl[f] * upl[f]) for f in range(len(n_chunks)) if fl[f] > 0 and upl[f] > 0]
    order = drr_order([s[k:] for s, k in zip(sizes, fl)], quanta(weights, Qe))
    unit_runs = runs([(f, p + fl[f]) for f, p in order])           # runs of layers
    unit_runs = [(f, first * upl[f], cnt * upl[f]) for f, first, cnt in unit_runs]
    ents = entries(front, E) + entries(unit_runs, E)
    rel = None
    if rates is not None:
        usz = [unit_sizes(n, L, tiles, tile_bytes) for n in n_chunks]
        rel = release_us(ents, usz, rates, [fl[f] * upl[f] for f in range(len(n_chunks))])
    return ents, rel


def bytes_by_flow_prefix(ents, unit_size_lists):
    """Byte-level view of a plan: for each entry boundary, (total bytes so far, per-flow bytes)."""
    n = len(unit_size_lists)
    per = [0] * n
    tot = 0
    out = [(0, tuple(per))]
    for f, first, cnt in ents:
        b = sum(unit_size_lists[f][first:first + cnt])
        per[f] += b
        tot += b
        out.append((tot, tuple(per)))
    return out
