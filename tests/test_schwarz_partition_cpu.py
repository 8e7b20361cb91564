"""The partitioned Chebyshev-Schwarz smoother (k_schwarz.cu)
exchanges fixed ghost planes between z-slabs: the element boxes of a slab read
node planes az = N-2, N-1 of the layer below and az = 0 of the layer above,
and the ASM sum over an owned node visits box plane z = N+2 of the layer
below and z = 0, 1 of the layer above -- nothing else crosses a slab.  This
checks that claim by enumerating the box geometry (the box of
element e spans global nodes e*N-1 .. e*N+N+1, owner of node g is (g-1)//N)
for every order the kernels instantiate and several partitions."""
import pytest


def owner(g, N, ne):
    """(owner element, local index) of global node g, None for Dirichlet nodes (k_schwarz.cu owner1d_s)."""
    if g <= 0 or g >= N * ne:
        return None
    oe = (g - 1) // N
    return oe, (g - 1) - oe * N


@pytest.mark.parametrize("N", [2, 3, 4, 5, 7])
@pytest.mark.parametrize("Ez,nranks", [(8, 2), (8, 4), (6, 3), (4, 4), (8, 8), (16, 8)])
def test_box_reads_cross_one_layer_in_fixed_planes(N, Ez, nranks):
    for rank in range(nranks):
        z0, z1 = rank * Ez // nranks, (rank + 1) * Ez // nranks
        below, above = set(), set()
        for ez in range(z0, z1):
            for c in range(N + 3):  # box z index
                o = owner(ez * N + c - 1, N, Ez)
                if o is None:
                    continue
                oez, az = o
                if oez < z0:
                    assert oez == z0 - 1
                    below.add(az)
                elif oez >= z1:
                    assert oez == z1
                    above.add(az)
        assert below <= {N - 2, N - 1} and above <= {0}
        if rank > 0:
            assert below == {N - 2, N - 1}
        if rank + 1 < nranks:
            assert above == {0}


@pytest.mark.parametrize("N", [2, 3, 4, 5, 7])
@pytest.mark.parametrize("Ez,nranks", [(8, 2), (8, 4), (6, 3), (4, 4), (8, 8), (16, 8)])
def test_asm_sum_visits_fixed_neighbour_box_planes(N, Ez, nranks):
    for rank in range(nranks):
        z0, z1 = rank * Ez // nranks, (rank + 1) * Ez // nranks
        lo, hi = set(), set()
        for ez in range(z0, z1):
            for c in range(N):  # owned node planes of the element
                gz = ez * N + c + 1
                if gz >= N * Ez:
                    continue
                for cz in range(gz // N - 2, gz // N + 2):  # k_asm_gather's candidate range
                    if cz < 0 or cz >= Ez or not (cz * N - 1 <= gz <= cz * N + N + 1):
                        continue
                    lc = gz - cz * N + 1
                    if cz < z0:
                        assert cz == z0 - 1
                        lo.add(lc)
                    elif cz >= z1:
                        assert cz == z1
                        hi.add(lc)
        assert lo <= {N + 2} and hi <= {0, 1}
        if rank > 0:
            assert lo == {N + 2}
        if rank + 1 < nranks:
            assert hi == {0, 1}


@pytest.mark.parametrize("N", [2, 3, 4, 5, 7])
def test_asm_candidate_range_is_complete(N):
    """Every element whose box covers node g lies in k_asm_gather's window g//N-2 .. g//N+1."""
    Ez = 6
    for gz in range(1, N * Ez):
        covering = {cz for cz in range(Ez) if cz * N - 1 <= gz <= cz * N + N + 1}
        window = {cz for cz in range(gz // N - 2, gz // N + 2) if 0 <= cz < Ez}
        assert covering <= window
