"""CPU oracle for the probe-streaming hot path.

TEST INFRASTRUCTURE ONLY.  Nothing in ``paper_2103_05875_b200`` imports this
package.  Only ``tests/``, ``__graft_entry__.smoke()`` and the
``cpu_baseline`` / ``--impl reference`` legs of ``bench.py`` may import it,
and only as the checker or as the timed CPU baseline -- never as the thing
measured or shipped.

Contents
--------
``stream_ops``  numpy restatement of the reference's change detection,
                budgeted selection, slot cache, update-atlas build, plane
                packing and the codec's temporal-delta/SKIP rule
                (``/root/reference/pkg/src/probestream/{selection,packing,
                codec}.py``).  Bit-exact targets.  Pinned against golden
                vectors produced by the reference itself
                (``tests/golden/make_golden.py``).
``ddgi``        float32 numpy restatement of the probe update (ray set,
                shading, irradiance / depth-moment blend, hysteresis,
                quantisation, guard band).  The reference has NO
                implementation of this stage: its pieces that
                do exist (fibonacci_sphere, oct_decode, texel centres, guard
                band rule, texel formats) are pinned against reference
                fixtures; the DDGI arithmetic itself is "parity unpinned".
``raycast.c``   C restatement of ``SceneGeometry.raycast`` for triangles
                (double precision brute force), the traversal oracle.
"""
