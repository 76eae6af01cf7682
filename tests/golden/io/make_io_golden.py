"""Generate tests/golden/io/ with the UNMODIFIED reference (oracle/_ref/io_ref,
minopt/io.hpp): files written by the reference's write_optd / write_optg,
malformed files, and the reference's verdict on reading each one
(verdicts.json).  Run here (needs /root/reference); the fixtures travel."""
import json
import os
import struct
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
IO_REF = os.path.join(HERE, "..", "..", "..", "oracle", "_ref", "io_ref")


def ref(*args):
    r = subprocess.run([IO_REF, *map(str, args)], capture_output=True, text=True)
    return r.stdout.strip()


def main():
    files = {}
    # reference-written arrays / graphs
    for name, args in {"f64_2d_c3.optd": (1, 3, 5, 4), "f32_2d_c1.optd": (0, 1, 7, 3),
                       "f32_3d_c2.optd": (0, 2, 2, 3, 4), "f64_0d_c4.optd": (1, 4),
                       "f64_empty.optd": (1, 2, 0, 5)}.items():
        ref("write_optd", os.path.join(HERE, name), *args)
        files[name] = {"written_by": "reference write_optd", "args": list(args)}
    for name, args in {"edges2.optg": (2, 9), "edges3.optg": (3, 4), "empty.optg": (1, 0)}.items():
        ref("write_optg", os.path.join(HERE, name), *args)
        files[name] = {"written_by": "reference write_optg", "args": list(args)}
    # malformed files
    good = open(os.path.join(HERE, "f64_2d_c3.optd"), "rb").read()
    bad = {
        "bad_magic.optd": b"OPTX" + good[4:],
        "bad_version.optd": good[:4] + struct.pack("<I", 2) + good[8:],
        "bad_dtype.optd": good[:8] + bytes([7]) + good[9:],
        "zero_channels.optd": good[:10] + struct.pack("<H", 0) + good[12:],
        "truncated_header.optd": good[:15],
        "truncated_payload.optd": good[:-3],
        "long_payload.optd": good + b"\0" * 8,
        "empty_file.optd": b"",
        "huge_extent.optd": good[:12] + struct.pack("<Q", (1 << 40) + 1) + good[20:],
    }
    g = open(os.path.join(HERE, "edges2.optg"), "rb").read()
    bad.update({
        "bad_magic.optg": b"OPTD" + g[4:],
        "bad_version.optg": g[:4] + struct.pack("<I", 9) + g[8:],
        "zero_arity.optg": g[:8] + struct.pack("<H", 0) + g[10:],
        "truncated.optg": g[:-1],
        "long.optg": g + b"\0" * 8,
        "empty_file.optg": b"",
    })
    for name, data in bad.items():
        with open(os.path.join(HERE, name), "wb") as f:
            f.write(data)
        files[name] = {"written_by": "make_io_golden.py (malformed)"}
    for name in files:
        cmd = "read_optd" if name.endswith(".optd") else "read_optg"
        files[name]["reference_read"] = ref(cmd, os.path.join(HERE, name))
    with open(os.path.join(HERE, "verdicts.json"), "w") as f:
        json.dump(files, f, indent=1, sort_keys=True)


if __name__ == "__main__":
    main()
