"""The reference's tests/test_dataio.py re-expressed against the drop-in
``dataio`` readers (IDX headers, native CSV parser) — CPU only
except the device loader at the end, which compares the streamed u8 -> f64 /
f32 device matrix with the host ``to_data_matrix``."""

import struct

import numpy as np
import pytest

from paper_2007_11919_b200 import FormatError
from paper_2007_11919_b200.dataio import read_csv_matrix, read_idx_images, read_idx_labels


def write_csv_matrix(matrix, path):
    """Test helper: headerless CSV with 17 significant digits (exact round trip)."""
    np.savetxt(path, np.asarray(matrix, dtype=np.float64), fmt="%.17g", delimiter=",")


def image_fixture_bytes():
    # two 2x2 images with hand-picked pixel values
    return struct.pack(">IIII", 0x00000803, 2, 2, 2) + bytes([0, 7, 255, 3, 10, 20, 30, 40])


class TestIdxImages:
    def test_hand_assembled_fixture(self, tmp_path):
        path = tmp_path / "img.idx"
        path.write_bytes(image_fixture_bytes())
        images = read_idx_images(path)
        assert images.count == 2 and images.height == 2 and images.width == 2
        m = images.to_data_matrix()
        assert m.dtype == np.float64 and m.shape == (2, 4)
        assert np.array_equal(m, [[0.0, 7.0, 255.0, 3.0], [10.0, 20.0, 30.0, 40.0]])

    def test_label_magic_rejected(self, tmp_path):
        path = tmp_path / "bad.idx"
        path.write_bytes(struct.pack(">IIII", 0x00000801, 2, 2, 2) + bytes(8))
        with pytest.raises(FormatError, match="magic"):
            read_idx_images(path)

    def test_truncated_payload_reports_counts(self, tmp_path):
        path = tmp_path / "short.idx"
        path.write_bytes(image_fixture_bytes()[:-3])
        with pytest.raises(FormatError, match="expected 24 bytes, got 21"):
            read_idx_images(path)

    def test_short_header(self, tmp_path):
        path = tmp_path / "tiny.idx"
        path.write_bytes(b"\x00\x00\x08")
        with pytest.raises(FormatError, match="too short"):
            read_idx_images(path)

    def test_zero_images(self, tmp_path):
        path = tmp_path / "empty.idx"
        path.write_bytes(struct.pack(">IIII", 0x00000803, 0, 28, 28))
        images = read_idx_images(path)
        assert images.count == 0 and images.to_data_matrix().shape == (0, 784)

    def test_missing_file(self, tmp_path):
        with pytest.raises(FileNotFoundError):
            read_idx_images(tmp_path / "nope.idx")


class TestIdxLabels:
    def test_fixture_values(self, tmp_path):
        path = tmp_path / "labels.idx"
        path.write_bytes(struct.pack(">II", 0x00000801, 3) + bytes([0, 1, 61]))
        assert np.array_equal(read_idx_labels(path), [0, 1, 61])

    def test_empty_file(self, tmp_path):
        path = tmp_path / "empty"
        path.write_bytes(b"")
        with pytest.raises(FormatError):
            read_idx_labels(path)


class TestCsvMatrix:
    def test_basic_read(self, tmp_path):
        path = tmp_path / "m.csv"
        path.write_text("1,2\n3,4\n")
        assert np.array_equal(read_csv_matrix(path), [[1.0, 2.0], [3.0, 4.0]])

    @pytest.mark.parametrize("text,line", [("1,2\n3\n", 2), ("1,2\n3,x\n", 2), ("1,2\n\n3,4\n", 2),
                                           ("1,2\n3,4\n5,6,7\n", 3), ("1,0x10\n", 1),
                                           ("1,2\n3,\n", 2), ("1,2\n3,1__0\n", 2)])
    def test_errors_report_line(self, tmp_path, text, line):
        path = tmp_path / "bad.csv"
        path.write_text(text)
        with pytest.raises(FormatError, match=f"line {line}"):
            read_csv_matrix(path)

    def test_header_skipped(self, tmp_path):
        path = tmp_path / "h.csv"
        path.write_text("a,b\n1,2\n")
        assert np.array_equal(read_csv_matrix(path, has_header=True), [[1.0, 2.0]])

    @pytest.mark.parametrize("text,header", [("", False), ("a,b\n", True), ("\n", False)])
    def test_no_data_rows(self, tmp_path, text, header):
        path = tmp_path / "e.csv"
        path.write_text(text)
        with pytest.raises(FormatError, match="no data rows"):
            read_csv_matrix(path, has_header=header)

    def test_python_float_syntax(self, tmp_path):
        """The accepted field syntax and the values are Python float()'s."""
        fields = [" 1.5 ", "1_000", "+.5", "5.", "-0", "1e400", "-inf", "Infinity", "NaN",
                  '"2.25"', "7e-400", "\t3\t", "0.1", "123456789012345678901234567890"]
        path = tmp_path / "s.csv"
        path.write_text(",".join(fields) + "\r\n" + ",".join(fields) + "\n")
        got = read_csv_matrix(path)
        want = np.array([float(f.strip('"')) for f in fields])
        assert got.shape == (2, len(fields))
        assert np.array_equal(got[0], want, equal_nan=True)
        assert np.array_equal(np.signbit(got[0]), np.signbit(want))

    def test_round_trip_exact_threads(self, tmp_path):
        path = tmp_path / "round.csv"
        matrix = np.random.default_rng(0).standard_normal((20000, 10)) * 10.0 ** \
            np.random.default_rng(1).integers(-300, 300, (20000, 10))
        write_csv_matrix(matrix, path)
        for t in (1, 7, 0):
            assert np.array_equal(read_csv_matrix(path, threads=t), matrix)

    def test_first_error_in_file_order(self, tmp_path):
        """Errors in several thread ranges: the lowest line is reported."""
        rows = [f"{i},{i + 0.5}" for i in range(20000)]
        rows[15000] = "1,x"
        rows[9000] = "1"
        path = tmp_path / "two.csv"
        path.write_text("\n".join(rows) + "\n")
        with pytest.raises(FormatError, match="ragged row at line 9001: expected 2 fields, got 1"):
            read_csv_matrix(path, threads=8)


@pytest.mark.gpu
@pytest.mark.parametrize("count,h,w", [(2, 2, 2), (5000, 28, 28), (20000, 28, 28)])
def test_idx_device_loader(cuda, tmp_path, count, h, w):
    """u8 streamed through pinned chunks and widened on the device == the
    reference's float64 host matrix, exactly; fp32 with a scale too."""
    import torch
    from paper_2007_11919_b200.dataio import load_idx_images
    rng = np.random.default_rng(count)
    pix = rng.integers(0, 256, (count, h, w), dtype=np.uint8)
    path = tmp_path / "img.idx"
    path.write_bytes(struct.pack(">IIII", 0x00000803, count, h, w) + pix.tobytes())
    images = read_idx_images(path)
    d64 = load_idx_images(path)
    assert d64.dtype == torch.float64 and d64.is_cuda
    assert np.array_equal(d64.cpu().numpy(), images.to_data_matrix())
    d32 = images.to_device(dtype=torch.float32, scale=1.0 / 255.0)
    ref = (pix.reshape(count, -1).astype(np.float64) * (1.0 / 255.0)).astype(np.float32)
    assert np.array_equal(d32.cpu().numpy(), ref)


REF_SRC = "/root/reference/pkg/src"


@pytest.mark.skipif(not __import__("os").path.isdir(REF_SRC), reason="reference sources absent")
def test_csv_fuzz_against_reference(tmp_path):
    """Random CSV texts (valid and broken) through the reference's
    read_csv_matrix (imported from the read-only tree, test-time only) and the
    native parser: same values, or FormatError on the same line."""
    import importlib
    import sys
    sys.path.insert(0, REF_SRC)
    try:
        ref = importlib.import_module("scalemds.dataio")
        ref_err = importlib.import_module("scalemds.errors").FormatError
    finally:
        sys.path.remove(REF_SRC)
    rng = np.random.default_rng(123)
    atoms = ["1", "-2.5", " 3 ", "4e3", "1_0", "x", "", "nan", "inf", '"5"', "0x1", "1__2", ".5",
             "6.", "-", "+7", "8e", "1e-5"]
    import re
    for trial in range(300):
        nrow, ncol = int(rng.integers(0, 5)), int(rng.integers(1, 4))
        lines = []
        for _ in range(nrow):
            w = ncol if rng.random() > 0.15 else int(rng.integers(0, 5))
            lines.append(",".join(atoms[int(rng.integers(0, len(atoms)))] if rng.random() < 0.2
                                  else f"{rng.standard_normal():.6g}" for _ in range(w)))
        text = "\n".join(lines) + ("\n" if rng.random() < 0.7 else "")
        header = bool(rng.random() < 0.2)
        path = tmp_path / f"f{trial}.csv"
        path.write_text(text)
        try:
            want = ref.read_csv_matrix(path, has_header=header)
            werr = None
        except ref_err as e:
            want, werr = None, str(e)
        try:
            got = read_csv_matrix(path, has_header=header)
            gerr = None
        except FormatError as e:
            got, gerr = None, str(e)
        if werr is None:
            assert gerr is None, (text, gerr)
            assert np.array_equal(got, want, equal_nan=True), text
        else:
            assert gerr is not None, (text, werr)
            wl = re.search(r"line (\d+)", werr)
            gl = re.search(r"line (\d+)", gerr)
            assert (wl and gl and wl.group(1) == gl.group(1)) or (not wl and not gl), (text, werr, gerr)
