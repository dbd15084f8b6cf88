// Dense row-major array of 32- or 64-bit reals, resident in device memory.
//
// Same value-type contract as the reference Tensor (proj/include/bcad/
// tensor.hpp:12-69): copyable (deep copy, device-to-device), single writer,
// no views. The storage lives in HBM, allocated stream-ordered from the
// device's caching pool through the C-ABI (bcad_cu_malloc); host access is
// explicit (from / to_host) or element-wise. Element reads go through a
// cached host window of the tensor (up to 64 Ki elements around the index,
// downloaded once) that stays valid until the next library call that can
// write device memory (errors.hpp device_generation) or a writable
// device_data() access, so reference-style loops over elements cost one
// copy per window, not one per element. Code that writes a tensor's device
// memory OUTSIDE this library (its own kernels through a pointer taken
// earlier) must call device_data() again, or invalidate_host_view(), before
// reading elements.
#pragma once

#include <cstdint>
#include <cstring>
#include <memory>
#include <mutex>
#include <ostream>
#include <span>
#include <vector>

#include "bcad/errors.hpp"
#include "bcad/rng.hpp"
#include "bcad/shape.hpp"

namespace bcad {

template <class T> struct dtype_of;
template <> struct dtype_of<float> { static constexpr int value = BCAD_CU_F32; };
template <> struct dtype_of<double> { static constexpr int value = BCAD_CU_F64; };

// The stream every device tensor and tape of this thread enqueues on
// (nullptr = the legacy default stream).
inline void*& current_stream() {
    static thread_local void* s = nullptr;
    return s;
}

// RAII scope that redirects the current stream.
class StreamGuard {
public:
    explicit StreamGuard(void* s) : prev_(current_stream()) { current_stream() = s; }
    ~StreamGuard() { current_stream() = prev_; }
    StreamGuard(const StreamGuard&) = delete;
    StreamGuard& operator=(const StreamGuard&) = delete;

private:
    void* prev_;
};

// Copies of one kind (0 host->device, 1 device->host, 2 device->device)
// collected and enqueued with ONE call (bcad_cu_memcpy_batch): a
// cudaMemcpyAsync costs 4-6 us of host time on B200, a batch of host
// transfers ~3.5 us in all, and device copies go out as one copy kernel.
// Submitted on destruction if not before.
class CopyBatch {
public:
    explicit CopyBatch(int kind) : kind_(kind) {}
    CopyBatch(const CopyBatch&) = delete;
    CopyBatch& operator=(const CopyBatch&) = delete;
    ~CopyBatch() {
        if (!dst_.empty()) {
            advance_device_generation();
            bcad_cu_memcpy_batch(dst_.size(), dst_.data(), src_.data(), size_.data(), kind_, current_stream());
        }
    }
    void add(void* dst, const void* src, std::size_t bytes) {
        dst_.push_back(dst);
        src_.push_back(src);
        size_.push_back(bytes);
    }
    void submit(void* stream) {
        if (!dst_.empty()) check(bcad_cu_memcpy_batch(dst_.size(), dst_.data(), src_.data(), size_.data(), kind_, stream));
        dst_.clear();
        src_.clear();
        size_.clear();
    }

private:
    int kind_;
    std::vector<void*> dst_;
    std::vector<const void*> src_;
    std::vector<std::size_t> size_;
};

namespace detail {

// Cached host copy of a window of a tensor's elements (element reads).
template <class T>
struct HostView {
    std::mutex mu;
    std::uint64_t generation = 0;  // 0: empty
    std::int64_t begin = 0;
    std::vector<T> data;
};

struct DeviceBuffer {
    void* ptr = nullptr;
    void* stream = nullptr;
    DeviceBuffer(std::size_t bytes, void* s) : stream(s) { check(bcad_cu_malloc(&ptr, bytes, s)); }
    ~DeviceBuffer() { bcad_cu_free(ptr, stream); }
    DeviceBuffer(const DeviceBuffer&) = delete;
    DeviceBuffer& operator=(const DeviceBuffer&) = delete;
};

}  // namespace detail

template <class T>
class Tensor {
public:
    using value_type = T;

    Tensor() : Tensor(Shape{}) {}
    explicit Tensor(Shape shape, T fill = T(0)) : shape_(std::move(shape)) {
        allocate();
        check(bcad_cu_fill(dtype_of<T>::value, buf_->ptr, volume(), static_cast<double>(fill), stream()));
    }

    // Allocation without initialisation (the device kernels overwrite it).
    static Tensor uninitialized(Shape shape) {
        Tensor t(NoInit{}, std::move(shape));
        return t;
    }

    static Tensor scalar(T value) { return Tensor(Shape{}, value); }

    static Tensor from(Shape shape, const std::vector<T>& data) {
        if (static_cast<std::int64_t>(data.size()) != shape.volume())
            throw ShapeMismatch("tensor data length " + std::to_string(data.size()) + " does not match shape " +
                                shape.str());
        return from_host(std::move(shape), data.data());
    }

    // Upload `shape.volume()` values from host memory (pinned memory makes
    // the copy asynchronous; pageable memory is staged by the driver).
    static Tensor from_host(Shape shape, const T* data) {
        Tensor t(NoInit{}, std::move(shape));
        check(bcad_cu_memcpy(t.buf_->ptr, data, t.bytes(), 0, t.stream()));
        return t;
    }

    // Deep copy of `shape.volume()` values already in device memory.
    static Tensor from_device(Shape shape, const T* data) {
        Tensor t(NoInit{}, std::move(shape));
        t.copy_in_device(data);
        return t;
    }

    Tensor(const Tensor& o) : shape_(o.shape_) {
        allocate();
        copy_in_device(o.buf_->ptr);
    }
    Tensor& operator=(const Tensor& o) {
        if (this != &o) *this = Tensor(o);
        return *this;
    }
    Tensor(Tensor&&) noexcept = default;
    Tensor& operator=(Tensor&&) noexcept = default;

    const Shape& shape() const { return shape_; }
    std::int64_t volume() const { return shape_.volume(); }
    std::size_t bytes() const { return static_cast<std::size_t>(volume()) * sizeof(T); }
    // A writable pointer may be used to change the contents: the cached host
    // view of the elements is dropped.
    T* device_data() {
        invalidate_host_view();
        return static_cast<T*>(buf_->ptr);
    }
    const T* device_data() const { return static_cast<const T*>(buf_->ptr); }
    void invalidate_host_view() const {
        if (view_) {
            std::lock_guard<std::mutex> lock(view_->mu);
            view_->generation = 0;
        }
    }
    void* stream() const { return buf_ ? buf_->stream : current_stream(); }

    void copy_to_host(T* dst) const {
        check(bcad_cu_memcpy(dst, buf_->ptr, bytes(), 1, stream()));
        check(bcad_cu_stream_synchronize(stream()));
    }
    std::vector<T> to_host() const {
        std::vector<T> h(static_cast<std::size_t>(volume()));
        copy_to_host(h.data());
        return h;
    }

    // Synchronous single-element access (reference element semantics,
    // tensor.hpp:40-51; a test / oracle convenience, not a hot path): a read
    // is one device->host copy, a write one host->device copy, each
    // synchronised on the tensor's stream.
    // Writable access (operator[] / at on an lvalue) goes through an
    // ElementRef; const and temporary tensors return the value, so no
    // reference can outlive its tensor.
    T operator[](std::int64_t flat) const& { return read(flat); }
    T operator[](std::int64_t flat) && { return read(flat); }
    T at(std::span<const std::int64_t> index) const& { return read(flat_index(index)); }
    T at(std::span<const std::int64_t> index) && { return read(flat_index(index)); }
    T at(std::initializer_list<std::int64_t> index) const& {
        return read(flat_index(std::span<const std::int64_t>(index.begin(), index.size())));
    }
    T at(std::initializer_list<std::int64_t> index) && {
        return read(flat_index(std::span<const std::int64_t>(index.begin(), index.size())));
    }

    class ElementRef {
    public:
        ElementRef(Tensor* t, std::int64_t flat) : t_(t), flat_(flat) {}
        operator T() const { return t_->read(flat_); }  // NOLINT: reads like the reference's Real&
        ElementRef& operator=(T v) {
            t_->write(flat_, v);
            return *this;
        }
        ElementRef& operator=(const ElementRef& o) { return *this = static_cast<T>(o); }
        ElementRef& operator+=(T v) { return *this = static_cast<T>(*this) + v; }
        ElementRef& operator-=(T v) { return *this = static_cast<T>(*this) - v; }
        ElementRef& operator*=(T v) { return *this = static_cast<T>(*this) * v; }

    private:
        Tensor* t_;
        std::int64_t flat_;
    };
    ElementRef operator[](std::int64_t flat) & { return ElementRef(this, flat); }
    ElementRef at(std::span<const std::int64_t> index) & { return ElementRef(this, flat_index(index)); }
    ElementRef at(std::initializer_list<std::int64_t> index) & {
        return ElementRef(this, flat_index(std::span<const std::int64_t>(index.begin(), index.size())));
    }

    void write_csv(std::ostream& os) const {  // tensor.hpp:53-61
        const std::vector<T> h = to_host();
        os << "# shape " << shape_.str() << "\n";
        const std::int64_t row = shape_.rank() > 0 ? shape_.dim(shape_.rank() - 1) : 1;
        for (std::int64_t i = 0; i < volume(); ++i) {
            os << h[static_cast<std::size_t>(i)];
            os << ((i % row == row - 1) ? '\n' : ',');
        }
    }

private:
    std::int64_t flat_index(std::span<const std::int64_t> index) const {
        std::int64_t flat = 0;
        for (int k = 0; k < shape_.rank(); ++k) flat = flat * shape_.dim(k) + index[static_cast<std::size_t>(k)];
        return flat;
    }
    static constexpr std::int64_t kViewWindow = std::int64_t(1) << 16;

    T read(std::int64_t flat) const {
        if (!view_) view_ = std::make_unique<detail::HostView<T>>();
        detail::HostView<T>& v = *view_;
        std::lock_guard<std::mutex> lock(v.mu);
        const std::uint64_t gen = device_generation().load(std::memory_order_relaxed);
        if (v.generation != gen || flat < v.begin || flat >= v.begin + static_cast<std::int64_t>(v.data.size())) {
            // the window around `flat` (the whole tensor when it is small)
            const std::int64_t vol = volume();
            const std::int64_t w = vol < kViewWindow ? vol : kViewWindow;
            std::int64_t b = flat - w / 2;
            if (b < 0) b = 0;
            if (b > vol - w) b = vol - w;
            v.data.resize(static_cast<std::size_t>(w));
            check_read(bcad_cu_memcpy(v.data.data(), static_cast<const T*>(buf_->ptr) + b, static_cast<std::size_t>(w) * sizeof(T),
                                      1, stream()));
            check_read(bcad_cu_stream_synchronize(stream()));
            v.begin = b;
            v.generation = gen;
        }
        return v.data[static_cast<std::size_t>(flat - v.begin)];
    }
    void write(std::int64_t flat, T x) {
        check_read(bcad_cu_memcpy(static_cast<T*>(buf_->ptr) + flat, &x, sizeof(T), 0, stream()));
        check_read(bcad_cu_stream_synchronize(stream()));
        if (view_) {  // keep a current view coherent (this write is the only change)
            std::lock_guard<std::mutex> lock(view_->mu);
            const std::int64_t o = flat - view_->begin;
            if (view_->generation == device_generation().load(std::memory_order_relaxed) && o >= 0 &&
                o < static_cast<std::int64_t>(view_->data.size()))
                view_->data[static_cast<std::size_t>(o)] = x;
        }
    }

    // device->device through the copy kernel (a launch is cheaper on the host
    // than a cudaMemcpyAsync)
    void copy_in_device(const void* src) {
        void* d = buf_->ptr;
        const std::size_t b = bytes();
        check(bcad_cu_memcpy_batch(1, &d, &src, &b, 2, stream()));
    }

    struct NoInit {};
    Tensor(NoInit, Shape shape) : shape_(std::move(shape)) { allocate(); }
    void allocate() { buf_ = std::make_unique<detail::DeviceBuffer>(bytes(), current_stream()); }

    Shape shape_;
    std::unique_ptr<detail::DeviceBuffer> buf_;
    mutable std::unique_ptr<detail::HostView<T>> view_;  // element reads
};

// Host-generated, bit-identical to the reference's inputs (tensor.hpp:71-84).
template <class T>
Tensor<T> random_pm1(Shape shape, Rng& rng) {
    std::vector<T> h(static_cast<std::size_t>(shape.volume()));
    for (T& v : h) v = static_cast<T>(rng.uniform_pm1());
    return Tensor<T>::from(std::move(shape), h);
}

template <class T>
Tensor<T> random_binary(Shape shape, Rng& rng, double p_one = 0.5) {
    std::vector<T> h(static_cast<std::size_t>(shape.volume()));
    for (T& v : h) v = static_cast<T>(rng.binary(p_one));
    return Tensor<T>::from(std::move(shape), h);
}

}  // namespace bcad
