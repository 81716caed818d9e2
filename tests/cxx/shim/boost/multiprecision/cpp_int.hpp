// cpp_int.hpp -- a minimal arbitrary-precision unsigned integer standing in for
// boost::multiprecision::cpp_int in the reference's test oracles (proj/tests/oracles.hpp:
// construction from integers, +=, *, *=, % u64, explicit conversion to u64).  Boost is not
// in this image.  TEST INFRASTRUCTURE ONLY.
#pragma once
#include <cstdint>
#include <vector>

namespace boost {
namespace multiprecision {

class cpp_int {
  public:
    cpp_int() = default;
    cpp_int(unsigned long long v) { set(v); }
    cpp_int(unsigned long v) { set(v); }
    cpp_int(unsigned v) { set(v); }
    cpp_int(long long v) { set(static_cast<unsigned long long>(v)); }
    cpp_int(long v) { set(static_cast<unsigned long long>(v)); }
    cpp_int(int v) { set(static_cast<unsigned long long>(v)); }

    cpp_int& operator+=(const cpp_int& o) {
        if (o.limbs_.size() > limbs_.size()) limbs_.resize(o.limbs_.size(), 0);
        unsigned long long carry = 0;
        for (size_t i = 0; i < limbs_.size(); ++i) {
            const unsigned long long s = (unsigned long long)limbs_[i] + (i < o.limbs_.size() ? o.limbs_[i] : 0) + carry;
            limbs_[i] = uint32_t(s);
            carry = s >> 32;
        }
        if (carry) limbs_.push_back(uint32_t(carry));
        return *this;
    }
    friend cpp_int operator*(const cpp_int& a, const cpp_int& b) {
        cpp_int r;
        if (a.limbs_.empty() || b.limbs_.empty()) return r;
        r.limbs_.assign(a.limbs_.size() + b.limbs_.size(), 0);
        for (size_t i = 0; i < a.limbs_.size(); ++i) {
            unsigned long long carry = 0;
            for (size_t j = 0; j < b.limbs_.size(); ++j) {
                const unsigned long long t =
                    (unsigned long long)a.limbs_[i] * b.limbs_[j] + r.limbs_[i + j] + carry;
                r.limbs_[i + j] = uint32_t(t);
                carry = t >> 32;
            }
            size_t k = i + b.limbs_.size();
            while (carry) {
                const unsigned long long t = (unsigned long long)r.limbs_[k] + carry;
                r.limbs_[k++] = uint32_t(t);
                carry = t >> 32;
            }
        }
        r.trim();
        return r;
    }
    cpp_int& operator*=(const cpp_int& o) { return *this = *this * o; }
    friend cpp_int operator+(cpp_int a, const cpp_int& b) { return a += b; }
    // remainder by a 64-bit modulus: Horner over the limbs with a 128-bit accumulator
    friend cpp_int operator%(const cpp_int& a, unsigned long long m) {
        unsigned __int128 r = 0;
        for (size_t i = a.limbs_.size(); i-- > 0;) r = ((r << 32) | a.limbs_[i]) % m;
        return cpp_int(static_cast<unsigned long long>(r));
    }
    friend cpp_int operator%(const cpp_int& a, unsigned long m) { return a % (unsigned long long)m; }
    friend cpp_int operator%(const cpp_int& a, unsigned m) { return a % (unsigned long long)m; }
    friend cpp_int operator%(const cpp_int& a, int m) { return a % (unsigned long long)m; }
    friend bool operator==(const cpp_int& a, const cpp_int& b) { return a.limbs_ == b.limbs_; }
    friend bool operator<(const cpp_int& a, const cpp_int& b) {
        if (a.limbs_.size() != b.limbs_.size()) return a.limbs_.size() < b.limbs_.size();
        for (size_t i = a.limbs_.size(); i-- > 0;)
            if (a.limbs_[i] != b.limbs_[i]) return a.limbs_[i] < b.limbs_[i];
        return false;
    }
    explicit operator unsigned long long() const {
        unsigned long long v = 0;
        for (size_t i = 0; i < limbs_.size() && i < 2; ++i) v |= (unsigned long long)limbs_[i] << (32 * i);
        return v;
    }
    explicit operator unsigned long() const { return (unsigned long)(unsigned long long)(*this); }

  private:
    void set(unsigned long long v) {
        limbs_.clear();
        while (v) {
            limbs_.push_back(uint32_t(v));
            v >>= 32;
        }
    }
    void trim() {
        while (!limbs_.empty() && limbs_.back() == 0) limbs_.pop_back();
    }
    std::vector<uint32_t> limbs_;  // little-endian base 2^32, no leading zero limbs
};

}  // namespace multiprecision
}  // namespace boost
