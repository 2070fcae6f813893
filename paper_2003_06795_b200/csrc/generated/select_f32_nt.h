#ifndef SELECT_F32_NT_H
#define SELECT_F32_NT_H

#include <stdint.h>

typedef struct {
    uint32_t acc;
    uint32_t row_tile;
    uint32_t col_tile;
    uint32_t wg_rows;
    uint32_t wg_cols;
} select_f32_nt_config;

static inline select_f32_nt_config select_f32_nt(int64_t m, int64_t k, int64_t n) {
    (void)m;
    (void)k;
    (void)n;
    if (m < INT64_C(2218)) {
        if (m < INT64_C(12)) {
            if (n < INT64_C(2024)) {
                if (k < INT64_C(2897)) {
                    select_f32_nt_config out = {8u, 1u, 1u, 8u, 8u};
                    return out;
                } else {
                    if (m < INT64_C(3)) {
                        select_f32_nt_config out = {8u, 1u, 1u, 8u, 8u};
                        return out;
                    } else {
                        select_f32_nt_config out = {4u, 1u, 1u, 8u, 8u};
                        return out;
                    }
                }
            } else {
                if (m < INT64_C(6)) {
                    if (m < INT64_C(2)) {
                        select_f32_nt_config out = {4u, 1u, 1u, 8u, 8u};
                        return out;
                    } else {
                        select_f32_nt_config out = {8u, 1u, 1u, 8u, 8u};
                        return out;
                    }
                } else {
                    select_f32_nt_config out = {4u, 1u, 1u, 8u, 8u};
                    return out;
                }
            }
        } else {
            if (n < INT64_C(176)) {
                if (m < INT64_C(555)) {
                    if (m < INT64_C(80)) {
                        if (m < INT64_C(57)) {
                            select_f32_nt_config out = {4u, 1u, 1u, 8u, 8u};
                            return out;
                        } else {
                            select_f32_nt_config out = {4u, 2u, 2u, 8u, 8u};
                            return out;
                        }
                    } else {
                        if (n < INT64_C(144)) {
                            if (k < INT64_C(471)) {
                                if (m < INT64_C(159)) {
                                    select_f32_nt_config out = {8u, 1u, 1u, 8u, 8u};
                                    return out;
                                } else {
                                    if (m < INT64_C(278)) {
                                        select_f32_nt_config out = {4u, 2u, 1u, 8u, 8u};
                                        return out;
                                    } else {
                                        if (n < INT64_C(79)) {
                                            select_f32_nt_config out = {8u, 1u, 1u, 8u, 8u};
                                            return out;
                                        } else {
                                            select_f32_nt_config out = {4u, 2u, 1u, 8u, 8u};
                                            return out;
                                        }
                                    }
                                }
                            } else {
                                select_f32_nt_config out = {8u, 1u, 1u, 8u, 8u};
                                return out;
                            }
                        } else {
                            if (m < INT64_C(139)) {
                                if (k < INT64_C(744)) {
                                    select_f32_nt_config out = {4u, 2u, 1u, 8u, 8u};
                                    return out;
                                } else {
                                    select_f32_nt_config out = {8u, 1u, 1u, 8u, 8u};
                                    return out;
                                }
                            } else {
                                select_f32_nt_config out = {4u, 2u, 1u, 8u, 8u};
                                return out;
                            }
                        }
                    }
                } else {
                    if (k < INT64_C(222)) {
                        if (m < INT64_C(1109)) {
                            select_f32_nt_config out = {4u, 2u, 2u, 8u, 8u};
                            return out;
                        } else {
                            if (k < INT64_C(167)) {
                                select_f32_nt_config out = {4u, 2u, 2u, 8u, 8u};
                                return out;
                            } else {
                                if (n < INT64_C(46)) {
                                    select_f32_nt_config out = {4u, 1u, 1u, 8u, 8u};
                                    return out;
                                } else {
                                    select_f32_nt_config out = {4u, 2u, 2u, 8u, 8u};
                                    return out;
                                }
                            }
                        }
                    } else {
                        if (k < INT64_C(444)) {
                            if (k < INT64_C(314)) {
                                select_f32_nt_config out = {4u, 2u, 1u, 8u, 8u};
                                return out;
                            } else {
                                select_f32_nt_config out = {4u, 2u, 1u, 8u, 8u};
                                return out;
                            }
                        } else {
                            if (k < INT64_C(1052)) {
                                select_f32_nt_config out = {4u, 2u, 2u, 8u, 8u};
                                return out;
                            } else {
                                if (m < INT64_C(1109)) {
                                    select_f32_nt_config out = {4u, 2u, 1u, 8u, 8u};
                                    return out;
                                } else {
                                    select_f32_nt_config out = {4u, 2u, 2u, 8u, 8u};
                                    return out;
                                }
                            }
                        }
                    }
                }
            } else {
                if (m < INT64_C(448)) {
                    if (n < INT64_C(1012)) {
                        if (m < INT64_C(317)) {
                            if (k < INT64_C(1145)) {
                                if (n < INT64_C(444)) {
                                    if (m < INT64_C(139)) {
                                        select_f32_nt_config out = {8u, 1u, 1u, 8u, 8u};
                                        return out;
                                    } else {
                                        if (m < INT64_C(224)) {
                                            if (k < INT64_C(182)) {
                                                select_f32_nt_config out = {4u, 2u, 1u, 8u, 8u};
                                                return out;
                                            } else {
                                                if (k < INT64_C(725)) {
                                                    select_f32_nt_config out = {4u, 2u, 2u, 8u, 8u};
                                                    return out;
                                                } else {
                                                    select_f32_nt_config out = {4u, 2u, 1u, 8u, 8u};
                                                    return out;
                                                }
                                            }
                                        } else {
                                            select_f32_nt_config out = {8u, 1u, 1u, 8u, 8u};
                                            return out;
                                        }
                                    }
                                } else {
                                    if (m < INT64_C(70)) {
                                        select_f32_nt_config out = {4u, 1u, 1u, 8u, 8u};
                                        return out;
                                    } else {
                                        select_f32_nt_config out = {4u, 2u, 2u, 8u, 8u};
                                        return out;
                                    }
                                }
                            } else {
                                if (k < INT64_C(2173)) {
                                    if (m < INT64_C(29)) {
                                        select_f32_nt_config out = {4u, 2u, 1u, 8u, 8u};
                                        return out;
                                    } else {
                                        if (m < INT64_C(99)) {
                                            select_f32_nt_config out = {4u, 1u, 1u, 8u, 8u};
                                            return out;
                                        } else {
                                            select_f32_nt_config out = {4u, 2u, 1u, 8u, 8u};
                                            return out;
                                        }
                                    }
                                } else {
                                    if (m < INT64_C(70)) {
                                        select_f32_nt_config out = {8u, 1u, 1u, 8u, 8u};
                                        return out;
                                    } else {
                                        if (m < INT64_C(139)) {
                                            select_f32_nt_config out = {4u, 1u, 1u, 8u, 8u};
                                            return out;
                                        } else {
                                            if (k < INT64_C(3259)) {
                                                select_f32_nt_config out = {4u, 1u, 1u, 8u, 8u};
                                                return out;
                                            } else {
                                                select_f32_nt_config out = {4u, 2u, 1u, 8u, 8u};
                                                return out;
                                            }
                                        }
                                    }
                                }
                            }
                        } else {
                            if (n < INT64_C(544)) {
                                select_f32_nt_config out = {4u, 2u, 2u, 8u, 8u};
                                return out;
                            } else {
                                if (k < INT64_C(124)) {
                                    select_f32_nt_config out = {8u, 4u, 4u, 8u, 8u};
                                    return out;
                                } else {
                                    select_f32_nt_config out = {8u, 4u, 4u, 16u, 8u};
                                    return out;
                                }
                            }
                        }
                    } else {
                        if (m < INT64_C(70)) {
                            if (k < INT64_C(405)) {
                                select_f32_nt_config out = {4u, 2u, 1u, 8u, 8u};
                                return out;
                            } else {
                                select_f32_nt_config out = {4u, 2u, 2u, 8u, 8u};
                                return out;
                            }
                        } else {
                            if (k < INT64_C(287)) {
                                select_f32_nt_config out = {8u, 4u, 4u, 16u, 8u};
                                return out;
                            } else {
                                if (m < INT64_C(139)) {
                                    if (k < INT64_C(405)) {
                                        select_f32_nt_config out = {4u, 2u, 2u, 8u, 8u};
                                        return out;
                                    } else {
                                        select_f32_nt_config out = {8u, 4u, 4u, 16u, 8u};
                                        return out;
                                    }
                                } else {
                                    if (n < INT64_C(1145)) {
                                        select_f32_nt_config out = {4u, 2u, 2u, 8u, 8u};
                                        return out;
                                    } else {
                                        if (m < INT64_C(278)) {
                                            select_f32_nt_config out = {8u, 4u, 4u, 8u, 8u};
                                            return out;
                                        } else {
                                            if (k < INT64_C(573)) {
                                                select_f32_nt_config out = {8u, 4u, 4u, 16u, 8u};
                                                return out;
                                            } else {
                                                select_f32_nt_config out = {8u, 4u, 4u, 8u, 8u};
                                                return out;
                                            }
                                        }
                                    }
                                }
                            }
                        }
                    }
                } else {
                    if (n < INT64_C(1145)) {
                        if (n < INT64_C(351)) {
                            if (m < INT64_C(1109)) {
                                if (n < INT64_C(287)) {
                                    select_f32_nt_config out = {4u, 2u, 2u, 8u, 8u};
                                    return out;
                                } else {
                                    select_f32_nt_config out = {8u, 4u, 4u, 16u, 8u};
                                    return out;
                                }
                            } else {
                                select_f32_nt_config out = {8u, 4u, 4u, 8u, 8u};
                                return out;
                            }
                        } else {
                            if (n < INT64_C(992)) {
                                select_f32_nt_config out = {8u, 4u, 4u, 8u, 8u};
                                return out;
                            } else {
                                if (m < INT64_C(896)) {
                                    select_f32_nt_config out = {8u, 4u, 4u, 8u, 8u};
                                    return out;
                                } else {
                                    if (m < INT64_C(1268)) {
                                        select_f32_nt_config out = {8u, 4u, 4u, 16u, 8u};
                                        return out;
                                    } else {
                                        select_f32_nt_config out = {8u, 8u, 4u, 16u, 8u};
                                        return out;
                                    }
                                }
                            }
                        }
                    } else {
                        select_f32_nt_config out = {8u, 4u, 4u, 16u, 8u};
                        return out;
                    }
                }
            }
        }
    } else {
        if (m < INT64_C(3584)) {
            if (n < INT64_C(444)) {
                if (k < INT64_C(46)) {
                    if (k < INT64_C(28)) {
                        select_f32_nt_config out = {8u, 4u, 4u, 16u, 8u};
                        return out;
                    } else {
                        select_f32_nt_config out = {8u, 8u, 4u, 16u, 8u};
                        return out;
                    }
                } else {
                    select_f32_nt_config out = {8u, 4u, 4u, 16u, 8u};
                    return out;
                }
            } else {
                if (k < INT64_C(111)) {
                    select_f32_nt_config out = {8u, 4u, 4u, 16u, 8u};
                    return out;
                } else {
                    if (k < INT64_C(363)) {
                        select_f32_nt_config out = {8u, 8u, 4u, 16u, 8u};
                        return out;
                    } else {
                        if (k < INT64_C(1087)) {
                            select_f32_nt_config out = {8u, 8u, 8u, 16u, 8u};
                            return out;
                        } else {
                            select_f32_nt_config out = {8u, 8u, 4u, 16u, 8u};
                            return out;
                        }
                    }
                }
            }
        } else {
            if (k < INT64_C(544)) {
                if (m < INT64_C(17740)) {
                    if (n < INT64_C(136)) {
                        if (k < INT64_C(168)) {
                            select_f32_nt_config out = {8u, 4u, 4u, 16u, 8u};
                            return out;
                        } else {
                            if (m < INT64_C(8870)) {
                                if (n < INT64_C(91)) {
                                    select_f32_nt_config out = {8u, 8u, 4u, 16u, 8u};
                                    return out;
                                } else {
                                    select_f32_nt_config out = {8u, 4u, 4u, 16u, 8u};
                                    return out;
                                }
                            } else {
                                if (n < INT64_C(91)) {
                                    if (k < INT64_C(222)) {
                                        select_f32_nt_config out = {8u, 8u, 4u, 16u, 8u};
                                        return out;
                                    } else {
                                        select_f32_nt_config out = {8u, 4u, 4u, 16u, 8u};
                                        return out;
                                    }
                                } else {
                                    select_f32_nt_config out = {8u, 8u, 4u, 16u, 8u};
                                    return out;
                                }
                            }
                        }
                    } else {
                        if (k < INT64_C(46)) {
                            if (m < INT64_C(8870)) {
                                select_f32_nt_config out = {8u, 8u, 4u, 16u, 8u};
                                return out;
                            } else {
                                select_f32_nt_config out = {8u, 8u, 8u, 16u, 8u};
                                return out;
                            }
                        } else {
                            select_f32_nt_config out = {8u, 8u, 4u, 16u, 8u};
                            return out;
                        }
                    }
                } else {
                    if (k < INT64_C(96)) {
                        if (m < INT64_C(35480)) {
                            if (n < INT64_C(46)) {
                                select_f32_nt_config out = {8u, 4u, 4u, 16u, 8u};
                                return out;
                            } else {
                                select_f32_nt_config out = {8u, 8u, 4u, 16u, 8u};
                                return out;
                            }
                        } else {
                            select_f32_nt_config out = {8u, 8u, 4u, 16u, 8u};
                            return out;
                        }
                    } else {
                        if (m < INT64_C(70960)) {
                            if (k < INT64_C(146)) {
                                if (m < INT64_C(35480)) {
                                    select_f32_nt_config out = {8u, 4u, 4u, 16u, 8u};
                                    return out;
                                } else {
                                    select_f32_nt_config out = {8u, 8u, 4u, 16u, 8u};
                                    return out;
                                }
                            } else {
                                select_f32_nt_config out = {8u, 8u, 4u, 16u, 8u};
                                return out;
                            }
                        } else {
                            select_f32_nt_config out = {8u, 8u, 8u, 16u, 8u};
                            return out;
                        }
                    }
                }
            } else {
                if (m < INT64_C(141920)) {
                    if (n < INT64_C(91)) {
                        if (m < INT64_C(17740)) {
                            if (m < INT64_C(8870)) {
                                select_f32_nt_config out = {8u, 8u, 4u, 16u, 8u};
                                return out;
                            } else {
                                select_f32_nt_config out = {8u, 4u, 4u, 16u, 8u};
                                return out;
                            }
                        } else {
                            if (m < INT64_C(35480)) {
                                select_f32_nt_config out = {8u, 8u, 4u, 16u, 8u};
                                return out;
                            } else {
                                if (m < INT64_C(70960)) {
                                    select_f32_nt_config out = {8u, 8u, 8u, 16u, 8u};
                                    return out;
                                } else {
                                    select_f32_nt_config out = {8u, 8u, 4u, 16u, 8u};
                                    return out;
                                }
                            }
                        }
                    } else {
                        if (m < INT64_C(17740)) {
                            if (n < INT64_C(182)) {
                                select_f32_nt_config out = {8u, 8u, 4u, 16u, 8u};
                                return out;
                            } else {
                                if (m < INT64_C(5069)) {
                                    select_f32_nt_config out = {8u, 8u, 8u, 16u, 8u};
                                    return out;
                                } else {
                                    select_f32_nt_config out = {8u, 8u, 4u, 16u, 8u};
                                    return out;
                                }
                            }
                        } else {
                            if (m < INT64_C(35480)) {
                                select_f32_nt_config out = {8u, 8u, 8u, 16u, 8u};
                                return out;
                            } else {
                                if (m < INT64_C(70960)) {
                                    if (n < INT64_C(182)) {
                                        select_f32_nt_config out = {8u, 8u, 4u, 16u, 8u};
                                        return out;
                                    } else {
                                        select_f32_nt_config out = {8u, 8u, 8u, 16u, 8u};
                                        return out;
                                    }
                                } else {
                                    select_f32_nt_config out = {8u, 8u, 8u, 16u, 8u};
                                    return out;
                                }
                            }
                        }
                    }
                } else {
                    select_f32_nt_config out = {8u, 8u, 8u, 16u, 8u};
                    return out;
                }
            }
        }
    }
}

#endif /* SELECT_F32_NT_H */
